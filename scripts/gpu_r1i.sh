timeout 600 python scripts/diag_e2e.py > gpurun_out/diag_e2e.txt 2>&1; cat gpurun_out/diag_e2e.txt | tail -6
bash scripts/gpu_profile.sh r1i "tests/test_gpu_backward.py tests/test_gpu_pipeline.py" 150
