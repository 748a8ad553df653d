AB_TEST="tests/test_gpu_forward.py tests/test_golden.py" bash scripts/gpu_ab.sh fbl "base=" "fbranchless=-DSK_FWD_BRANCHLESS=1" > gpurun_out/ab_fbl.txt 2>&1; cat gpurun_out/ab_fbl.txt
