AB_TEST="tests/test_gpu_forward.py tests/test_golden.py" bash scripts/gpu_ab.sh k1 "base=" "pf1=-DSK_K1_PREFETCH=1" "pf2=-DSK_K1_PREFETCH=2" > gpurun_out/ab_k1.txt 2>&1; cat gpurun_out/ab_k1.txt
