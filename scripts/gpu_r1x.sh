AB_TEST="tests/test_gpu_backward.py tests/test_golden.py" bash scripts/gpu_ab.sh pf "base=" "k1pf3=-DSK_K1_PREFETCH=3" "k8pf=-DSK_BWD_L1PF=1" > gpurun_out/ab_pf.txt 2>&1; cat gpurun_out/ab_pf.txt
