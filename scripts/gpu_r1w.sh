AB_TEST="tests/test_gpu_backward.py tests/test_golden.py" bash scripts/gpu_ab.sh k9 "base=" "nopf=-DSK_K9_PREFETCH=0" "pf2=-DSK_K9_PREFETCH=2" > gpurun_out/ab_k9.txt 2>&1; cat gpurun_out/ab_k9.txt
