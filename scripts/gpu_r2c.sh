AB_TEST="tests/test_gpu_backward.py tests/test_gpu_density.py" bash scripts/gpu_ab.sh bl "base=" "branchless=-DSK_BWD_BRANCHLESS=1" > gpurun_out/ab_bl.txt 2>&1; cat gpurun_out/ab_bl.txt
