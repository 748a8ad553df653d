AB_TEST="tests/test_gpu_backward.py tests/test_gpu_density.py" bash scripts/gpu_ab.sh basync "base=" "nobasync=-DSK_BWD_ASYNC_GATHER=0" > gpurun_out/ab_basync.txt 2>&1; cat gpurun_out/ab_basync.txt
