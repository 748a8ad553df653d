AB_TEST="tests/test_gpu_backward.py" bash scripts/gpu_ab.sh ss "base=" "unroll7=-DSK_SSIM_UNROLL=7" "unroll4=-DSK_SSIM_UNROLL=4" > gpurun_out/ab_ss.txt 2>&1; cat gpurun_out/ab_ss.txt
