AB_TEST="tests/test_gpu_backward.py" bash scripts/gpu_ab.sh ssim "base=" "ty32=-DSK_SSIM_TY=32" > gpurun_out/ab_ssim.txt 2>&1; cat gpurun_out/ab_ssim.txt
