AB_TEST="tests/test_gpu_forward.py" bash scripts/gpu_ab.sh bin "base=" "hagg=-DSK_HIST_AGG=1" "nodup=-DSK_DUP_RCP=0" > gpurun_out/ab_bin.txt 2>&1; cat gpurun_out/ab_bin.txt
