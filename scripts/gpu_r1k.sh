timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r1k.log 2>&1; tail -3 gpurun_out/pytest_r1k.log
AB_TEST="tests/test_gpu_backward.py" bash scripts/gpu_ab.sh cm "base=" "nocmask=-DSK_BWD_USE_CMASK=0" "minb7=-DSK_BWD_MINB=7" "minb8=-DSK_BWD_MINB=8" > gpurun_out/ab_cm.txt 2>&1; cat gpurun_out/ab_cm.txt
