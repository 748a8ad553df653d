bash scripts/gpu_ab.sh bwd "base=" "minb10=-DSK_BWD_MINB=10" "minb12=-DSK_BWD_MINB=12" > gpurun_out/ab_bwd.txt 2>&1
cat gpurun_out/ab_bwd.txt
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_io.py tests/test_gpu_density.py -m gpu -x -q > gpurun_out/pytest_r1c.log 2>&1; tail -5 gpurun_out/pytest_r1c.log
timeout 600 python bench.py --workload event --no-cpu-baseline --steps 3 > gpurun_out/event_r1c.json 2> gpurun_out/event_r1c.err; tail -c 1500 gpurun_out/event_r1c.json
