timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r1h.log 2>&1; tail -3 gpurun_out/pytest_r1h.log
timeout 600 python bench.py > gpurun_out/bench_r1h.json 2> gpurun_out/bench_r1h.err; tail -c 400 gpurun_out/bench_r1h.err
SK_TRACE_EVENTS=1 timeout 600 python bench.py --workload event --no-cpu-baseline --steps 3 > gpurun_out/event_r1h.json 2> gpurun_out/event_r1h.err
grep "\[event\]" gpurun_out/event_r1h.err | tail -11
