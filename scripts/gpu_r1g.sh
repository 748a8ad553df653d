timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r1g.log 2>&1; tail -3 gpurun_out/pytest_r1g.log
timeout 600 python bench.py > gpurun_out/bench_r1g.json 2> gpurun_out/bench_r1g.err; tail -c 400 gpurun_out/bench_r1g.err
SK_TRACE_EVENTS=1 timeout 600 python bench.py --workload event --no-cpu-baseline --steps 3 > gpurun_out/event_r1g.json 2> gpurun_out/event_r1g.err
grep "\[event\]" gpurun_out/event_r1g.err | tail -20
AB_TEST="tests/test_gpu_forward.py" bash scripts/gpu_ab.sh sort "base=" "ballot=-DSK_SORT_BALLOT_RANK=1" > gpurun_out/ab_sort.txt 2>&1; cat gpurun_out/ab_sort.txt
