timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2a.log 2>&1; tail -2 gpurun_out/pytest_r2a.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
python -c "import json; d=json.load(open('gpurun_out/bench_r2a.json')); print(d['value'], d['e2e']['value'], d['phase_ms'])"
