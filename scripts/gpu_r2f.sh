timeout 900 python -m pytest tests/test_gpu_density.py tests/test_gpu_trainer_options.py tests/test_cli.py -m gpu -x -q 2>&1 | tail -2
for v in 1 0; do
  SK_NVCC_EXTRA="-DSK_SCORE_TWO_STREAMS=$v" python -c "import paper_2511_04283_b200 as sk; sk.build(force=True)"
  timeout 600 python bench.py --workload event --no-cpu-baseline --steps 3 > gpurun_out/event_ts$v.json 2>/dev/null
  python -c "import json; e=json.load(open('gpurun_out/event_ts$v.json')); print('two_streams=$v', round(e['value'],2), round(e['late_event_ms'],2), e['early']['phase_ms'], e['n_after_early'], e['n_after_late'])"
done
python -c "import paper_2511_04283_b200 as sk; sk.build(force=True)"
