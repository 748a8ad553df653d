#!/bin/bash
# Launch list (ncu duration + DRAM bytes) of $STEPS timed bench iterations,
# summarised per launch. CC=none keeps caches warm between kernels (as in a
# real step); the default flushes them (cold, ncu's default).
# usage: TAG=x STEPS=3 [CC=none] bash scripts/gpu_launches.sh
python -c "import __graft_entry__ as g; g.build()" || exit 1
TAG=${TAG:-ll}
timeout 900 ncu --profile-from-start off --clock-control none --cache-control ${CC:-all} \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --profile --steps ${STEPS:-3} --warmup 5 --no-event > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_$TAG.csv | tail -30
