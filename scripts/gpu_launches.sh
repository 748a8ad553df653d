#!/bin/bash
# ncu launch list (gpu__time_duration per kernel) of the bench's timed
# iteration 1 (after --warmup 3 and the restore). ncu numbers are
# cold-cache / serialised: shares, not bench values.
python -c "import __graft_entry__ as g; g.build()" || exit 1
TAG=${TAG:-r2}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --profile --steps 1 --warmup 3 --no-event > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_$TAG.csv | tail -30
