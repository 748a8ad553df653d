#!/bin/bash
# Round profile evidence at the bench's own settings (the driver runs
# `bench.py --steps 20 --warmup 5`; every run restores the same start state
# after warm-up, so the timed region is always training iterations 1..20).
# ncu runs with --profile-from-start off: bench.py --profile brackets exactly
# the timed iterations with cudaProfilerStart/Stop.
#   launch list : the 20 timed iterations (19 launches each), averaged per launch
#   full set    : iteration 1 (--steps 1), every kernel
#   usage: bash scripts/gpu_profile.sh <tag>
TAG=${1:-r2}
python -c "import __graft_entry__ as g; g.build()" || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
NCU="ncu --profile-from-start off --clock-control none"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --profile --steps 20 --warmup 5 --no-event > /dev/null 2>&1
timeout 1500 $NCU --set full --import-source on -o gpurun_out/full_$TAG -f \
  python bench.py --profile --steps 1 --warmup 5 --no-event > gpurun_out/ncu_full_$TAG.log 2>&1
tail -n 2 gpurun_out/ncu_full_$TAG.log
python scripts/ncu_summary.py launches gpurun_out/launches_$TAG.csv | tail -25
