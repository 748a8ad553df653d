#!/bin/bash
# ncu --set full of one launch of the kernels matching $KERNELS at the bench's
# fixed start state (timed iteration $ITER, 1-based, after --warmup 3 and the
# restore; ncu replays each kernel, never a bench number).
# usage: KERNELS=blend_bwd TAG=r2a bash scripts/gpu_ncu.sh
python -c "import __graft_entry__ as g; g.build()" || exit 1
TAG=${TAG:-r2}
ITER=${ITER:-1}
K=${KERNELS:-blend_bwd}
# launches of each kernel before the timed iteration: the warm-up steps (3)
SKIP=$((3 + ITER - 1))
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"$K" -s $SKIP -c ${COUNT:-1} \
  -o gpurun_out/full_$TAG -f python bench.py --profile --steps $ITER --warmup 3 --no-event > gpurun_out/ncu_$TAG.log 2>&1
tail -n 3 gpurun_out/ncu_$TAG.log
