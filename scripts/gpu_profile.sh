# One GPU call: parity tests, bench lines, ncu launch list + full-set capture
# of the steady-state training step (after WARM warm-up iterations, the state
# bench.py's timed region sees).
# usage: bash scripts/gpu_profile.sh <tag> [pytest-selection] [warm]
TAG=${1:-r1}
SEL=${2:-tests}
WARM=${3:-150}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt
timeout 900 python -m pytest $SEL -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 600 gpurun_out/bench_$TAG.err
timeout 600 python bench.py --workload event --no-cpu-baseline --steps 3 > gpurun_out/event_$TAG.json 2> gpurun_out/event_$TAG.err; tail -c 600 gpurun_out/event_$TAG.err
# launch list around the first timed iteration after WARM warm-ups (19 launches per step)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -s $((19 * WARM)) -c 60 \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --profile --steps 2 --warmup $WARM > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"blend_fwd|blend_bwd" -s $((2 * WARM + 1)) -c 2 \
  -o gpurun_out/full_$TAG -f python bench.py --profile --steps 2 --warmup $WARM > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"preprocess|duplicate|onesweep|ssim|project_bwd|adam|scan_gather|tile_ranges" -s $((14 * WARM + 10)) -c 14 \
  -o gpurun_out/fullb_$TAG -f python bench.py --profile --steps 1 --warmup $WARM > gpurun_out/ncu_fullb_$TAG.log 2>&1
tail -n 2 gpurun_out/ncu_full_$TAG.log gpurun_out/ncu_fullb_$TAG.log
