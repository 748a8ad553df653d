# One GPU call: parity tests, bench lines, ncu launch list + full-set capture.
# usage: bash scripts/gpu_profile.sh <tag> [pytest-selection]
TAG=${1:-r1}
SEL=${2:-tests}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt
timeout 900 python -m pytest $SEL -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 600 gpurun_out/bench_$TAG.err
timeout 600 python bench.py --workload event --no-cpu-baseline --steps 3 > gpurun_out/event_$TAG.json 2> gpurun_out/event_$TAG.err; tail -c 600 gpurun_out/event_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"preprocess|duplicate|onesweep|blend_fwd|blend_bwd|ssim|project_bwd|adam" -s 14 -c 14 \
  -o gpurun_out/full_$TAG -f python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/ncu_full_$TAG.log
