# Larger configurations (SURVEY §8 configs 4 and 5 geometry) on one GPU:
# short bench runs that check the path at 3M / 8M Gaussians.
mkdir -p gpurun_out
timeout 900 python bench.py --n 3000000 --width 1297 --height 840 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/scale_3m.json 2> gpurun_out/scale_3m.err; tail -c 300 gpurun_out/scale_3m.err
timeout 900 python bench.py --n 8000000 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/scale_8m.json 2> gpurun_out/scale_8m.err; tail -c 300 gpurun_out/scale_8m.err
timeout 900 python bench.py --workload event --n 3000000 --width 1297 --height 840 --views 64 --steps 2 --no-cpu-baseline > gpurun_out/scale_event_3m.json 2> gpurun_out/scale_event_3m.err; tail -c 300 gpurun_out/scale_event_3m.err
for f in scale_3m scale_8m scale_event_3m; do python -c "
import json,sys
d=json.load(open('gpurun_out/$f.json'))
print('$f', d['value'], d['unit'], d.get('phase_ms', d.get('early')), d.get('tile_pairs'), d.get('e2e'))
" 2>&1 | tail -1; done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
