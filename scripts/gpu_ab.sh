# A/B of compile-time variants on one box: for each "name=flags" argument,
# rebuild with SK_NVCC_EXTRA=flags and run a short bench; then restore the
# default build. usage: bash scripts/gpu_ab.sh TAG "base=" "fast=-DSOME_FLAG=1" ...
TAG=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}
  SK_NVCC_EXTRA="$flags" python -c "import paper_2511_04283_b200 as sk; sk.build(force=True)" || continue
  if [ -n "$AB_TEST" ]; then
    timeout 600 python -m pytest $AB_TEST -m gpu -x -q 2>&1 | tail -1 | sed "s/^/$name tests: /"
  fi
  timeout 300 python bench.py --steps ${AB_STEPS:-100} --warmup ${AB_WARM:-100} --no-cpu-baseline > gpurun_out/ab_${TAG}_$name.json 2>/dev/null
  python - "$name" gpurun_out/ab_${TAG}_$name.json <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    print(sys.argv[1], round(d["value"], 1), "it/s", json.dumps(d["phase_ms"]))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
python -c "import paper_2511_04283_b200 as sk; sk.build(force=True)"
