#!/bin/bash
# A/B of run-time environment variants: for each "name=VAR=value ..." argument
# run the config-2 phase split (bench --profile). usage:
#   bash scripts/gpu_envab.sh "base=" "c1k=SK_BIN_CHUNK=1024"
python -c "import __graft_entry__ as g; g.build()" || exit 1
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest $TESTS -x -q -m gpu 2>&1 | tail -${TAIL:-4}; fi
for spec in "$@"; do
  name=${spec%%=*}; envs=${spec#*=}
  echo -n "$name: "
  env $envs timeout 300 python bench.py --profile --steps ${STEPS:-30} --warmup 5 --no-event 2>&1 | tail -1
done
