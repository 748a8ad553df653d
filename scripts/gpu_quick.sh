#!/bin/bash
# Quick GPU iteration: build, the tests in $TESTS, then the phase split of
# the config-2 step (bench --profile: no baselines, no event).
python -c "import __graft_entry__ as g; g.build()" || exit 1
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest $TESTS -x -q -m gpu 2>&1 | tail -${TAIL:-8}; fi
timeout 600 python bench.py --profile --steps ${STEPS:-30} --warmup 5 --no-event 2>&1 | tail -2
