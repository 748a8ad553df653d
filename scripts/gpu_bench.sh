#!/bin/bash
# The driver's two bench arms at N=1 (reference first), plus the GPU tests
# named in $TESTS (default: none).
python -c "import __graft_entry__ as g; g.build()" || exit 1
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest $TESTS -x -q -m gpu 2>&1 | tail -15; fi
( time timeout 900 python bench.py --impl reference --gpus 1 --steps ${STEPS:-20} --warmup ${WARMUP:-5} ) > gpurun_out/ref1.out 2> gpurun_out/ref1.err
( time timeout 900 python bench.py --gpus 1 --steps ${STEPS:-20} --warmup ${WARMUP:-5} ) > gpurun_out/n1.out 2> gpurun_out/n1.err
tail -3 gpurun_out/ref1.err gpurun_out/n1.err
cat gpurun_out/ref1.out gpurun_out/n1.out
