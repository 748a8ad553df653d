#!/bin/bash
# Round-2 parity gates on the B200: the new scale / capped-branch tests with
# the unfloored error report collected into gpurun_out/parity_report.jsonl.
set -x
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.build()"
rm -f gpurun_out/parity_report.jsonl
SK_PARITY_REPORT=gpurun_out/parity_report.jsonl timeout 1500 python -m pytest tests/test_gpu_parity_scale.py -x -q -m gpu -rA ${PYTEST_ARGS} 2>&1 | tail -40
