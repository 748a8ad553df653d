#!/bin/bash
# GPU test suite (or the files in $TESTS) on the B200, with the parity report.
python -c "import __graft_entry__ as g; g.build()" || exit 1
rm -f gpurun_out/parity_report.jsonl
SK_PARITY_REPORT=gpurun_out/parity_report.jsonl timeout ${TMO:-2400} python -m pytest ${TESTS:-tests} -x -q -m gpu ${PYTEST_ARGS} 2>&1 | tail -${TAIL:-30}
