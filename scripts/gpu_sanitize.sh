#!/bin/bash
# compute-sanitizer over the library's kernels (memcheck, racecheck, synccheck).
python -c "import __graft_entry__ as g; g.build()" || exit 1
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  ( time timeout 1200 compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 20 \
      python tests/tools/sanitizer_workload.py ${PART:-all} ) > gpurun_out/san_$tool.log 2>&1
  echo "rc=$?"
  tail -25 gpurun_out/san_$tool.log
done
