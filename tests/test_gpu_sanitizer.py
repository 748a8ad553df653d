"""compute-sanitizer over the library's kernels: memcheck,
racecheck and synccheck on a 4K-Gaussian training run, one density event
(two-stream score pass, selection, compaction) and a 200K-key depth sort
whose onesweep passes span 50+ tiles of decoupled look-back
(tests/tools/sanitizer_workload.py). Warp-private shared staging with
__syncwarp, cp.async double buffers and the relaxed look-back loads / stores
are exactly what racecheck and synccheck are for."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for cand in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if cand and os.path.exists(cand):
            return cand
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    import paper_2511_04283_b200 as sk
    sk.build()
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "7", "--print-limit", "20", sys.executable,
           os.path.join(ROOT, "tests", "tools", "sanitizer_workload.py"), "all"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "train+event ok" in out and "sort ok" in out, out[-2000:]
    summary = "0 hazards displayed (0 errors, 0 warnings)" if tool == "racecheck" else "ERROR SUMMARY: 0 errors"
    assert summary in out, out[-2000:]
