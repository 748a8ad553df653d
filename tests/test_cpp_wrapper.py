"""The splat:: C++ surface (include/splatkit_b200.hpp) over the C ABI: the
reference's own densify / prune, optimizer and trainer KATs
(tests/test_adc.cpp:39-332, test_adam.cpp:13-97, test_trainer.cpp:60-137),
ported onto this API in tests/cpp/test_api_kats.cpp, compile here and pass on
the GPU."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    import paper_2511_04283_b200 as sk
    sk.build()
    cxx = shutil.which("g++")
    if cxx is None:
        pytest.skip("no g++")
    exe = os.path.join(str(tmp_path), "test_api_kats")
    libdir = os.path.dirname(sk.LIB_PATH)
    cmd = [cxx, "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_api_kats.cpp"), "-o", exe, "-L", libdir, "-lsplatkit_b200",
           f"-Wl,-rpath,{libdir}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_wrapper_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_wrapper_runs_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300, env=dict(os.environ, SK_TMP=str(tmp_path)))
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
