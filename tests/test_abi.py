"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/*.h declares (no compute calls: no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    syms = set()
    for name in os.listdir(os.path.join(ROOT, "include")):
        if not name.endswith(".h"):
            continue
        text = open(os.path.join(ROOT, "include", name)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(sk_[a-z0-9_]+)\s*\(", text):
            syms.add(m.group(1))
    return syms


@pytest.fixture(scope="module")
def libsk():
    import paper_2511_04283_b200 as pkg
    pkg.build()
    return ctypes.CDLL(pkg.LIB_PATH)


def test_library_exports_every_declared_symbol(libsk):
    syms = _declared_symbols()
    assert len(syms) > 20
    missing = [s for s in sorted(syms) if not hasattr(libsk, s)]
    assert not missing, missing


def test_version_string(libsk):
    libsk.sk_version.restype = ctypes.c_char_p
    assert b"sm_100a" in libsk.sk_version()


def test_null_arguments_are_rejected_without_a_gpu(libsk):
    assert libsk.sk_scene_size(None, None) != 0
    assert libsk.sk_frame_num_projected(None, None) != 0


def test_sass_targets_sm100a():
    import shutil
    import subprocess
    import paper_2511_04283_b200 as pkg
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", pkg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_train_config_layout_matches_oracle():
    import ctypes
    import paper_2511_04283_b200 as sk
    from oracle import oracle as orc
    a, b = sk.SkTrainConfig, orc.OrTrainConfig
    assert ctypes.sizeof(a) == ctypes.sizeof(b)
    for (na, ta), (nb, tb) in zip(a._fields_, b._fields_):
        assert na == nb and getattr(a, na).offset == getattr(b, nb).offset
