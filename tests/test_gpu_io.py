"""Checkpoint PLY and dataset directories through device-resident scenes and
datasets; ports tests/test_dataset.cpp's checkpoint and
load_dataset cases."""
import os

import numpy as np
import pytest

from tests.util import random_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2511_04283_b200 as sk
    sk.build()
    c = sk.Context(0)
    yield c
    c.close()


def _ref_rows(p, deg):
    """save_checkpoint's row layout (ply.hpp:227-246) from planar params."""
    n = p.shape[1]
    nsh = (deg + 1) ** 2
    cols = [p[0], p[1], p[2], np.zeros(n), np.zeros(n), np.zeros(n)]
    cols += [p[11 + c] for c in range(3)]
    cols += [p[11 + 3 * m + c] for c in range(3) for m in range(1, nsh)]
    cols += [p[10], p[7], p[8], p[9], p[3], p[4], p[5], p[6]]
    return np.stack(cols, 1).astype(np.float32)


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_checkpoint_round_trip_exact(ctx, tmp_path, deg):
    """test_dataset.cpp:109-128 / 130-143 / 145-170: exact at float32, the
    header the reference writes, no f_rest at degree 0, body = n x props x 4."""
    import paper_2511_04283_b200 as sk
    rng = np.random.default_rng(102 + deg)
    n = 17 if deg != 3 else 5003
    p = random_scene(rng, n, deg)
    scene = ctx.scene(p, deg, capacity=2 * n)
    path = tmp_path / "checkpoint.ply"
    scene.save_checkpoint(path)
    data = path.read_bytes()
    head, body = data.split(b"end_header\n", 1)
    lines = head.decode().splitlines()
    props = [ln.split()[2] for ln in lines if ln.startswith("property ")]
    nsh = (deg + 1) ** 2
    assert f"element vertex {n}" in lines
    assert props[:9] == ["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"]
    assert props[9:9 + 3 * (nsh - 1)] == [f"f_rest_{i}" for i in range(3 * (nsh - 1))]
    assert props[9 + 3 * (nsh - 1):] == ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2",
                                         "rot_3"]
    assert len(body) == n * len(props) * 4
    assert np.array_equal(np.frombuffer(body, np.float32).reshape(n, -1), _ref_rows(p, deg))
    back = sk.Scene.load_checkpoint(ctx, path)
    assert back.sh_degree == deg and back.size == n
    assert np.array_equal(back.download(), p)
    # byte-deterministic
    scene.save_checkpoint(tmp_path / "again.ply")
    assert (tmp_path / "again.ply").read_bytes() == data


def test_checkpoint_ascii_and_missing_field(ctx, tmp_path):
    import paper_2511_04283_b200 as sk
    p = tmp_path / "bad.ply"
    p.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 1\n"
                  b"property float x\nproperty float y\nproperty float z\nend_header\n" + bytes(12))
    with pytest.raises(sk.SplatError, match="missing property '"):
        sk.Scene.load_checkpoint(ctx, p)
    # ASCII degree-0 checkpoint with a double column takes the generic path
    names = ["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1",
             "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
    vals = [[0.5, -1, 2, 0, 0, 0, 0.1, 0.2, 0.3, -0.4, -3, -2.5, -2, 1, 0, 0, 0]]
    txt = "ply\nformat ascii 1.0\nelement vertex 1\n" + "".join(
        f"property {'double' if k == 'opacity' else 'float'} {k}\n" for k in names) + "end_header\n"
    txt += " ".join(str(v) for v in vals[0]) + "\n"
    a = tmp_path / "a.ply"
    a.write_text(txt)
    s = sk.Scene.load_checkpoint(ctx, a)
    got = s.download()[:, 0]
    want = np.array([0.5, -1, 2, 1, 0, 0, 0, -3, -2.5, -2, -0.4, 0.1, 0.2, 0.3], np.float32)
    assert s.sh_degree == 0 and np.array_equal(got, want)
    bad = tmp_path / "rest.ply"
    bad.write_text(txt.replace("property float rot_3\n", "property float rot_3\nproperty float f_rest_0\n")
                   .replace(" 0\n", " 0 0\n"))
    with pytest.raises(sk.SplatError, match="f_rest count must be divisible by 3"):
        sk.Scene.load_checkpoint(ctx, bad)


def test_dataset_save_load_idempotent(ctx, tmp_path):
    """test_dataset.cpp:50-62 and 223-251: synthetic dataset -> files ->
    load_dataset: cameras, every-8th split, 8-bit images and points survive."""
    import paper_2511_04283_b200 as sk
    ds, gt, xyz, rgb = sk.Dataset.synthetic(ctx, n_gaussians=20, n_views=9, width=32, seed=1)
    d1 = tmp_path / "d1"
    ds.save(d1)
    assert sorted(os.listdir(d1 / "images")) == [f"{i:05d}.png" for i in range(9)]
    back = sk.Dataset.load(ctx, d1)
    assert back.num_views == 9
    assert back.train_indices().tolist() == [1, 2, 3, 4, 5, 6, 7]
    assert back.extent > 1.0
    for v in range(9):
        a, b = ds.camera(v), back.camera(v)
        assert np.abs(np.array(a.world_to_cam) - np.array(b.world_to_cam)).max() < 1e-6
        assert (a.fx, a.cx, a.width, a.height) == (b.fx, b.cx, b.width, b.height)
        assert np.array_equal(ds.image_u8(v), back.image_u8(v))
        assert np.array_equal(sk.read_png(d1 / "images" / f"{v:05d}.png"), ds.image_u8(v))
    bx, brgb = back.init_points()
    assert np.array_equal(bx, xyz) and np.abs(brgb - rgb).max() <= 0.5 / 255 + 1e-6
    # load -> save -> load is idempotent on the parsed values
    d2 = tmp_path / "d2"
    back.save(d2)
    again = sk.Dataset.load(ctx, d2)
    for v in range(9):
        assert np.array_equal(again.image_u8(v), back.image_u8(v))
        assert list(again.camera(v).world_to_cam) == list(back.camera(v).world_to_cam)
    assert again.extent == back.extent
    assert (d1 / "cameras.json").read_bytes() == (d2 / "cameras.json").read_bytes()


def test_dataset_loader_errors(ctx, tmp_path):
    """test_dataset.cpp:199-221: missing cameras.json, wrong image size."""
    import paper_2511_04283_b200 as sk
    with pytest.raises(sk.SplatError, match="cameras.json"):
        sk.Dataset.load(ctx, tmp_path)
    ds, _, _, _ = sk.Dataset.synthetic(ctx, n_gaussians=5, n_views=2, width=16, seed=1)
    ds.save(tmp_path)
    sk.write_png(tmp_path / "images" / "00000.png", np.zeros((8, 8, 3), np.float32))
    with pytest.raises(sk.SplatError, match="8x8"):
        sk.Dataset.load(ctx, tmp_path)
    sk.write_png(tmp_path / "images" / "00000.png", ds.image_u8(0))
    os.remove(tmp_path / "images" / "00001.png")
    with pytest.raises(sk.SplatError, match="missing image"):
        sk.Dataset.load(ctx, tmp_path)


def test_trained_scene_checkpoint_renders_identically(ctx, tmp_path, orc):
    """A checkpoint written from the device reloads bit-identically and renders
    the same image through the GPU path and the oracle."""
    import paper_2511_04283_b200 as sk
    from tests.util import ring_camera, synthetic_scene
    p = synthetic_scene(3000, deg=3, seed=9)
    scene = ctx.scene(p, 3)
    scene.save_checkpoint(tmp_path / "c.ply")
    back = sk.Scene.load_checkpoint(ctx, tmp_path / "c.ply")
    cam = ring_camera(orc, 96, 64, 1.0)
    ctx.preprocess(back, cam)
    ctx.build_tile_grid()
    got = ctx.blend_forward()
    ref = orc.render_scene(p, 3, cam)
    assert np.array_equal(got.image, ref.image)
