"""Edge cases of the training path through the C ABI: empty and fully culled
scenes, one Gaussian covering every tile, images smaller than a tile, tile
sizes 8 and 32, and a non-square view — each step must match the oracle's
render bit for bit and produce finite gradients."""
import numpy as np
import pytest

from tests.util import random_scene, ring_camera, synthetic_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2511_04283_b200 as sk
    sk.build()
    c = sk.Context(0)
    yield c
    c.close()


def _render_both(ctx, orc, p, deg, cam, b):
    ref = orc.render_scene(p, deg, cam, b)
    scene = ctx.scene(p, deg)
    ctx.preprocess(scene, cam, b)
    pairs = ctx.build_tile_grid()
    got = ctx.blend_forward()
    assert pairs == ref.pairs
    assert np.array_equal(got.image, ref.image)
    assert np.array_equal(got.transmittance, ref.transmittance)
    return got, scene


def test_empty_and_culled_scenes(ctx, orc):
    cam = orc.default_camera(40, 24)
    p = random_scene(np.random.default_rng(1), 0, 1)
    got, _ = _render_both(ctx, orc, p, 1, cam, orc.binning())
    assert not got.image.any() and (got.transmittance == 1).all()
    p = random_scene(np.random.default_rng(2), 50, 1)
    p[2] = -5.0  # behind the camera: every Gaussian culled at the near plane
    got, scene = _render_both(ctx, orc, p, 1, cam, orc.binning())
    assert not got.image.any()
    v = ctx.training_loss(np.full((24, 40, 3), 0.5, np.float32), 0.2)
    assert np.isfinite(v.loss)
    g = ctx.blend_backward()
    assert not g.d_mu2d.any()


@pytest.mark.parametrize("ts", [8, 16, 32])
def test_one_gaussian_covering_every_tile(ctx, orc, ts):
    p = random_scene(np.random.default_rng(3), 1, 0)
    p[0:3, 0] = [0.0, 0.0, 3.0]
    p[7:10, 0] = np.log(2.0)  # huge: its 3-sigma box covers the whole view
    p[10, 0] = 2.0
    cam = orc.default_camera(70, 45)
    got, _ = _render_both(ctx, orc, p, 0, cam, orc.binning(tile_size=ts))
    assert got.contrib.sum() > 0.5 * got.contrib.size
    ctx.training_loss(np.zeros((45, 70, 3), np.float32), 0.2)
    g = ctx.blend_backward()
    assert np.isfinite(g.d_mu2d).all() and np.abs(g.d_color).sum() > 0


@pytest.mark.parametrize("w,h", [(5, 3), (17, 9), (333, 61)])
def test_small_and_odd_images(ctx, orc, w, h):
    p = synthetic_scene(600, deg=1, seed=4)
    cam = ring_camera(orc, w, h, 0.5)
    for ts in (8, 16):
        _render_both(ctx, orc, p, 1, cam, orc.binning(tile_size=ts))


def test_train_step_tile32_nonsquare(ctx, orc):
    """A full host-input training step at tile size 32 on a 200x120 view (the
    bench path uses 16): loss finite and equal to the oracle's render loss."""
    import paper_2511_04283_b200 as sk
    p = synthetic_scene(3000, deg=3, seed=5)
    cam = ring_camera(orc, 200, 120, 1.3)
    gt = np.clip(orc.render_scene(synthetic_scene(3000, deg=3, seed=6), 3, cam).image * 255 + 0.5, 0, 255)
    gt = gt.astype(np.uint8)
    cfg = sk.default_config()
    cfg.tile_size = 32
    scene = ctx.scene(p, 3)
    row = sk.train_step_host(ctx, scene, cam, gt, cfg, 3.0, 1)
    ref = orc.render_scene(p, 3, cam, orc.binning(tile_size=32))
    loss_ref, _, _, _ = orc.training_loss(ref.image, gt.astype(np.float32) / np.float32(255), 0.2)
    assert row["loss"] == pytest.approx(loss_ref, rel=1e-3)
    after = scene.download()
    assert np.isfinite(after).all() and not np.array_equal(after, p)
