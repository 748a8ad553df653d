"""Trainer options off the default path on the GPU:
the lazy SH-rest schedule (trainer.hpp:160-169, adam.hpp:146-159) and the
opacity reset (trainer.hpp:104-106, 245-249), against the oracle trainer.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2511_04283_b200 as sk
    sk.build()
    c = sk.Context(0)
    yield c
    c.close()


def _setup(ctx, orc, lazy, reset_every):
    import paper_2511_04283_b200 as sk
    ds = orc.Dataset(1500, 8, 96, seed=4)
    xyz, rgb = ds.points()
    p0 = orc.init_from_points(xyz, rgb, 3)
    cfg = sk.default_config()
    cfg.iterations = 30000
    cfg.densify_from = cfg.densify_until = 1 << 30  # no density events in this window
    cfg.prune_every_late = 1 << 30
    cfg.lazy_opt_enabled = int(lazy)
    cfg.opacity_reset_every = reset_every
    ocfg = orc.default_config()
    for name, _ in ocfg._fields_:
        setattr(ocfg, name, getattr(cfg, name))
    cams = [ds.camera(v) for v in range(ds.num_views)]
    imgs = [ds.image_u8(v) for v in range(ds.num_views)]
    data = sk.Dataset(ctx, cams, imgs, ds.train_indices(), ds.extent)
    scene = ctx.scene(p0, 3)
    tr = sk.Trainer(ctx, scene, data, cfg)
    otr = orc.Trainer(p0, 3, ds, ocfg)
    return tr, otr, scene, data, ds, p0


def test_lazy_sh_rest_schedule(ctx, orc):
    """From iteration 15000 the SH-rest group steps only every 32 iterations,
    on the gradient accumulated since the last step."""
    tr, otr, scene, data, ds, p0 = _setup(ctx, orc, lazy=True, reset_every=0)
    rest = slice(11 + 3, None)
    tr.set_iteration(15010)
    otr.set_iteration(15010)
    tr.run(29)  # 15011 .. 15039: no SH-rest update
    p = scene.download()
    assert np.array_equal(p[rest], p0[rest])
    assert not np.array_equal(p[:11], p0[:11])
    tr.run(1)  # 15040: due
    p40 = scene.download()
    assert not np.array_equal(p40[rest], p0[rest])
    tr.run(31)  # 15041 .. 15071: unchanged again
    assert np.array_equal(scene.download()[rest], p40[rest])
    tr.run(1)  # 15072
    assert not np.array_equal(scene.download()[rest], p40[rest])
    otr.run(62)
    ref = otr.scene()
    got = scene.download()
    # same schedule on both sides; trajectories agree to the blend-gradient tolerance
    d = np.abs(got - ref).max(axis=1)
    assert d[rest].max() < 2e-3 and d[:11].max() < 2e-2, d


def test_opacity_reset(ctx, orc):
    import math
    tr, otr, scene, data, ds, p0 = _setup(ctx, orc, lazy=False, reset_every=20)
    cap = np.float32(math.log(np.float32(0.01) / (np.float32(1) - np.float32(0.01))))
    tr.run(19)
    assert scene.download()[10].max() > cap
    tr.run(1)  # iteration 20: step, then reset
    op = scene.download()[10]
    assert op.max() <= cap
    otr.run(20)
    ref = otr.scene()[10]
    assert np.abs(op - ref).max() < 1e-3
    # the opacity group's moments restart from zero (Adam's first step is +-lr)
    m, v, t = scene.adam_state()
    assert np.all(m[10][: scene.size] == 0) and np.all(v[10][: scene.size] == 0)
