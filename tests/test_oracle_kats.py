"""Pins the CPU oracle to the reference's own known-answer tests.

Each test names the reference test it ports (proj/tests/*.cpp). The oracle is
the checker for every GPU parity test, so it must reproduce these first.
"""
import math

import numpy as np
import pytest

pytestmark = []


def _scene_one(mu, deg=1, dc=(0.5, 0.5, 0.5), log_scale=(0.0, 0.0, 0.0), op_logit=0.0, rot=(1, 0, 0, 0)):
    from oracle.oracle import n_components
    p = np.zeros((n_components(deg), 1), np.float64)
    p[0:3, 0] = mu
    p[3:7, 0] = rot
    p[7:10, 0] = log_scale
    p[10, 0] = op_logit
    p[11:14, 0] = dc
    return p


# ---- detmath ----------------------------------------------------------------

def test_detmath_exp_log_within_2ulp(orc):
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(-87, 88, 20000), rng.uniform(-10, 10, 20000), np.linspace(-1, 1, 2001)])
    xs = xs.astype(np.float32)
    got = np.array([orc.lib().or_expf(float(x)) for x in xs], np.float32)
    ref = np.exp(xs.astype(np.float64)).astype(np.float32)
    ulp = np.abs(got.view(np.int32).astype(np.int64) - ref.view(np.int32).astype(np.int64))
    assert ulp.max() <= 2, ulp.max()
    ys = np.exp(rng.uniform(-80, 80, 20000)).astype(np.float32)
    got = np.array([orc.lib().or_logf(float(y)) for y in ys], np.float32)
    ref = np.log(ys.astype(np.float64)).astype(np.float32)
    ulp = np.abs(got.view(np.int32).astype(np.int64) - ref.view(np.int32).astype(np.int64))
    assert ulp.max() <= 3, ulp.max()
    assert orc.lib().or_expf(-200.0) == 0.0
    assert math.isinf(orc.lib().or_expf(100.0))


# ---- scene (tests/test_scene.cpp:14-74, acceptance.cpp:449-466) ---------------

def test_covariance_kats(orc):
    np.testing.assert_allclose(orc.covariance_3d([1, 0, 0, 0], [1, 1, 1]), np.eye(3), atol=1e-12)
    np.testing.assert_allclose(orc.covariance_3d([1, 0, 0, 0], [2, 1, 1]), np.diag([4, 1, 1]), atol=1e-12)
    r = math.sqrt(0.5)
    np.testing.assert_allclose(orc.covariance_3d([r, 0, 0, r], [2, 1, 1]), np.diag([1, 4, 1]), atol=1e-12)
    # spectrum = scale^2, double cover q / -q identical
    rng = np.random.default_rng(3)
    for _ in range(10):
        q = rng.normal(size=4)
        s = rng.uniform(0.1, 2, 3)
        c = orc.covariance_3d(q, s)
        np.testing.assert_allclose(np.sort(np.linalg.eigvalsh(c)), np.sort(s ** 2), atol=1e-9)
        assert np.array_equal(c, orc.covariance_3d(-q, s))
    with pytest.raises(ValueError):
        orc.covariance_3d([1, 0, 0, 0], [1, 0, 1])
    with pytest.raises(ValueError):
        orc.covariance_3d([1, 0, 0, 0], [1, np.nan, 1])


# ---- SH (tests/test_sh.cpp:11-46) ---------------------------------------------

def test_sh_kats(orc):
    c0 = 1 / (2 * math.sqrt(math.pi))
    sh = np.zeros((4, 3))
    assert np.allclose(orc.evaluate_sh(sh, 1, [0, 0, 1]), 0.5)
    sh[0] = 1.0
    np.testing.assert_allclose(orc.evaluate_sh(sh, 0, [0, 0, 1]), c0 + 0.5, rtol=1e-12)
    sh = np.zeros((4, 3))
    sh[2] = 1.0  # basis[2] = C1 z
    np.testing.assert_allclose(orc.evaluate_sh(sh, 1, [0, 0, 1]), 0.4886025119029199 + 0.5, rtol=1e-12)
    sh[2] = 2.0
    np.testing.assert_allclose(orc.evaluate_sh(sh, 1, [0, 0, -1]), 0.0, atol=1e-12)  # clamp at 0


# ---- camera (tests/test_camera.cpp:23-106) ------------------------------------

def test_project_principal_point_and_cov(orc):
    cam = orc.camera(64, 64, 100, 100, 32, 32)
    pr = orc.project_scene(_scene_one([0, 0, 5]), 1, cam, dtype=np.float64)
    assert pr.visible[0] == 1
    np.testing.assert_allclose(pr.mu2d[0], [32, 32])
    assert pr.depth[0] == pytest.approx(5.0)
    cam = orc.camera(64, 64, 120, 80, 31.5, 31.5)
    pr = orc.project_scene(_scene_one([0, 0, 4.0]), 1, cam, dtype=np.float64)
    jx, jy = 120 / 4.0, 80 / 4.0
    assert pr.cov2d[0, 0] == pytest.approx(jx * jx + 0.3, rel=1e-6)
    assert pr.cov2d[0, 3] == pytest.approx(jy * jy + 0.3, rel=1e-6)
    assert abs(pr.cov2d[0, 1]) < 1e-9


def test_project_culling(orc):
    cam = orc.default_camera()
    pr = orc.project_scene(np.concatenate([_scene_one([0, 0, 0.05]), _scene_one([0, 0, -3]),
                                           _scene_one([50, 0, 2], log_scale=[math.log(0.01)] * 3)], 1), 1, cam,
                           dtype=np.float64)
    assert list(pr.visible) == [0, 0, 0]


def test_cov_floor(orc):
    rng = np.random.default_rng(32)
    cam = orc.default_camera()
    n = 50
    p = np.zeros((orc.n_components(2), n))
    p[0] = rng.uniform(-0.6, 0.6, n)
    p[1] = rng.uniform(-0.6, 0.6, n)
    p[2] = rng.uniform(2, 5, n)
    q = rng.normal(size=(4, n))
    p[3:7] = q / np.linalg.norm(q, axis=0)
    p[7:10] = np.log(rng.uniform(0.03, 0.15, (3, n)))
    pr = orc.project_scene(p, 2, cam, dtype=np.float64)
    for i in np.nonzero(pr.visible)[0]:
        assert np.linalg.eigvalsh(pr.cov2d[i].reshape(2, 2)).min() >= 0.3 - 1e-9


# ---- binning (tests/test_raster.cpp:49-131, acceptance.cpp:528-543) --------------

def test_bin_aabb_kats(orc):
    b = orc.binning("aabb", tile_size=16)
    s = (2.0 / 3.0) ** 2
    cov = np.diag([s, s]).reshape(4)
    assert orc.bin_one([8, 8], cov, np.linalg.inv(cov.reshape(2, 2)).reshape(4), 0.5, 64, 64, b) == [0]
    cov = np.diag([1600.0, 1600.0]).reshape(4)
    assert len(orc.bin_one([32, 32], cov, np.linalg.inv(cov.reshape(2, 2)).reshape(4), 0.5, 64, 64, b)) == 16


def test_compact_threshold_kats(orc):
    e = 2.0 * math.log(0.9999 * 255.0)
    assert e == pytest.approx(11.082, rel=1e-3)
    assert orc.compact_threshold(0.9999, 1 / 255, 1.0) == pytest.approx(e, rel=1e-12)
    assert orc.compact_threshold(0.9999, 1 / 255, 0.5) == pytest.approx(5.541, rel=1e-3)
    b = orc.binning("compact")
    cov = np.diag([9.0, 9.0]).reshape(4)
    inv = np.diag([1 / 9.0, 1 / 9.0]).reshape(4)
    assert orc.bin_one([32, 32], cov, inv, 1 / 255, 64, 64, b) == []
    assert orc.bin_one([32, 32], cov, inv, 0.5 / 255, 64, 64, b) == []


def _pixel_level_bin(mu, conic, w, h, ts, maha):
    ys, xs = np.mgrid[0:h, 0:w]
    dx = xs - mu[0]
    dy = ys - mu[1]
    q = conic[0] * dx * dx + 2 * conic[1] * dx * dy + conic[3] * dy * dy
    tx = (w + ts - 1) // ts
    sel = q <= maha
    return set(((ys[sel] // ts) * tx + xs[sel] // ts).tolist())


def test_bin_compact_subset_monotone_cover(orc):
    rng = np.random.default_rng(42)
    for _ in range(60):
        pg = orc.random_projected(rng, 1, 80, 64, 0.98, 0.01)
        aabb = set(orc.bin_one(pg.mu2d[0], pg.cov2d[0], pg.conic[0], pg.opacity[0], 80, 64, orc.binning("aabb")))
        assert _pixel_level_bin(pg.mu2d[0], pg.conic[0], 80, 64, 16, 9.0) <= aabb
        prev = None
        for beta in (1.0, 0.9, 0.7, 0.4, 0.15):
            cur = set(orc.bin_one(pg.mu2d[0], pg.cov2d[0], pg.conic[0], pg.opacity[0], 80, 64,
                                  orc.binning("compact", beta=beta)))
            if beta == 1.0:
                assert cur <= aabb
                if pg.opacity[0] > 1 / 255:
                    a_star = min(orc.compact_threshold(pg.opacity[0], 1 / 255, 1.0), 9.0)
                    assert _pixel_level_bin(pg.mu2d[0], pg.conic[0], 80, 64, 16, a_star) <= cur
            if prev is not None:
                assert cur <= prev
            prev = cur


# ---- blend (tests/test_raster.cpp:133-192, acceptance.cpp:470-487) ---------------

def _pg_single(x, y, cov, op, color, depth):
    cov = np.asarray(cov, np.float64)
    inv = np.linalg.inv(cov)
    from oracle.oracle import PG
    return PG(np.array([[x, y]], float), cov.reshape(1, 4), inv.reshape(1, 4), np.array([depth], float),
              np.array([color], float), np.array([op], float))


def _cat(*pgs):
    from oracle.oracle import PG
    return PG(*(np.concatenate([getattr(p, f) for p in pgs]) for f in
                ("mu2d", "cov2d", "conic", "depth", "color", "opacity")))


def test_blend_single_capped(orc):
    c = [0.2, 0.7, 1.0]
    r = orc.render_pg(_pg_single(3, 3, np.eye(2), 0.9999, c, 1.0), 8, 8, orc.binning(tile_size=16))
    np.testing.assert_allclose(r.image[3, 3], 0.99 * np.array(c, np.float32), atol=1e-6)
    assert r.transmittance[3, 3] == pytest.approx(0.01, rel=1e-5)
    assert r.contrib[3, 3] == 1


def test_blend_two_term(orc):
    pg = _cat(_pg_single(3, 3, np.eye(2), 0.5, [1, 0, 0], 1.0), _pg_single(3, 3, np.eye(2), 0.5, [0, 1, 0], 2.0))
    pg.conic[:] = np.eye(2).reshape(4)
    r = orc.render_pg(pg, 8, 8, orc.binning(tile_size=8), dtype=np.float64)
    np.testing.assert_allclose(r.image[3, 3], [0.5, 0.25, 0], atol=1e-12)
    assert r.transmittance[3, 3] == pytest.approx(0.25)


def test_tiled_equals_brute_bitwise(orc):
    rng = np.random.default_rng(44)
    for _ in range(20):
        n = 1 + int(rng.integers(12))
        pg = orc.random_projected(rng, n, 32, 32, dtype=np.float32)
        t = orc.render_pg(pg, 32, 32)
        img, tr, cc, _ = orc.brute_render_pg(pg, 32, 32)
        assert np.array_equal(t.image, img)
        assert np.array_equal(t.transmittance, tr)
        assert np.array_equal(t.contrib, cc)


def test_footprint_counts_exact(orc):
    rng = np.random.default_rng(45)
    for _ in range(10):
        n = 2 + int(rng.integers(10))
        pg = orc.random_projected(rng, n, 32, 32, 0.9, dtype=np.float32)
        mask = (rng.uniform(size=(32, 32)) < 0.4).astype(np.uint8)
        t = orc.render_pg(pg, 32, 32, mask=mask)
        _, _, _, expected = orc.brute_render_pg(pg, 32, 32, mask=mask)
        assert np.array_equal(t.counts, expected)


def test_pairs_ordering_aabb_cb(orc):
    rng = np.random.default_rng(46)
    pg = orc.random_projected(rng, 60, 128, 128, 0.95, 0.02)
    p_aabb = orc.render_pg(pg, 128, 128, orc.binning("aabb"), dtype=np.float64).pairs
    p_cb1 = orc.render_pg(pg, 128, 128, orc.binning("compact", 1.0), dtype=np.float64).pairs
    p_cb08 = orc.render_pg(pg, 128, 128, orc.binning("compact", 0.8), dtype=np.float64).pairs
    assert p_cb08 <= p_cb1 <= p_aabb


def test_worker_independence(orc):
    rng = np.random.default_rng(49)
    pg = orc.random_projected(rng, 40, 64, 64, 0.9, dtype=np.float32)
    up = rng.uniform(-1, 1, (64, 64, 3)).astype(np.float32)
    ref = orc.render_pg(pg, 64, 64, workers=1)
    g1 = orc.blend_backward_pg(pg, 64, 64, up, workers=1)
    mask = np.ones((64, 64), np.uint8)
    c1 = orc.render_pg(pg, 64, 64, mask=mask, workers=1).counts
    for w in (2, 4):
        assert np.array_equal(orc.render_pg(pg, 64, 64, workers=w).image, ref.image)
        assert np.array_equal(orc.render_pg(pg, 64, 64, mask=mask, workers=w).counts, c1)
        g = orc.blend_backward_pg(pg, 64, 64, up, workers=w)
        # per-worker accumulators change the fp32 summation order (raster.hpp:352-353)
        assert np.abs(g.d_mu2d - g1.d_mu2d).max() < 1e-6 * max(1.0, np.abs(g1.d_mu2d).max())
        assert np.abs(g.d_opacity - g1.d_opacity).max() < 2e-6 * max(1.0, np.abs(g1.d_opacity).max())


# ---- finite differences (tests/test_raster.cpp:230-297) ----------------------------

def test_blend_backward_fd(orc):
    rng = np.random.default_rng(48)
    w = h = 16
    for _ in range(2):
        n = 4 + int(rng.integers(6))
        pg = orc.random_projected(rng, n, w, h, 0.8)
        up = rng.uniform(-1, 1, (h, w, 3))

        def loss(p):
            img, _, _, _ = orc.brute_render_pg(p, w, h, dtype=np.float64)
            return float((img * up).sum())

        g = orc.blend_backward_pg(pg, w, h, up, orc.binning(), dtype=np.float64)
        eps = 1e-5

        def fd(field, idx, sym=False):
            a = pg.astype(np.float64)
            b = pg.astype(np.float64)
            getattr(a, field)[idx] += eps
            getattr(b, field)[idx] -= eps
            if sym:
                i, k = idx
                getattr(a, field)[i, 2] += eps
                getattr(b, field)[i, 2] -= eps
            return (loss(a) - loss(b)) / (2 * eps)

        def rel(a, b):
            return abs(a - b) / max(abs(a), abs(b), 1e-7)

        for i in range(n):
            for d in range(2):
                assert rel(g.d_mu2d[i, d], fd("mu2d", (i, d))) < 1e-4
            assert rel(g.d_opacity[i], fd("opacity", i)) < 1e-4
            assert rel(g.d_conic[i, 1] + g.d_conic[i, 2], fd("conic", (i, 1), sym=True)) < 1e-4
            for c in range(3):
                assert rel(g.d_color[i, c], fd("color", (i, c))) < 1e-4


def test_abs_grad_cancellation(orc):
    """tests/test_raster.cpp:299-333."""
    pg = _pg_single(3.5, 3.0, np.eye(2) * 4.0, 0.5, [1, 1, 1], 1.0)
    up = np.zeros((8, 8, 3))
    up[3, 3] = 1
    up[3, 4] = 1
    g = orc.blend_backward_pg(pg, 8, 8, up, orc.binning(tile_size=8), dtype=np.float64)
    assert abs(g.d_mu2d[0, 0]) < 1e-12
    assert g.abs_grad[0, 0] > 1e-4


# ---- loss / metrics (tests/test_metrics_loss.cpp, acceptance.cpp:545-552) ---------

def test_psnr_ssim_kats(orc):
    a = np.zeros((4, 4, 3))
    b = np.zeros((4, 4, 3))
    assert orc.psnr(a, b, np.float64) == 100.0
    b[:] = 0.1
    assert orc.psnr(a, b, np.float64) == pytest.approx(20.0, abs=1e-9)
    x = np.random.default_rng(5).uniform(size=(16, 16, 3))
    assert orc.ssim(x, x, np.float64) == pytest.approx(1.0, abs=1e-12)


def test_loss_fd(orc):
    rng = np.random.default_rng(64)
    r = rng.uniform(size=(12, 10, 3))
    g = rng.uniform(size=(12, 10, 3))
    _, _, _, d = orc.training_loss(r, g, 0.2, np.float64)
    eps = 1e-6
    for (y, x, c) in [(0, 0, 0), (5, 4, 1), (11, 9, 2), (6, 0, 2), (3, 7, 0)]:
        a = r.copy()
        b = r.copy()
        a[y, x, c] += eps
        b[y, x, c] -= eps
        fd = (orc.training_loss(a, g, 0.2, np.float64)[0] - orc.training_loss(b, g, 0.2, np.float64)[0]) / (2 * eps)
        assert abs(fd - d[y, x, c]) / max(abs(fd), 1e-7) < 1e-4


# ---- error maps (tests/test_error_maps.cpp) -------------------------------------

def test_error_map_kats(orc):
    r = np.zeros((1, 2, 3))
    g = np.zeros((1, 2, 3))
    r[0, 0] = [0.5, 0.3, 0.1]
    g[0, 0] = [0.1, 0.3, 0.5]
    raw, _, _, _ = orc.error_maps(r, g)
    assert raw[0, 0] == pytest.approx(0.8 / 3, abs=1e-12)
    assert raw[0, 1] == 0.0
    r = np.zeros((1, 3, 3))
    for x in range(3):
        r[0, x] = 0.25 * (x + 1)
    _, nrm, mask, _ = orc.error_maps(r, np.zeros_like(r))
    np.testing.assert_allclose(nrm[0], [0, 0.5, 1])
    assert list(mask[0]) == [0, 0, 1]
    r = np.full((4, 4, 3), 0.3)
    _, nrm, mask, _ = orc.error_maps(r, np.zeros_like(r), 0.25)
    assert nrm.max() == 0 and mask.max() == 0
    rng = np.random.default_rng(62)
    r = rng.uniform(size=(16, 16, 3))
    g = rng.uniform(size=(16, 16, 3))
    raw, _, _, ph = orc.error_maps(r, g)
    assert ph == pytest.approx(0.8 * raw.mean() + 0.2 * (1 - orc.ssim(r, g, np.float64)), rel=1e-12)


# ---- scores / selection (tests/test_adc.cpp) ------------------------------------

def test_score_kats(orc):
    s_d, _, _ = orc.scores_from_counts([[3], [5]], [0.1, 0.1])
    assert s_d[0] == pytest.approx(4.0)
    _, raw, sp = orc.scores_from_counts([[4, 0]], [0.25])
    assert list(raw) == [1.0, 0.0] and list(sp) == [1.0, 0.0]
    _, _, sp = orc.scores_from_counts([[7, 7, 7]], [0.1])
    assert list(sp) == [0, 0, 0]


def _two_gaussian_scene():
    from oracle.oracle import n_components
    p = np.zeros((n_components(0), 2), np.float32)
    p[0] = [-0.3, 0.3]
    p[2] = [3, 3]
    p[3] = 1
    p[7:10] = math.log(0.08)
    p[10] = math.log(0.8 / 0.2)
    p[11:14, 0] = [1.2, 0.2, 0.2]
    p[11:14, 1] = [-0.8, 0.2, 0.2]
    return p


def test_select_densify_kats(orc):
    p = _two_gaussian_scene()
    p[7:10, 0] = math.log(0.001)
    t = orc.make_table(2, s_d=[3, 0], grad_norm_acc=[1, 0], views_seen=[1, 1])
    c, s = orc.select_densify(p, 0, t)
    assert c.sum() == 0
    t = orc.make_table(2, s_d=[100, 0], grad_norm_acc=[1e-6, 0], views_seen=[1, 1])
    c, s = orc.select_densify(p, 0, t)
    assert c.sum() == 0 and s.sum() == 0
    t = orc.make_table(2, s_d=[6, 0], grad_norm_acc=[4e-4, 0], views_seen=[1, 1])
    c, s = orc.select_densify(p, 0, t)
    assert list(c) == [1, 0] and s.sum() == 0
    p = _two_gaussian_scene()
    p[7:10, 0] = math.log(0.5)
    t = orc.make_table(2, s_d=[9, 9], abs_grad_acc=[2e-3, 0], views_seen=[1, 1])
    c, s = orc.select_densify(p, 0, t)
    assert list(s) == [1, 0] and c.sum() == 0


def test_select_prune_kats(orc):
    p = np.concatenate([_two_gaussian_scene(), _two_gaussian_scene()[:, :1]], 1)
    lg = lambda x: math.log(x / (1 - x))
    p[10] = [lg(0.05), lg(0.5), lg(0.5)]
    t = orc.make_table(3, s_p=[0.2, 0.95, 0.5])
    assert list(orc.select_prune(p, 0, t, 15000)) == [1, 1, 0]
    from oracle.oracle import n_components
    p = np.zeros((n_components(0), 6), np.float32)
    p[2] = 3
    p[3] = 1
    p[7:10] = math.log(0.05)
    p[10] = [lg(0.004)] * 4 + [lg(0.5)] * 2
    t = orc.make_table(6, s_p=[0.1, 0.2, 0.8, 0.9, 0.0, 0.0])
    assert list(np.nonzero(orc.select_prune(p, 0, t, 1000))[0]) == [2, 3]
    p = _two_gaussian_scene()
    p[10, 0] = lg(0.004)
    t = orc.make_table(2, s_p=[0, 0])
    assert list(orc.select_prune(p, 0, t, 1000, use_vcp=False)) == [1, 0]
    p = _two_gaussian_scene()
    p[7:10, 0] = math.log(0.5)
    t = orc.make_table(2, s_p=[1.0, 0.0])
    assert orc.select_prune(p, 0, t, 1000).sum() == 0
    assert list(orc.select_prune(p, 0, t, 4000)) == [1, 0]
    p = _two_gaussian_scene()
    p[10] = lg(0.01)
    t = orc.make_table(2, s_p=[0.4, 0.6])
    assert list(orc.select_prune(p, 0, t, 20000)) == [0, 1]


def test_expon_lr_endpoints(orc):
    assert orc.lib().or_expon_lr_f(1.6e-4, 1.6e-6, 0, 30000) == pytest.approx(1.6e-4, rel=1e-6)
    assert orc.lib().or_expon_lr_f(1.6e-4, 1.6e-6, 30000, 30000) == pytest.approx(1.6e-6, rel=1e-6)
    assert orc.lib().or_expon_lr_f(1.6e-4, 1.6e-6, 15000, 30000) == pytest.approx(math.sqrt(1.6e-4 * 1.6e-6),
                                                                                   rel=1e-6)


def test_schedule_30k(orc):
    """acceptance.cpp:400-438 / test_trainer.cpp:106-137: 30 densify events, late prunes."""
    c = orc.default_config()
    dens = [it for it in range(1, 30001) if orc.lib().or_densify_due(it, orc.C.byref(c))] if hasattr(orc, "C") else None
    import ctypes
    dens = [it for it in range(1, 30001) if orc.lib().or_densify_due(it, ctypes.byref(c))]
    prune = [it for it in range(15001, 30001) if orc.lib().or_prune_due(it, ctypes.byref(c))]
    assert len(dens) == 30
    assert prune == [18000, 21000, 24000, 27000, 30000]


def test_detmath_vs_std_exp_render_close(orc):
    """The deterministic exp/log substitution changes renders only at the ulp level."""
    rng = np.random.default_rng(7)
    pg = orc.random_projected(rng, 40, 64, 64, 0.9, dtype=np.float32)
    a = orc.render_pg(pg, 64, 64)
    orc.set_detmath(False)
    try:
        b = orc.render_pg(pg, 64, 64)
    finally:
        orc.set_detmath(True)
    assert np.abs(a.image - b.image).max() < 1e-4


def test_pge_visited_counter(orc):
    """The oracle's visited counter: every list entry up to and including the
    terminating one (raster.hpp:219-235); workers do not change it."""
    rng = np.random.default_rng(77)
    pg = orc.random_projected(rng, 40, 40, 24, 0.95, dtype=np.float32)
    r1 = orc.render_pg(pg, 40, 24, orc.binning(tile_size=8), workers=1)
    v1 = orc.last_pge_visited()
    r3 = orc.render_pg(pg, 40, 24, orc.binning(tile_size=8), workers=3)
    assert orc.last_pge_visited() == v1
    tiles_x = (40 + 7) // 8
    lo = hi = 0
    for y in range(24):
        for x in range(40):
            b, e = r1.ranges[(y // 8) * tiles_x + x // 8]
            hi += int(e - b)
            # unterminated pixels visit their whole list; terminated ones at
            # least every contributor
            lo += int(e - b) if r1.transmittance[y, x] >= 1e-4 else int(r1.contrib[y, x])
    assert lo <= v1 <= hi and v1 > int(r1.contrib.sum())
    assert np.array_equal(r1.image, r3.image)


def test_project_backward_fd(orc):
    """tests/test_camera.cpp:136-219: project_backward is the exact adjoint of
    project (mu2d, conic, colour, opacity) for every parameter, fp64, 1e-4."""
    from tests.util import random_scene
    rng = np.random.default_rng(136)
    for deg in (0, 1, 3):
        p = random_scene(rng, 3, deg).astype(np.float64)
        cam = orc.default_camera(64, 48)
        w_mu = rng.uniform(-1, 1, (3, 2))
        w_co = rng.uniform(-1, 1, (3, 4))
        w_co[:, 2] = w_co[:, 1]  # symmetric upstream (full-matrix convention)
        w_col = rng.uniform(-1, 1, (3, 3))
        w_op = rng.uniform(-1, 1, 3)

        def loss(q):
            pr = orc.project_scene(q, deg, cam, dtype=np.float64)
            assert pr.visible.all()
            return float((pr.mu2d * w_mu).sum() + (pr.conic * w_co).sum() + (pr.color * w_col).sum()
                         + (pr.opacity * w_op).sum())

        g = orc.project_backward(p, deg, cam, w_mu, w_co, w_col, w_op, dtype=np.float64)
        eps = 1e-6
        for c in range(p.shape[0]):
            for i in range(p.shape[1]):
                a, b = p.copy(), p.copy()
                a[c, i] += eps
                b[c, i] -= eps
                fd = (loss(a) - loss(b)) / (2 * eps)
                assert abs(fd - g[c, i]) <= 1e-4 * max(abs(fd), abs(g[c, i]), 1e-3), (deg, c, i, fd, g[c, i])
