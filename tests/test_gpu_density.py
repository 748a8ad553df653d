"""GPU parity of the multi-view density control (K11-K15) and of the full
training loop (config 1) against the CPU oracle.

Footprint counts, s_d and all selection flags are exact integers / bit-exact
given identical inputs; s_p carries the photometric tolerance; compaction is
bit-exact. The 500-iteration config-1 run compares final PSNR (<= 0.05 dB)
and reports per-event mask agreement.
"""
import math
import os

import numpy as np
import pytest

from tests.util import random_scene, rel_err_vec, ring_camera, synthetic_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2511_04283_b200 as sk
    sk.build()
    c = sk.Context(0)
    yield c
    c.close()


def test_accumulate_scores_matches_oracle(ctx, orc):
    p = synthetic_scene(3000, deg=3, seed=11)
    gt_p = synthetic_scene(3000, deg=3, seed=12)
    cams = [ring_camera(orc, 96, 80, a) for a in (0.0, 1.3, 2.9)]
    gts = [orc.render_scene(gt_p, 3, c).image for c in cams]
    counts_ref, photo_ref, s_d_ref, s_p_raw_ref, s_p_ref = orc.accumulate_scores(p, 3, cams, gts, 0.5, 0.2)
    scene = ctx.scene(p, 3)
    counts, photo = ctx.accumulate_scores(scene, cams, gts, 0.5, 0.2)
    assert np.array_equal(counts, counts_ref)
    np.testing.assert_allclose(photo, photo_ref, rtol=1e-5)
    t = scene.score_table()
    assert np.array_equal(t.s_d, s_d_ref)  # exact: integer counts, same fp32 order
    assert rel_err_vec(t.s_p_raw, s_p_raw_ref).max() < 1e-3
    assert np.abs(t.s_p - s_p_ref).max() < 1e-3


def test_accumulate_scores_culled_gaussian_scores_zero(ctx, orc):
    """tests/test_adc.cpp:112-131."""
    p = random_scene(np.random.default_rng(2), 2, 0)
    p[0:3, 0] = [-0.3, 0, 3]
    p[0:3, 1] = [0, 0, -5]
    cam = orc.default_camera(24, 24)
    scene = ctx.scene(p, 0)
    ctx.accumulate_scores(scene, [cam], [np.zeros((24, 24, 3), np.float32)])
    t = scene.score_table()
    assert t.s_d[1] == 0 and t.s_p_raw[1] == 0
    scene.set_score_table(grad_norm_acc=[0, 100.0], abs_grad_acc=[0, 100.0], views_seen=[0, 0])
    clone, split = ctx.select_densify(scene)
    assert clone[1] == 0 and split[1] == 0


def _random_table(rng, n):
    return dict(s_d=rng.uniform(0, 12, n), s_p=rng.uniform(0, 1, n), grad_norm_acc=rng.uniform(0, 6e-4, n),
                abs_grad_acc=rng.uniform(0, 6e-4, n), views_seen=rng.integers(0, 10, n),
                max_radius2d=rng.uniform(0, 40, n), grad3d_acc=rng.normal(size=(n, 3)))


@pytest.mark.parametrize("use_vcd", [True, False])
def test_select_densify_bit_exact(ctx, orc, use_vcd):
    rng = np.random.default_rng(72)
    n = 5000
    p = random_scene(rng, n, 2)
    p[7:10] = np.log(rng.uniform(0.001, 0.05, (3, n)))
    tb = _random_table(rng, n)
    scene = ctx.scene(p, 2)
    scene.set_score_table(**tb)
    clone, split = ctx.select_densify(scene, use_vcd=use_vcd, extent=1.0)
    rc, rs = orc.select_densify(p, 2, orc.make_table(n, **tb), use_vcd=use_vcd, extent=1.0)
    assert np.array_equal(clone, rc) and np.array_equal(split, rs)
    assert clone.sum() > 0 and split.sum() > 0


@pytest.mark.parametrize("iteration,use_vcp", [(1000, True), (4000, True), (1000, False), (20000, True),
                                               (20000, False)])
def test_select_prune_bit_exact(ctx, orc, iteration, use_vcp):
    rng = np.random.default_rng(73 + iteration)
    n = 6000
    p = random_scene(rng, n, 1)
    op = rng.uniform(0.001, 0.3, n)
    p[10] = np.log(op / (1 - op))
    p[7:10] = np.log(rng.uniform(0.01, 0.2, (3, n)))
    tb = _random_table(rng, n)
    tb["s_p"][::7] = 0.5  # ties: broken by index
    scene = ctx.scene(p, 1)
    scene.set_score_table(**tb)
    got = ctx.select_prune(scene, iteration, use_vcp=int(use_vcp), extent=1.0)
    ref = orc.select_prune(p, 1, orc.make_table(n, **tb), iteration, use_vcp=use_vcp, extent=1.0)
    assert np.array_equal(got, ref)
    assert 0 < got.sum() < n


def test_select_prune_never_empties(ctx, orc):
    p = random_scene(np.random.default_rng(3), 2, 0)
    p[10] = math.log(0.01 / 0.99)
    scene = ctx.scene(p, 0)
    scene.set_score_table(s_p=[0.4, 0.6])
    assert list(ctx.select_prune(scene, 20000)) == [0, 1]


def test_compaction_bit_exact(ctx, orc):
    rng = np.random.default_rng(74)
    n = 4000
    deg = 2
    p = random_scene(rng, n, deg)
    prune = (rng.uniform(size=n) < 0.1).astype(np.uint8)
    kind = rng.uniform(size=n)
    clone = (kind < 0.1).astype(np.uint8)
    split = ((kind >= 0.1) & (kind < 0.2)).astype(np.uint8)
    tb = _random_table(rng, n)
    n_split = int(((split == 1) & (prune == 0)).sum())
    eps = rng.normal(size=6 * n_split).astype(np.float32)
    scene = ctx.scene(p, deg)
    # give the optimizer non-zero moments first
    scene.set_grads(rng.normal(size=p.shape).astype(np.float32))
    ctx.adam_step(scene)
    p0 = scene.download()
    m0, v0, _ = scene.adam_state()
    scene.set_score_table(**tb)
    o2n, new_n = ctx.apply_prune_densify(scene, prune, clone, split, np.float32(0.01), eps)
    ref_p, ref_m, ref_v, ref_o2n = orc.apply_prune_densify(p0, deg, prune, clone, split, tb["grad3d_acc"],
                                                           tb["views_seen"], np.float32(0.01), eps, m0, v0)
    assert new_n == ref_p.shape[1]
    assert np.array_equal(o2n, ref_o2n)
    assert np.array_equal(scene.download(), ref_p)
    m1, v1, _ = scene.adam_state()
    assert np.array_equal(m1, ref_m) and np.array_equal(v1, ref_v)
    t = scene.score_table()
    assert t.views_seen.sum() == 0 and np.abs(t.grad_norm_acc).sum() == 0


def test_densify_kats_gpu(ctx, orc):
    """tests/test_adc.cpp:209-260: cardinality, child scale / 1.6, clone offset."""
    p = random_scene(np.random.default_rng(73), 5, 2)
    scene = ctx.scene(p, 2)
    split = np.zeros(5, np.uint8)
    split[2] = 1
    eps = np.random.default_rng(1).normal(size=6).astype(np.float32)
    o2n, new_n = ctx.apply_prune_densify(scene, split=split, eps=eps)
    assert new_n == 6 and o2n[2] == -1
    q = scene.download()
    for c in (4, 5):
        np.testing.assert_allclose(q[7:10, c], p[7:10, 2] - np.float32(math.log(1.6)), rtol=1e-6)
        assert np.array_equal(q[3:7, c], p[3:7, 2]) and q[10, c] == p[10, 2]
    scene = ctx.scene(p, 2)
    scene.set_score_table(grad3d_acc=np.array([[0, 0, 0], [1.0, -2.0, 0.5], [0, 0, 0], [0, 0, 0], [0, 0, 0]]),
                          views_seen=[0, 2, 0, 0, 0])
    clone = np.zeros(5, np.uint8)
    clone[1] = 1
    o2n, new_n = ctx.apply_prune_densify(scene, clone=clone, clone_step_lr=np.float32(0.01))
    q = scene.download()
    assert new_n == 6 and o2n[1] == 1
    np.testing.assert_allclose(q[0:3, 5], p[0:3, 1] - 0.01 * np.array([0.5, -1.0, 0.25]), atol=1e-6)


def _config1(orc):
    cfg = orc.default_config()
    cfg.iterations = 500
    cfg.densify_from = 100
    cfg.densify_until = 400
    cfg.densify_every = 100
    cfg.prune_every_early = 100
    cfg.prune_every_late = 100
    cfg.size_prune_from = 200
    cfg.k = 10
    cfg.seed = 17
    cfg.workers = os.cpu_count() or 1
    return cfg


@pytest.mark.slow
def test_config1_training_parity(ctx, orc):
    """BASELINE config 1: 10K Gaussians, 8 views 256x256, 500 iterations with
    multi-view densify/prune; CPU oracle vs GPU trainer on the same seeds."""
    import paper_2511_04283_b200 as sk
    ds = orc.Dataset(10000, 8, 256, seed=1)
    xyz, rgb = ds.points()
    p0 = orc.init_from_points(xyz, rgb, 3)
    cfg = _config1(orc)
    cams = [ds.camera(v) for v in range(ds.num_views)]
    imgs = [ds.image_u8(v) for v in range(ds.num_views)]
    data = sk.Dataset(ctx, cams, imgs, ds.train_indices(), ds.extent)
    scene = ctx.scene(p0, 3)
    tr = sk.Trainer(ctx, scene, data, cfg, record_events=True)
    rows = tr.run(500)
    gpu_events = tr.events()
    final_gpu = scene.download()

    # The oracle replays the GPU's decisions ("follow" mode) so that a single
    # near-threshold flip does not desynchronise the shared Rng (the split
    # noise count depends on the split set); its own selection is kept in its
    # event records and every disagreement is reported as a flip.
    otr = orc.Trainer(p0, 3, ds, cfg)
    orc.trainer_force_events(otr, gpu_events)
    orows, secs = otr.run(500)
    final_cpu = otr.scene()
    cpu_events = otr.events()

    test_gt = imgs[0].astype(np.float32) / np.float32(255)
    ps_gpu = orc.psnr(orc.render_scene(final_gpu, 3, cams[0]).image, test_gt)
    ps_cpu = orc.psnr(orc.render_scene(final_cpu, 3, cams[0]).image, test_gt)
    print(f"config1: test-view PSNR gpu {ps_gpu:.3f} dB cpu {ps_cpu:.3f} dB; N gpu {final_gpu.shape[1]} "
          f"cpu {final_cpu.shape[1]}; oracle {secs:.1f} s")
    assert len(gpu_events) == len(cpu_events)
    total_flips = 0
    for ge, ce in zip(gpu_events, cpu_events):
        assert ge["iteration"] == ce["iteration"]
        assert list(ge["sampled"]) == list(ce["sampled"])
        n = ge["n_before"]
        assert ce["n_before"] == n and ce["n_after"] == ge["n_after"]
        flips = {}
        for key in ("clone", "split", "prune"):
            own = np.zeros(n, np.uint8)
            own[ce[key]] = 1
            flips[key] = int((own != ge[key]).sum())
            # direction: selected by the GPU only / by the oracle only
            flips[key + "_dir"] = (int(((ge[key] != 0) & (own == 0)).sum()), int(((ge[key] == 0) & (own != 0)).sum()))
        total_flips += sum(flips[k] for k in ("clone", "split", "prune"))
        print(f"  event {ge['iteration']}: N {n}->{ge['n_after']} clone {ge['n_clone']} split {ge['n_split']} "
              f"prune {ge['n_prune']} | near-threshold flips {flips}")
        # flips come from near-threshold statistics (atomic summation order,
        # Adam sign flips on near-zero gradients); they stay a small fraction
        assert sum(flips[k] for k in ("clone", "split", "prune")) <= max(3, n // 100)
    assert abs(ps_gpu - ps_cpu) <= 0.05
    assert abs(rows[-1]["loss"] - orows[-1, 0]) < 0.05 * abs(orows[-1, 0]) + 1e-3

    # Independent runs: the oracle on its own decisions (its Rng then draws
    # the split noise for its own split sets). The trajectories separate at
    # the first near-threshold flip and the densify/prune dynamics amplify it
    # (GPU runs of one seed differ by 2x in event-300 split counts), so the
    # bar is a sanity bound on a chaotic outcome, not a parity gate (that is
    # the follow-mode 0.05 dB above). Measured on B200: the oracle over seeds
    # 17-20 ends at 24.82-24.91 dB, N 4923 at seed 17; six GPU runs of seed
    # 17 (atomic summation order varies run to run) at 23.99-24.96 dB, N
    # 4698-5006.
    itr = orc.Trainer(p0, 3, ds, cfg)
    irows, isecs = itr.run(500)
    final_ind = itr.scene()
    ps_ind = orc.psnr(orc.render_scene(final_ind, 3, cams[0]).image, test_gt)
    print(f"config1 independent: test-view PSNR gpu {ps_gpu:.3f} dB oracle {ps_ind:.3f} dB "
          f"(delta {ps_gpu - ps_ind:+.3f}); N gpu {final_gpu.shape[1]} oracle {final_ind.shape[1]}; "
          f"final loss gpu {rows[-1]['loss']:.5f} oracle {irows[-1, 0]:.5f}")
    assert abs(ps_gpu - ps_ind) <= 1.25
    assert abs(final_gpu.shape[1] - final_ind.shape[1]) <= 0.1 * final_ind.shape[1]


def test_two_stream_score_pass_identical(ctx, orc):
    """The density event's two-stream score pass (views split over two host
    threads / streams) gives exactly the single-stream result: same sampled
    views, photometric scores, selections and compacted scene. No training
    beforehand (its atomic gradient sums are not bit-reproducible); the
    gradient statistics are a seeded table instead."""
    import os

    import paper_2511_04283_b200 as sk
    ds, gt, xyz, rgb = sk.Dataset.synthetic(ctx, n_gaussians=4000, n_views=12, width=96, seed=7)
    p0 = orc.init_from_points(xyz, rgb, 3)
    cfg = sk.default_config()
    cfg.k = 9
    cfg.tau_d = 0.5
    cfg.size_prune_from = 0
    out = []
    for one in ("1", "0"):
        os.environ["SK_SCORE_ONE_STREAM"] = one
        try:
            scene = ctx.scene(p0, 3)
            tr = sk.Trainer(ctx, scene, ds, cfg, record_events=True)
            scene.set_score_table(**_random_table(np.random.default_rng(3), scene.size))
            tr.density_event(600, True, True)
            out.append((scene.download(), tr.events()[-1]))
            tr.close()
        finally:
            os.environ.pop("SK_SCORE_ONE_STREAM", None)
    (p1, e1), (p2, e2) = out
    assert e1["n_after"] == e2["n_after"] and list(e1["sampled"]) == list(e2["sampled"])
    assert len(e1["sampled"]) == 9
    assert e1["n_clone"] + e1["n_split"] + e1["n_prune"] > 0
    for key in ("clone", "split", "prune", "photometric"):
        assert np.array_equal(np.asarray(e1[key]), np.asarray(e2[key])), key
    assert np.array_equal(p1, p2)
