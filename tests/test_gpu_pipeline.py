"""The pipelined end-to-end entry point (sk_train_step_host_async): the same
training steps as the synchronous sk_train_step_host, with the GT uploads on a
copy stream and each step's loss delivered one call later."""
import os

import numpy as np
import pytest

from tests.util import ring_camera, synthetic_scene

pytestmark = pytest.mark.gpu


def test_async_host_steps_match_sync(orc):
    import torch

    import paper_2511_04283_b200 as sk
    sk.build()
    ctx = sk.Context(0)
    p = synthetic_scene(4000, deg=3, seed=21)
    cams = [ring_camera(orc, 128, 96, a) for a in (0.0, 0.9, 2.1)]
    gts = []
    for v, cam in enumerate(cams):
        r = orc.render_scene(synthetic_scene(4000, deg=3, seed=22), 3, cam)
        g = torch.empty(r.image.size, dtype=torch.uint8, pin_memory=True).numpy().reshape(r.image.shape)
        g[...] = np.clip(np.rint(r.image * 255), 0, 255).astype(np.uint8)
        gts.append(g)
    cfg = sk.default_config()
    cfg.densify_from = cfg.densify_until = 1 << 30
    a = ctx.scene(p, 3)
    b = ctx.scene(p, 3)
    sync_rows = [sk.train_step_host(ctx, a, cams[k % 3], gts[k % 3], cfg, 3.0, k + 1) for k in range(9)]
    pipe = sk.HostStepPipeline(ctx)
    for k in range(9):
        pipe.step(b, cams[k % 3], gts[k % 3], cfg, 3.0, k + 1)
    rows = pipe.flush()
    graph_steps = sk.C.c_int64()
    ctx.check(ctx._lib.sk_ctx_graph_steps(ctx.h, sk.C.byref(graph_steps)))
    if os.environ.get("SK_STEP_GRAPH", "1") != "0":
        assert graph_steps.value >= 6  # steady-state steps ran as the captured graph
    assert [r["iteration"] for r in rows] == list(range(1, 10))
    for s, r in zip(sync_rows, rows):
        assert r["tile_pairs"] == s["tile_pairs"]
        assert r["loss"] == pytest.approx(s["loss"], rel=1e-4)
    np.testing.assert_allclose(b.download(), a.download(), rtol=1e-4, atol=1e-5)
    # a synchronous step after async ones completes the pending step first
    pipe.step(b, cams[0], gts[0], cfg, 3.0, 10)
    sk.train_step_host(ctx, b, cams[1], gts[1], cfg, 3.0, 11)
    assert pipe.flush()[0]["iteration"] == 10
    ctx.close()


def test_pair_buffer_overflow_replays_the_step(orc, monkeypatch):
    """Training steps keep the pair count on the device: the scatter fills the
    frame's existing pair buffer and a step whose P outgrew it is skipped on
    the device (kErrPairOverflow) and replayed once the host reads P with the
    loss. A frame whose first pair buffer holds 300 pairs must give the same
    rows and parameters as one sized normally — through the pipelined host
    step, the synchronous one and Trainer::run."""
    import torch

    import paper_2511_04283_b200 as sk
    sk.build()
    p = synthetic_scene(4000, deg=3, seed=41)
    cams = [ring_camera(orc, 128, 96, a) for a in (0.3, 1.4, 2.8)]
    gts = []
    for cam in cams:
        r = orc.render_scene(synthetic_scene(4000, deg=3, seed=42), 3, cam)
        g = torch.empty(r.image.size, dtype=torch.uint8, pin_memory=True).numpy().reshape(r.image.shape)
        g[...] = np.clip(np.rint(r.image * 255), 0, 255).astype(np.uint8)
        gts.append(g)
    cfg = sk.default_config()
    cfg.densify_from = cfg.densify_until = 1 << 30

    def run(ctx):
        a, b, c = ctx.scene(p, 3), ctx.scene(p, 3), ctx.scene(p, 3)
        pipe = sk.HostStepPipeline(ctx)
        for k in range(6):
            pipe.step(a, cams[k % 3], gts[k % 3], cfg, 3.0, k + 1)
        rows = pipe.flush()
        frame = ctx._new_frame()
        sync = [sk.train_step_host(ctx, b, cams[k % 3], gts[k % 3], cfg, 3.0, k + 1, frame=frame) for k in range(3)]
        data = sk.Dataset(ctx, cams, [np.ascontiguousarray(g) for g in gts], [0, 1, 2], 3.0)
        tr = sk.Trainer(ctx, c, data, cfg)
        trows = tr.run(4)
        return rows, sync, trows, a.download(), b.download(), c.download()

    ref = run(sk.Context(0))
    monkeypatch.setenv("SK_INITIAL_PAIR_CAP", "300")
    got = run(sk.Context(0))
    assert ref[0][0]["tile_pairs"] > 300  # every frame's first step overflowed and was replayed
    for r, g in zip(ref[0] + ref[1] + ref[2], got[0] + got[1] + got[2]):
        assert g["tile_pairs"] == r["tile_pairs"]
        assert g["loss"] == pytest.approx(r["loss"], rel=1e-4)
    for r, g in zip(ref[3:], got[3:]):
        np.testing.assert_allclose(g, r, rtol=1e-4, atol=1e-5)


def test_nccl_single_rank_communicator(orc):
    """The NCCL plumbing on one GPU: the library resolves NCCL, a one-rank
    communicator is created from a unique id, and a view-parallel Trainer
    and the pipelined host step run with it (all collectives degenerate to
    no-ops at world size 1, so results equal the communicator-free run)."""
    import paper_2511_04283_b200 as sk
    sk.build()
    ctx = sk.Context(0)
    uid = sk.comm_unique_id()
    assert len(uid) == sk.COMM_ID_BYTES and any(uid)
    comm = sk.Comm(ctx, uid, 1, 0)
    p = synthetic_scene(3000, deg=3, seed=31)
    cam = ring_camera(orc, 96, 64, 0.4)
    gt = np.clip(orc.render_scene(synthetic_scene(3000, deg=3, seed=32), 3, cam).image * 255 + 0.5, 0, 255)
    gt = gt.astype(np.uint8)
    cfg = sk.default_config()
    cfg.densify_from = cfg.densify_until = 1 << 30
    a = ctx.scene(p, 3)
    data = sk.Dataset(ctx, [cam], [gt], [0], 3.0)
    tr = sk.Trainer(ctx, a, data, cfg)
    tr.set_comm(comm)
    rows = tr.run(3)
    assert all(np.isfinite(r["loss"]) for r in rows)
    pipe = sk.HostStepPipeline(ctx, comm=comm)
    pipe.step(a, cam, gt, cfg, 3.0, 4)
    assert np.isfinite(pipe.flush()[0]["loss"])
    comm.close()
    ctx.close()


def _poke_device_param(ctx, scene, comp, index, value):
    """Writes one parameter straight into the device scene (no upload, so
    the Adam state is kept) through __cuda_array_interface__."""
    import torch

    import paper_2511_04283_b200 as sk
    ptr = sk.C.POINTER(sk.C.c_float)()
    stride = sk.C.c_int64()
    ctx.check(ctx._lib.sk_scene_device_params(scene.h, sk.C.byref(ptr), sk.C.byref(stride)))
    addr = sk.C.cast(ptr, sk.C.c_void_p).value + 4 * (comp * stride.value + index)

    class One:
        __cuda_array_interface__ = {"shape": (1,), "typestr": "<f4", "data": (addr, False), "version": 3}
    ctx.synchronize()
    torch.as_tensor(One(), device="cuda").fill_(value)
    torch.cuda.synchronize()


def test_device_error_leaves_scene_untouched(orc):
    """covariance_3d throws before any state changes (scene.hpp:89-92): a train
    step whose K1 raises leaves parameters, Adam moments and step counters and
    the score table as they were — on the synchronous path and on the
    pipelined path (which reports the error one call late)."""
    import paper_2511_04283_b200 as sk
    from tests.util import random_scene
    sk.build()
    ctx = sk.Context(0)
    rng = np.random.default_rng(31)
    p = random_scene(rng, 300, 3)
    cam = orc.default_camera(64, 48)
    gt8 = rng.integers(0, 256, (48, 64, 3), dtype=np.uint8)
    cfg = sk.default_config()
    scene = ctx.scene(p, 3)
    sk.train_step_host(ctx, scene, cam, gt8, cfg, 2.64, 1)  # one good step: non-zero moments and stats
    _poke_device_param(ctx, scene, 7, 5, float("nan"))
    before = scene.download()
    assert np.isnan(before[7, 5])
    m0, v0, t0 = scene.adam_state()
    assert np.abs(m0).max() > 0 and list(t0) == [1] * 6
    tab0 = scene.score_table()
    with pytest.raises(ValueError, match="covariance_3d"):
        sk.train_step_host(ctx, scene, cam, gt8, cfg, 2.64, 2)
    assert np.array_equal(scene.download(), before, equal_nan=True)
    m1, v1, t1 = scene.adam_state()
    assert np.array_equal(m1, m0) and np.array_equal(v1, v0) and list(t1) == list(t0)
    tab1 = scene.score_table()
    assert np.array_equal(tab1.views_seen, tab0.views_seen)
    assert np.array_equal(tab1.grad_norm_acc, tab0.grad_norm_acc)
    # pipelined: the error surfaces at the next call (or flush), state untouched
    import torch
    pinned = torch.empty(gt8.size, dtype=torch.uint8, pin_memory=True).numpy().reshape(gt8.shape)
    pinned[...] = gt8
    pipe = sk.HostStepPipeline(ctx)
    with pytest.raises(ValueError, match="covariance_3d"):
        pipe.step(scene, cam, pinned, cfg, 2.64, 3)
        pipe.step(scene, cam, pinned, cfg, 2.64, 4)
        pipe.flush()
    assert np.array_equal(scene.download(), before, equal_nan=True)
    m2, v2, t2 = scene.adam_state()
    assert np.array_equal(m2, m0) and np.array_equal(v2, v0) and list(t2) == list(t0)
    ctx.close()
