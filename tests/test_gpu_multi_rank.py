"""The library's own multi-GPU exchange (csrc/comm.cu) executed
with two ranks: two processes share the one GPU of the test box and talk
through the host-callback communicator (sk_comm_create_host) over
torch.distributed/gloo — NCCL refuses two ranks on one device, and the code
path above the transport (sharded C1: reduce-scatter -> K10 on this rank's
slice -> in-place all-gather; C2 statistics; C3 all-gather of the score rows)
is the same for both backends.

Checked against single-process runs of the same library on the same inputs:
  * train steps: every rank ends with identical parameters and (gathered)
    Adam moments, equal to one process that sums the two views' gradients
    (K9 per view, host sum in rank order) before a replicated K10 — up to
    K8's atomic ordering; with the lazy SH-rest schedule the replicated C1
    (all-reduce of the n gradients) runs instead and must agree too;
  * a density event: the two ranks score K/2 views each, exchange rows
    (C3) and statistics (C2), and must select and compact exactly as one
    process scoring all K views with the summed statistics: identical
    flags, photometric values and compacted parameters, bit for bit.
"""
import json
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N, W, H, VIEWS, STEPS = 3000, 96, 80, 6, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    from oracle import oracle as orc
    from tests.util import ring_camera, synthetic_scene
    p = synthetic_scene(N, deg=3, seed=41)
    gt_p = synthetic_scene(N, deg=3, seed=42)
    cams = [ring_camera(orc, W, H, 0.3 + 1.05 * j) for j in range(VIEWS)]
    gts = [np.clip(np.rint(orc.render_scene(gt_p, 3, c).image * 255), 0, 255).astype(np.uint8) for c in cams]
    return p, cams, gts


def _config(lazy):
    import paper_2511_04283_b200 as sk
    cfg = sk.default_config()
    cfg.iterations = 30000
    cfg.densify_from = cfg.densify_until = 1 << 30
    cfg.seed = 17
    cfg.k = 4
    cfg.lazy_opt_enabled = int(lazy)
    return cfg


def _table_half(rng_seed, rank, n):
    """Rank r's share of one ScoreTable: the two shares sum (max) exactly to
    the full table (x * 0.5 is exact in binary floating point)."""
    rng = np.random.default_rng(rng_seed)
    vs = rng.integers(1, 11, n).astype(np.int32)
    g = rng.uniform(0, 6e-4, n).astype(np.float32) * vs
    a = rng.uniform(0, 6e-4, n).astype(np.float32) * vs
    g3 = rng.normal(0, 1e-4, (n, 3)).astype(np.float32)
    rad = rng.uniform(0, 30, n).astype(np.float32)
    full = dict(grad_norm_acc=g, abs_grad_acc=a, grad3d_acc=g3, views_seen=vs, max_radius2d=rad)
    if rank is None:
        return full
    half = np.float32(0.5)
    vs0 = vs // 2
    return dict(grad_norm_acc=g * half, abs_grad_acc=a * half, grad3d_acc=g3 * half,
                views_seen=vs0 if rank == 0 else vs - vs0,
                max_radius2d=rad if rank == 0 else rad * half)


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2511_04283_b200 as sk
    ctx = sk.Context(0)
    comm = sk.HostComm(ctx, dist, rank, world)
    p, cams, gts = _inputs()
    out = {}
    for lazy in (0, 1):
        data = sk.Dataset(ctx, cams, gts, list(range(VIEWS)), 2.64)
        scene = ctx.scene(p, 3)
        tr = sk.Trainer(ctx, scene, data, _config(lazy))
        tr.set_comm(comm)
        rows = tr.run(STEPS)
        m, v, t = scene.adam_state()
        np.savez(os.path.join(out_dir, f"train_l{lazy}_r{rank}.npz"), params=scene.download(), m=m, v=v,
                 t=np.array(t), views=np.array([r["view"] for r in rows]))
        tr.close()
        scene.close()
        data.close()
    # density event: C2 + C3 + identical selection / compaction
    data = sk.Dataset(ctx, cams, gts, list(range(VIEWS)), 2.64)
    scene = ctx.scene(p, 3, capacity=2 * N)
    tr = sk.Trainer(ctx, scene, data, _config(0), record_events=True)
    tr.set_comm(comm)
    scene.set_score_table(**_table_half(5, rank, N))
    tr.density_event(4000, True, True)
    ev = tr.events()[0]
    np.savez(os.path.join(out_dir, f"event_r{rank}.npz"), params=scene.download(), clone=ev["clone"],
             split=ev["split"], prune=ev["prune"], photometric=ev["photometric"], sampled=ev["sampled"])
    out["n_after"] = int(ev["n_after"])
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(out, f)
    comm.close()
    ctx.close()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def two_ranks(tmp_path_factory):
    import torch.multiprocessing as mp
    import paper_2511_04283_b200 as sk
    from oracle import oracle as orc
    sk.build()
    orc.build()
    d = tmp_path_factory.mktemp("ranks")
    mp.spawn(_worker, args=(2, _free_port(), str(d)), nprocs=2, join=True)
    return d


@pytest.mark.parametrize("lazy", [0, 1])
def test_two_rank_train_steps_match_single_process(two_ranks, lazy):
    import paper_2511_04283_b200 as sk
    r0 = np.load(two_ranks / f"train_l{lazy}_r0.npz")
    r1 = np.load(two_ranks / f"train_l{lazy}_r1.npz")
    # replicated state, bit for bit
    for f in ("params", "m", "v", "t"):
        assert np.array_equal(r0[f], r1[f]), f
    # the views: one shared Rng draw per rank per step, rank order
    from tests.util import rel_err_vec
    p, cams, gts = _inputs()
    cfg = _config(lazy)
    ctx = sk.Context(0)
    scene = ctx.scene(p, 3)
    lrs = sk.default_learning_rates()
    p0 = p.copy()
    for step in range(STEPS):
        g = None
        for views in (r0["views"], r1["views"]):
            ctx.preprocess(scene, cams[views[step]])
            ctx.build_tile_grid()
            ctx.blend_forward()
            ctx.training_loss(gts[views[step]], float(cfg.lambda_))
            ctx.blend_backward()
            gv = ctx.project_backward(scene, stats=False)
            g = gv if g is None else (g + gv).astype(np.float32)
        scene.set_grads(g)
        ext = np.float32(2.64)
        pos_lr = sk.expon_lr(np.float32(cfg.lr_position) * ext, np.float32(cfg.lr_position_final) * ext, step + 1,
                             cfg.iterations)
        ctx.adam_step(scene, lrs, position_lr=pos_lr)
    exp = scene.download()
    m, v, t = scene.adam_state()
    ctx.close()
    assert list(t) == list(r0["t"])
    d_got, d_exp = r0["params"] - p0, exp - p0
    bad = np.abs(d_got - d_exp) > 1e-3 * np.abs(d_exp).max(axis=1, keepdims=True) + 1e-12
    assert bad.mean() < 1e-3, bad.mean()
    assert rel_err_vec(r0["m"], m).max() < 1e-2
    assert r0["views"][0] != r1["views"][0] or r0["views"][1] != r1["views"][1]


def test_two_rank_density_event_matches_single_process(two_ranks):
    import paper_2511_04283_b200 as sk
    e0 = np.load(two_ranks / "event_r0.npz")
    e1 = np.load(two_ranks / "event_r1.npz")
    for f in ("params", "clone", "split", "prune", "photometric", "sampled"):
        assert np.array_equal(e0[f], e1[f]), f
    p, cams, gts = _inputs()
    ctx = sk.Context(0)
    data = sk.Dataset(ctx, cams, gts, list(range(VIEWS)), 2.64)
    scene = ctx.scene(p, 3, capacity=2 * N)
    tr = sk.Trainer(ctx, scene, data, _config(0), record_events=True)
    scene.set_score_table(**_table_half(5, None, N))
    tr.density_event(4000, True, True)
    ev = tr.events()[0]
    assert np.array_equal(ev["sampled"], e0["sampled"])
    assert np.array_equal(ev["photometric"], e0["photometric"])
    for f in ("clone", "split", "prune"):
        assert np.array_equal(ev[f], e0[f]), f
    assert ev["clone"].sum() + ev["split"].sum() > 0 and ev["prune"].sum() > 0
    assert np.array_equal(scene.download(), e0["params"])
    ctx.close()


@pytest.mark.slow
def test_bench_two_ranks_share_the_gpu(tmp_path):
    """bench.py under torchrun with two ranks on this one-GPU box: the
    multi-rank legs (training steps, end-to-end pipeline, density event) run
    over the host-callback communicator and rank 0 prints one JSON line that
    says it is a plumbing check (the driver's 2/4/8-GPU runs use NCCL)."""
    import subprocess
    import sys
    out = tmp_path / "bench.out"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--gaussians", "20000", "--width", "256", "--height", "192",
           "--views", "4", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, stdout=open(out, "w"), stderr=subprocess.PIPE, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in open(out).read().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert "plumbing check" in d["config"]["parallelism"]
    assert d["event"]["value"] > 0 and d["event"]["n_after_early"] > 0
