"""World-size-2 CPU tests (gloo) of the view-sharded multi-GPU algorithm
(SURVEY §8e). The GPU collectives are NCCL calls inside the library; here the
same exchange pattern runs over gloo on the restated reference so that the
semantics are checked on every CPU run:
  - the NCCL communicator id reaches every rank intact (torch.distributed);
  - C3: scoring a round-robin shard of the K views per rank and summing the
    zero-padded count rows / photometric scalars reproduces the single-process
    accumulate_scores exactly (s_d bit-exact);
  - C1: summing per-rank view gradients gives the identical gradient on every
    rank (replicated Adam stays in lock step);
  - C2: sum / max reductions of the ScoreTable statistics.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2511_04283_b200 as sk
    from oracle import oracle as orc
    from tests.util import ring_camera, synthetic_scene

    res = {}
    # NCCL id broadcast
    uid = sk.share_comm_id(dist, rank)
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    res["id_ok"] = len(uid) == sk.COMM_ID_BYTES and all(i == ids[0] for i in ids)

    deg = 3
    p = synthetic_scene(1500, deg=deg, seed=21)
    gt_p = synthetic_scene(1500, deg=deg, seed=22)
    K = 5
    cams = [ring_camera(orc, 64, 48, 0.4 + 1.1 * j) for j in range(K)]
    gts = [orc.render_scene(gt_p, deg, c).image for c in cams]

    # C3: sharded score pass
    mine = sk.shard_assign(K, world, rank)
    counts_r, photo_r, _, _, _ = orc.accumulate_scores(p, deg, [cams[j] for j in mine], [gts[j] for j in mine])
    rows = np.zeros((K, p.shape[1]), np.int32)
    photo = np.zeros(K, np.float32)
    rows[mine] = counts_r
    photo[mine] = photo_r
    tr = torch.from_numpy(rows)
    tp = torch.from_numpy(photo)
    dist.all_reduce(tr)
    dist.all_reduce(tp)
    s_d, s_p_raw, s_p = orc.scores_from_counts(tr.numpy(), tp.numpy())
    _, _, ref_sd, ref_spr, ref_sp = orc.accumulate_scores(p, deg, cams, gts)
    res["c3_sd_exact"] = bool(np.array_equal(s_d, ref_sd))
    res["c3_sp_raw_exact"] = bool(np.array_equal(s_p_raw, ref_spr))
    res["c3_sp_exact"] = bool(np.array_equal(s_p, ref_sp))

    # C1: per-rank view gradient, summed
    g_mine, _ = orc.view_grads(p, deg, cams[rank], gts[rank])
    tg = torch.from_numpy(g_mine.copy())
    dist.all_reduce(tg)
    g0, _ = orc.view_grads(p, deg, cams[0], gts[0])
    g1, _ = orc.view_grads(p, deg, cams[1], gts[1])
    res["c1_sum_ok"] = bool(np.array_equal(tg.numpy(), g0 + g1))
    allg = [None] * world
    dist.all_gather_object(allg, tg.numpy().tobytes())
    res["c1_replicated"] = all(a == allg[0] for a in allg)

    # C2: statistics sum / max
    rng = np.random.default_rng(100 + rank)
    gn = rng.uniform(0, 1, 64).astype(np.float32)
    vs = rng.integers(0, 5, 64).astype(np.int32)
    mr = rng.uniform(0, 30, 64).astype(np.float32)
    tg2, tv, tm = torch.from_numpy(gn.copy()), torch.from_numpy(vs.copy()), torch.from_numpy(mr.copy())
    dist.all_reduce(tg2)
    dist.all_reduce(tv)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    others = [np.random.default_rng(100 + r) for r in range(world)]
    exp_gn = np.zeros(64, np.float32)
    exp_vs = np.zeros(64, np.int32)
    exp_mr = np.zeros(64, np.float32)
    for o in others:
        a = o.uniform(0, 1, 64).astype(np.float32)
        b = o.integers(0, 5, 64).astype(np.int32)
        c = o.uniform(0, 30, 64).astype(np.float32)
        exp_gn = exp_gn + a
        exp_vs = exp_vs + b
        exp_mr = np.maximum(exp_mr, c)
    res["c2_ok"] = bool(np.allclose(tg2.numpy(), exp_gn, rtol=1e-6) and np.array_equal(tv.numpy(), exp_vs)
                        and np.array_equal(tm.numpy(), exp_mr))
    import json
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)
    dist.destroy_process_group()


def test_view_sharded_collectives_gloo(tmp_path):
    import torch.multiprocessing as mp
    from oracle import oracle as orc
    orc.build()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    import json
    for r in range(2):
        res = json.load(open(tmp_path / f"rank{r}.json"))
        for k, v in res.items():
            assert v, (r, k)


def test_shard_assign_partitions():
    import paper_2511_04283_b200 as sk
    for k in range(0, 12):
        for world in (1, 2, 3, 8):
            parts = [sk.shard_assign(k, world, r) for r in range(world)]
            flat = sorted(x for p in parts for x in p)
            assert flat == list(range(k))
