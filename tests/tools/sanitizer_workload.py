"""Workload run under compute-sanitizer by tests/test_gpu_sanitizer.py:
a 4K-Gaussian training step (K1-K10), one density event (K11-K15 with a
two-stream score pass), and a 200K-key depth sort whose onesweep passes span
dozens of tiles (decoupled look-back), and the float64 value path. No torch:
only the library's kernels. The training run is long enough for the step to
be captured into a CUDA graph and replayed.

  python tests/tools/sanitizer_workload.py [train|sort|fp64|all]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main(part):
    import paper_2511_04283_b200 as sk
    from tests.util import synthetic_scene
    import paper_2511_04283_b200.synthetic as syn
    ctx = sk.Context(0)
    if part in ("train", "all"):
        p = synthetic_scene(4000, deg=3, seed=3)
        cams = [syn.ring_camera(v, 8, 128, 96) for v in range(3)]
        gts = []
        for cam in cams:
            gts.append(syn.render_gt_u8(ctx, synthetic_scene(4000, deg=3, seed=4), 3, cam))
        cfg = sk.default_config()
        cfg.iterations = 30000
        cfg.densify_from = cfg.densify_until = 1 << 30
        scene = ctx.scene(p, 3)
        data = sk.Dataset(ctx, cams, gts, [0, 1, 2], 2.64)
        tr = sk.Trainer(ctx, scene, data, cfg)
        rows = tr.run(4)
        assert all(np.isfinite(r["loss"]) for r in rows)
        # the event: score pass over both streams, selection, compaction
        cfg.k = 3
        tr2 = sk.Trainer(ctx, scene, data, cfg)
        n = scene.size
        rng = np.random.default_rng(1)
        vs = rng.integers(1, 5, n).astype(np.int32)
        scene.set_score_table(grad_norm_acc=rng.uniform(0, 6e-4, n) * vs, abs_grad_acc=rng.uniform(0, 6e-4, n) * vs,
                              views_seen=vs, max_radius2d=rng.uniform(0, 30, n))
        tr2.density_event(4000, True, True)
        print("train+event ok", scene.size)
    if part in ("sort", "all"):
        n = 200_000
        p = synthetic_scene(n, deg=0, seed=5)
        cam = syn.ring_camera(0, 8, 256, 192)
        scene = ctx.scene(p, 0)
        ctx.preprocess(scene, cam)
        pairs = ctx.build_tile_grid()
        tl = ctx.tile_lists()
        assert tl.pairs == pairs
        print("sort ok", pairs)
    if part in ("fp64", "all"):
        p = synthetic_scene(500, deg=3, seed=6).astype(np.float64)
        cam = syn.ring_camera(0, 8, 96, 72)
        for mode in ("aabb", "compact"):
            _, vals = ctx.fp64_render_loss(p, 3, cam, np.full((72, 96, 3), 0.5), 0.2, sk.binning(mode))
            assert np.isfinite(vals[0])
        print("fp64 ok", vals)
    ctx.synchronize()
    ctx.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
