"""Diagnostic: GPU trainer vs CPU oracle on config 1, iteration by iteration."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_04283_b200 as sk  # noqa: E402
from oracle import oracle as orc  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 500
ds = orc.Dataset(10000, 8, 256, seed=1)
xyz, rgb = ds.points()
p0 = orc.init_from_points(xyz, rgb, 3)
cfg = orc.default_config()
cfg.iterations = 500
cfg.densify_from = 100
cfg.densify_until = 400
cfg.densify_every = 100
cfg.prune_every_early = 100
cfg.prune_every_late = 100
cfg.size_prune_from = 200
cfg.seed = 17
cfg.workers = os.cpu_count()
ctx = sk.Context(0)
cams = [ds.camera(v) for v in range(ds.num_views)]
imgs = [ds.image_u8(v) for v in range(ds.num_views)]
data = sk.Dataset(ctx, cams, imgs, ds.train_indices(), ds.extent)
scene = ctx.scene(p0, 3)
tr = sk.Trainer(ctx, scene, data, cfg, record_events=True)
otr = orc.Trainer(p0, 3, ds, cfg)
chunk = 50
test_gt = imgs[0].astype(np.float32) / np.float32(255)
for start in range(0, iters, chunk):
    g = tr.run(chunk)
    o, secs = otr.run(chunk)
    pg, po = scene.download(), otr.scene()
    ps_g = orc.psnr(orc.render_scene(pg, 3, cams[0]).image, test_gt)
    ps_o = orc.psnr(orc.render_scene(po, 3, cams[0]).image, test_gt)
    same = pg.shape == po.shape
    dmax = float(np.abs(pg - po).max()) if same else float("nan")
    views_g = [r["view"] for r in g]
    print(f"it {start + chunk}: loss gpu {g[-1]['loss']:.5f} cpu {o[-1, 0]:.5f} | N {pg.shape[1]} {po.shape[1]} | "
          f"pairs {g[-1]['tile_pairs']} {int(o[-1, 3])} | test psnr {ps_g:.3f} {ps_o:.3f} | max|dp| {dmax:.3g} "
          f"| cpu {secs:.1f}s", flush=True)
ge, ce = tr.events(), otr.events()
for a, b in zip(ge, ce):
    n = a["n_before"]
    def flags(e, key, n):
        f = np.zeros(n, np.uint8)
        f[e[key]] = 1
        return f
    line = f"event {a['iteration']}: N {a['n_before']}->{a['n_after']} cpu {b['n_before']}->{b['n_after']} " \
           f"views {list(a['sampled'])} {list(b['sampled'])} photo {np.round(a['photometric'], 5)} " \
           f"{np.round(b['photometric'], 5)}"
    if a["n_before"] == b["n_before"]:
        for key in ("clone", "split", "prune"):
            cf = flags(b, key, n)
            line += f" | {key} gpu {int(a[key].sum())} cpu {int(cf.sum())} flips {int((a[key] != cf).sum())}"
    print(line, flush=True)
