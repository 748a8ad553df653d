"""Diagnostic: where the end-to-end step loses time against the device-resident
step (config 2). Times trainer.run(1), the pipelined host-input step, the
synchronous host-input step and a bare 6.2 MB pinned H2D copy."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_04283_b200 as sk  # noqa: E402
import paper_2511_04283_b200.synthetic as syn  # noqa: E402
from bench import train_config  # noqa: E402

n, W, H = 1_000_000, 1920, 1080
ctx = sk.Context(0)
stream = torch.cuda.current_stream()
ctx.check(ctx._lib.sk_ctx_set_stream(ctx.h, sk.C.c_void_p(stream.cuda_stream)))
extent = syn.ring_extent()
gt_params = syn.gaussians(n, 1, 3)
cam = syn.ring_camera(0, 64, W, H)
gt8 = syn.render_gt_u8(ctx, gt_params, 3, cam)
params = syn.perturb_positions(gt_params, 0.02 * extent, 2)
cfg = train_config(sk)
scene = ctx.scene(params, 3)
data = sk.Dataset(ctx, [cam], [gt8], [0], extent)
tr = sk.Trainer(ctx, scene, data, cfg)
tr.run(20)
pinned = torch.empty(gt8.size, dtype=torch.uint8, pin_memory=True)
gt_host = pinned.numpy().reshape(gt8.shape)
gt_host[...] = gt8
K = 100


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K, 1000 * (time.perf_counter() - t0) / K


print("trainer.run(1)      dev %.3f ms  wall %.3f ms" % timed(lambda: [tr.run(1) for _ in range(K)]))
it = [1000]
pipe = sk.HostStepPipeline(ctx)


def piped():
    for _ in range(K):
        it[0] += 1
        pipe.step(scene, cam, gt_host, cfg, extent, it[0])
    pipe.flush()


print("pipelined host step dev %.3f ms  wall %.3f ms" % timed(piped))


def sync_steps():
    for _ in range(K):
        it[0] += 1
        sk.train_step_host(ctx, scene, cam, gt_host, cfg, extent, it[0])


print("sync host step      dev %.3f ms  wall %.3f ms" % timed(sync_steps))
dev = torch.empty(gt8.size, dtype=torch.uint8, device="cuda")
side = torch.cuda.Stream()


def copies():
    with torch.cuda.stream(side):
        for _ in range(K):
            dev.copy_(pinned, non_blocking=True)
    side.synchronize()


t0 = time.perf_counter()
copies()
print("bare 6.2 MB H2D      wall %.3f ms per copy" % (1000 * (time.perf_counter() - t0) / K))
