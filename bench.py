#!/usr/bin/env python
"""Benchmark: the 3DGS training iteration at 1M Gaussians / 1920x1080
(BASELINE.json config 2: "synthetic 1M-Gaussian scene, single 1920x1080 view,
forward+backward raster step on 1 B200").

A step is one training iteration (reference Trainer::train_iteration,
trainer.hpp:124-175): K1 preprocess, K2-K5 binning/sort, K6 forward blend,
K7 L1+D-SSIM loss, K8 backward blend, K9+K10 project-backward + dense Adam.
With N ranks each rank renders its own ring view; gradients are summed over
NCCL before Adam (view-parallel data parallelism), so a step processes N views.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints one JSON line (rank 0). `value` = train iterations (views) / s for the
whole job, inputs resident in HBM; `e2e` = the same through the C-ABI entry
point sk_train_step_host_async with every step's GT image copied from pinned
host memory (copy stream, overlapping the previous step) and every step's
loss read back (one step deferred, the last one inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0
METRIC = "train iters/s (1M Gaussians, 1080p)"
DATA = ("synthetic (numpy RNG, reference generate_synthetic distribution; GT rendered and quantised to 8 bits; "
        "trained scene = GT with perturbed positions)")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    # --gaussians under torchrun: its option parser takes "--n" for an abbreviation of its own flags
    ap.add_argument("--n", "--gaussians", dest="n", type=int, default=1_000_000)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no baselines, no clocks)")
    ap.add_argument("--workload", choices=["train", "event"], default="train",
                    help="train: config-2 training iteration (default); event: config-3 density event")
    ap.add_argument("--views", type=int, default=64, help="event workload: scored views (K)")
    ap.add_argument("--no-event", action="store_true", help="train workload: skip the config-3 event sub-object")
    return ap.parse_args()


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, 1965.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._h = None

    _BITS = [(0x8, "hw_slowdown"), (0x40, "hw_thermal_slowdown"), (0x20, "sw_thermal_slowdown"),
             (0x4, "sw_power_cap")]

    def _nvml_open(self):
        """NVML handle opened before the timed region starts (its first call
        can take longer than a short timed region), or None."""
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._pynvml = pynvml
            return h
        except Exception:
            return None

    def _sample_nvml(self):
        pynvml, h = self._pynvml, self._h
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        self.samples.append([str(sm), str(self._mx), "0"] + ["Active" if r & b else "Not Active" for b, _ in self._BITS])

    def _run_nvml(self):
        while not self._stop.is_set():
            self._sample_nvml()
            self._stop.wait(0.005)

    def _run(self):
        if self._h is not None:
            try:
                self._run_nvml()
                return
            except Exception:
                pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._h = self._nvml_open()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        # the region just ended with the GPU still clocked for it: a region
        # shorter than the sampling period still gets one sample
        if self._h is not None and not self.samples:
            try:
                self._sample_nvml()
            except Exception:
                pass
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# Ranks sharing GPUs (more ranks than visible devices: a one-GPU box checking
# the multi-rank path) run over gloo with the library's host-callback
# communicator (sk.HostComm), since NCCL refuses two ranks on one device. Such
# a run checks the plumbing; it is not a scaling measurement and says so.
_SHARED = False


def init_dist(world, local):
    """torch.cuda device + process group; returns (dist or None, device)."""
    global _SHARED
    import torch
    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev
    torch.cuda.set_device(dev)
    if world <= 1:
        return None, dev
    import torch.distributed as dist
    _SHARED = ndev < world
    if _SHARED:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    return dist, dev


def make_comm(sk, ctx, dist, rank, world):
    return sk.HostComm(ctx, dist, rank, world) if _SHARED else sk.Comm.from_torch(ctx, dist, rank, world)


def allmax(dist, x):
    """max over ranks of a host float (the timing rule: slowest rank)."""
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if _SHARED else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def bench_config(args, world):
    """The `config` object of both arms (identical by construction)."""
    return {"workload": "config2: synthetic 1M-Gaussian scene (SH deg 3), 1920x1080 ring view per rank, "
                        "train iteration K1-K10 (fwd+loss+bwd+Adam)",
            "n_gaussians": args.n, "width": args.width, "height": args.height, "sh_degree": 3,
            "views_per_step": world,
            "start_state": "timed steps are training iterations 1..K from the perturbed initial scene with fresh "
                           "Adam state (warm-up steps run first, then scene and optimizer are restored)",
            "l2": "inputs larger than L2 (944 MB params+moments+grads state per step)",
            "parallelism": (f"view-parallel dp{world} (gradient reduce-scatter / all-gather)"
                            + (" - ranks sharing one GPU over host collectives: a plumbing check, not a scaling "
                               "number" if _SHARED else "")) if world > 1 else "single device"}


def train_config(default_config, iterations=30000):
    """TrainConfig of the bench step; `default_config` is the arm's own
    (sk.default_config for ours, orc.default_config for the reference)."""
    cfg = default_config()
    cfg.iterations = iterations
    cfg.densify_from = cfg.densify_until = 1 << 30  # the bench step has no density events
    return cfg


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle (restated reference) on the host cores
# ---------------------------------------------------------------------------

def run_reference(args, world, rank):
    """The reference's CPU implementation of the path (the oracle restatement,
    oracle/; the reference itself cannot be built here)
    on this box's host cores, on our arm's config, metric and unit. Nothing of
    the product (libsplatkit_b200.so) is loaded in this process."""
    if rank != 0:
        return
    import paper_2511_04283_b200.synthetic as syn  # pure numpy; never loads the CUDA library
    from oracle import oracle as orc
    cores = os.cpu_count() or 1
    gt = syn.gaussians(args.n, 1, 3)
    cam = syn.ring_camera(0, 64, args.width, args.height, camera_fn=orc.camera)
    r = orc.render_scene(gt, 3, cam, workers=cores, values_cap=64 * args.n)
    gt8 = syn.quantize_u8(r.image)
    extent = syn.ring_extent()
    p = syn.perturb_positions(gt, 0.02 * extent, 2)
    del gt, r
    cfg = train_config(orc.default_config)
    cfg.workers = cores
    budget_s = float(os.environ.get("SK_REF_BUDGET_S", "150"))
    # warm-up on a throw-away trainer, then iterations 1..K from the initial
    # scene (the same start state as our arm); bounded by a time budget
    warm = orc.ViewTrainer(p, 3, cam, gt8, cfg, extent)
    wsecs = [warm.run(1)[1] for _ in range(args.warmup)]
    del warm
    tr = orc.ViewTrainer(p, 3, cam, gt8, cfg, extent)
    secs = []
    while len(secs) < args.steps and (not secs or sum(secs) + sum(wsecs) < budget_s):
        secs.append(tr.run(1)[1])
    del tr
    ms = 1000.0 * sum(secs) / len(secs)
    value = 1000.0 / ms
    # the reference's bit-reproducible mode (workers=1, proj/README.md:75-78):
    # one iteration from the initial scene
    w1 = None
    if not os.environ.get("SK_REF_NO_W1"):
        cfg1 = train_config(orc.default_config)
        cfg1.workers = 1
        t1 = orc.ViewTrainer(p, 3, cam, gt8, cfg1, extent)
        s1 = t1.run(1)[1]
        w1 = {"value": 1.0 / s1, "unit": "iter/s", "cores": 1, "kind": "port",
              "sample": "1 full config-2 training iteration (iteration 1) at workers=1"}
    line = {"impl": "reference", "metric": METRIC, "value": value,
            "unit": "iter/s", "n_gpus": world, "steps": len(secs), "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": DATA, "config": bench_config(args, world),
            "cpu_baseline": {"value": value, "unit": "iter/s", "cores": cores, "kind": "port",
                             "sample": f"{len(secs)} full config-2 training iterations (1..{len(secs)}) after "
                                       f"{args.warmup} warm-up iterations (oracle, workers={cores}; bounded to "
                                       f"~{budget_s:.0f} s)"},
            "cpu_baseline_workers1": w1,
            "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

PHASES = ["K1 preprocess", "K2-K5 bin+sort", "K6 blend fwd", "K7 loss", "K8 blend bwd", "K9 proj-bwd", "K10 Adam"]


def algorithmic_bytes(phase, n, visible, pairs, pixels, tiles, comps=59):
    """Algorithmic HBM bytes per launch of each phase, SURVEY.md §8(d)'s
    per-unit figures x the units one launch processes."""
    culled = n - visible
    if phase == 0:  # K1: 236 B params read + 52 B projected record written per visible, 44 B per culled
        return (4 * comps + 52) * visible + 44 * culled
    if phase == 1:  # K2 scan 8 B/Gaussian; K3 12 B/pair + 20 B/visible; K4 8 + 6x24 B/pair; K5 8 B/pair + 8 B/tile
        return 8 * n + 12 * pairs + 20 * visible + 152 * pairs + 8 * pairs + 8 * tiles
    if phase == 2:  # K6 HBM side: 36 B per pair + 20 B per pixel
        return 36 * pairs + 20 * pixels
    if phase == 3:  # K7: 36 B per pixel minimum (read r, g; write dL)
        return 36 * pixels
    if phase == 4:  # K8 HBM side: per pair record + per pixel T, last, dL/dimage + 11 gradient floats per visible
        return 36 * pairs + 20 * pixels + 44 * visible
    if phase == 5:  # K9: 236 B read + 44 B blend grads + 236 B written + 56 B stats RMW per visible
        return (4 * comps * 2 + 44 + 56) * visible
    if phase == 6:  # K10 Adam: 59 x 28 B per Gaussian
        return 28 * comps * n
    return 0


def implementation_bytes(phase, n, visible, pairs, pixels, fused=False):
    """Bytes the kernels of this implementation must move at minimum (the
    B200 design moves less than the SURVEY's figures: a 4-pass depth sort
    over N slots + the counting scatter of the tile lists instead of a 64-bit
    pair sort; K9+K10 fused keep the gradients on chip)."""
    if phase == 0:
        # params: 236 B read per visible Gaussian, 44 B (mean, rotation, scale,
        # opacity) per culled one; written: mean2d 8 + conic/opacity 16 +
        # colour/depth 16 + full conic 16 + radius 4 + tile rect 16 + depth key
        # 4 = 80 B per visible, radius + rect + key = 24 B per culled slot
        return (4 * 59 + 80) * visible + (44 + 24) * (n - visible)
    if phase == 1:
        # depth sort: hist read 4 B + 4 passes x 16 B per slot; K3: order +
        # rectangle (20 B) twice per slot, the Gaussian index per pair
        return 4 * n + 64 * n + 40 * n + 4 * pairs
    if phase == 5 and fused:
        # params / m / v read + written (6 x 236 B per Gaussian), projected
        # radius + conic (20 B), blend gradients + statistics per visible (100 B)
        return 6 * 4 * 59 * n + 20 * n + 100 * visible
    return None


def phase_names(fused):
    names = list(PHASES)
    if fused:
        names[5] = "K9+K10 proj-bwd+Adam (fused)"
    return names


# SURVEY §8(d) FP32 work of the blend kernels per pixel-Gaussian evaluation:
# forward 14 flop per visited + 9 per contributing (+1 ex2 per visited);
# backward 14 per visited + 52 per contributing (+1 ex2 per visited, +1 ex2
# and 1 division per contributing). "Visited" = the entries the reference's
# per-pixel loop examines (raster.hpp:219-235), measured by sk_frame_pge_counts.
FLOP_FWD = (14, 9)
FLOP_BWD = (14, 52)


def ncu_traffic(kernel_prefix):
    """DRAM bytes per launch of a kernel from the committed ncu capture
    (profiles/traffic.json, written by scripts/ncu_summary.py traffic)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        for k, v in d["kernels"].items():
            if k.startswith(kernel_prefix):
                return v
    except Exception:
        pass
    return None


def run_ours(args, world, rank, local):
    import torch

    import paper_2511_04283_b200 as sk
    import paper_2511_04283_b200.synthetic as syn

    dist, dev = init_dist(world, local)
    ctx = sk.Context(dev)
    stream = torch.cuda.current_stream()
    ctx.check(ctx._lib.sk_ctx_set_stream(ctx.h, sk.C.c_void_p(stream.cuda_stream)))

    extent = syn.ring_extent()
    gt_params = syn.gaussians(args.n, 1, 3)
    cam = syn.ring_camera(rank, 64, args.width, args.height)
    gt8 = syn.render_gt_u8(ctx, gt_params, 3, cam)
    params = syn.perturb_positions(gt_params, 0.02 * extent, 2)
    del gt_params
    cfg = train_config(sk.default_config)
    scene = ctx.scene(params, 3)
    data = sk.Dataset(ctx, [cam], [gt8], [0], extent)
    trainer = sk.Trainer(ctx, scene, data, cfg)
    comm = None
    if world > 1:
        comm = make_comm(sk, ctx, dist, rank, world)
        trainer.set_comm(comm)

    def barrier():
        if dist is not None:
            dist.barrier()

    def restore():
        """The fixed start state of every timed region: the perturbed initial
        scene, fresh Adam moments / step counters and score table
        (sk_scene_upload resets both), iteration counter 0."""
        ctx.check(ctx._lib.sk_scene_upload(ctx.h, scene.h, sk._p(params), sk.C.c_int64(args.n)))
        trainer.set_iteration(0)

    for _ in range(args.warmup):
        trainer.run(1)
    restore()
    torch.cuda.synchronize()

    # ---- device-resident timed region: iterations 1..K --------------------
    # No phase marks inside the timed region (as event-record nodes of the
    # captured step they cost time); the phase split comes from a second pass
    # over the same iterations below. --profile (ncu) keeps one marked run.
    ctx.check(ctx._lib.sk_ctx_reset_timing(ctx.h))
    ctx.check(ctx._lib.sk_ctx_enable_timing(ctx.h, 1 if args.profile else 0))
    launches0 = ctx.launch_count()
    gs0 = sk.C.c_int64()
    ctx.check(ctx._lib.sk_ctx_graph_steps(ctx.h, sk.C.byref(gs0)))
    graph_steps0 = gs0.value
    clock = ClockSampler(dev)
    rows = []
    with (clock if not args.profile else _Null()):
        barrier()
        torch.cuda.synchronize()
        if args.profile:  # `ncu --profile-from-start off` then captures exactly the timed steps
            torch.cuda.cudart().cudaProfilerStart()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rows = trainer.run(args.steps)  # Trainer::run: each step's readback completes during the next
        e1.record(stream)
        torch.cuda.synchronize()
        if args.profile:
            torch.cuda.cudart().cudaProfilerStop()
        barrier()
    launches = ctx.launch_count() - launches0
    gs = sk.C.c_int64()
    ctx.check(ctx._lib.sk_ctx_graph_steps(ctx.h, sk.C.byref(gs)))
    graph_steps = gs.value - graph_steps0
    ctx.check(ctx._lib.sk_ctx_enable_timing(ctx.h, 0))
    ms = e0.elapsed_time(e1) / args.steps
    if not args.profile:
        # phase split: iterations 1..K again from the same start state, with
        # CUDA-event marks between the phases
        restore()
        torch.cuda.synchronize()
        ctx.check(ctx._lib.sk_ctx_reset_timing(ctx.h))
        ctx.check(ctx._lib.sk_ctx_enable_timing(ctx.h, 1))
        trainer.run(args.steps)
        torch.cuda.synchronize()
        ctx.check(ctx._lib.sk_ctx_enable_timing(ctx.h, 0))
    phase_ms = (sk.C.c_double * len(PHASES))()
    nsteps = sk.C.c_int64()
    ctx._lib.sk_ctx_get_timing(ctx.h, phase_ms, sk.C.byref(nsteps))
    phase_avg = [phase_ms[i] / max(1, nsteps.value) for i in range(len(PHASES))]
    # one GPU: K9 and K10 run as one fused kernel (optim.cu project_bwd_adam_kernel),
    # timed as one phase; the K10 slot is then empty
    fused = world == 1
    if fused:
        phase_avg[5] += phase_avg[6]
        phase_avg[6] = 0.0
    if dist is not None:
        ms = allmax(dist, ms)
    if args.profile:
        if rank == 0:
            print(json.dumps({"profile": True, "ms_per_step": ms, "phase_ms": phase_avg,
                              "tile_pairs_last": rows[-1]["tile_pairs"] if rows else None}), flush=True)
        return

    # ---- end-to-end through the C ABI with host buffers -----------------
    pinned = torch.empty(gt8.size, dtype=torch.uint8, pin_memory=True)
    gt_host = pinned.numpy().reshape(gt8.shape)
    gt_host[...] = gt8
    # Same start state and trajectory as the device-timed run: warm-up steps
    # (the e2e frame allocates its buffers on first use), then restore and
    # time iterations 1..K.
    e2e_scene = scene
    pipe = sk.HostStepPipeline(ctx, comm=comm)
    for k in range(args.warmup):
        pipe.step(e2e_scene, cam, gt_host, cfg, extent, 1 + k)
    pipe.flush()
    restore()
    it0 = 0
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    # every step: H2D of its GT from pinned host memory (copy stream,
    # overlapping the previous step) and a D2H read of its loss (completed
    # when the next step is issued; the last one by flush())
    for k in range(args.steps):
        pipe.step(e2e_scene, cam, gt_host, cfg, extent, it0 + 1 + k)
    e2e_rows = pipe.flush()
    f1.record(stream)
    torch.cuda.synchronize()
    assert len(e2e_rows) == args.steps and all(np.isfinite(r["loss"]) for r in e2e_rows)
    wall_ms = 1000.0 * (time.perf_counter() - t0) / args.steps
    e2e_ms = max(f0.elapsed_time(f1) / args.steps, wall_ms)
    if dist is not None:
        e2e_ms = allmax(dist, e2e_ms)

    # ---- workload units of the timed steps --------------------
    # visible Gaussians and the reference loop's visited / contributing
    # pixel-Gaussian evaluations, measured at the start state (iteration 1)
    # and at the end state (after iteration K) and averaged; pairs = the
    # mean over the timed steps' own counts.
    def units():
        prj = ctx.project_scene(scene, cam)
        ctx.build_tile_grid()
        ctx.blend_forward()
        return (int(prj.visible.sum()),) + tuple(ctx.pge_counts())
    end_units = units()
    restore()
    start_units = units()
    visible, visited, contribs = (int(round((a + b) / 2)) for a, b in zip(start_units, end_units))
    pairs = int(round(sum(r["tile_pairs"] for r in rows) / len(rows))) if rows else 0

    # ---- the paper's contribution: one config-3 density event ---------------
    event = None
    if not args.no_event:
        event = measure_event(ctx, sk, torch, dist, rank, args.n, args.views, args.width, args.height, reps=3,
                              warm=1)

    if rank != 0:
        return
    # ---- roofline of the dominant kernel ------------------------------------
    hbm_peak, sm_max, peak_kind = measured_peaks()
    pixels = args.width * args.height
    tiles = ((args.width + 15) // 16) * ((args.height + 15) // 16)
    clocks = clock.summary()
    # FP32 SIMT roof: 148 SMs x 128 lanes x 2 flop (FFMA) x SM clock. The SM
    # clock is the max clock (MEASURED_PEAKS sm_max_mhz), which the run held.
    fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12
    mufu_peak = 148 * 16 * sm_max * 1e6 / 1e12  # ex2 per s (T/s)
    blend = {}
    for ph, (fv, fc), ex in ((4, FLOP_BWD, (1, 1)), (2, FLOP_FWD, (1, 0))):
        fl = fv * visited + fc * contribs
        t = phase_avg[ph] * 1e-3
        blend[ph] = {"achieved": fl / t / 1e12, "peak": fp32_peak, "unit": "TFLOP/s",
                     "frac": fl / t / 1e12 / fp32_peak, "flop": fl,
                     "flop_per_visited": fv, "flop_per_contributing": fc, "kernel_ms": phase_avg[ph],
                     "ex2_frac_of_mufu": (ex[0] * visited + ex[1] * contribs) / t / 1e12 / mufu_peak,
                     "hbm_GB/s": algorithmic_bytes(ph, args.n, visible, pairs, pixels, tiles) / t / 1e9}
    phase_kernel = {4: "blend_bwd_kernel", 2: "blend_fwd_warp_kernel", 5: "project_bwd_kernel", 6: "adam_kernel",
                    0: "preprocess_kernel"}
    dom = int(np.argmax(phase_avg))
    if dom in blend:
        r = blend[dom]
        roofline = {"bound": "fp32", "kernel": PHASES[dom], "achieved": r["achieved"], "peak": r["peak"],
                    "unit": "TFLOP/s", "frac": r["frac"], "traffic": ncu_traffic(phase_kernel[dom]),
                    "peak_kind": "computed: 148 SMs x 128 FP32 lanes x 2 x sm_max_mhz (MEASURED_PEAKS)",
                    "algorithmic_flop": r["flop"], "kernel_ms": r["kernel_ms"],
                    "note": "blend kernels are FP32/issue-bound (SURVEY 8(d)); HBM side in hbm_GB/s of roofline_fp32; "
                            "traffic = ncu DRAM bytes per launch"}
    else:
        alg = algorithmic_bytes(dom, args.n, visible, pairs, pixels, tiles)
        ach = alg / (phase_avg[dom] * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": PHASES[dom], "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                    "frac": ach / hbm_peak, "traffic": ncu_traffic(phase_kernel.get(dom, "?")),
                    "peak_kind": peak_kind, "algorithmic_bytes": alg, "kernel_ms": phase_avg[dom]}
    roofline_fp32 = {PHASES[ph]: blend[ph] for ph in (4, 2)}
    # K7: ~1.15 kflop per pixel (24 filtered maps x 2 separable
    # 11-tap passes + the per-pixel SSIM terms), FP32-bound
    k7_flop = 1150.0 * pixels
    roofline_fp32[PHASES[3]] = {"achieved": k7_flop / (phase_avg[3] * 1e-3) / 1e12, "peak": fp32_peak,
                                "unit": "TFLOP/s", "frac": k7_flop / (phase_avg[3] * 1e-3) / 1e12 / fp32_peak,
                                "flop": k7_flop, "flop_per_pixel": 1150, "kernel_ms": phase_avg[3]}
    roofline_fp32["pge_visited"] = visited
    roofline_fp32["pge_contributing"] = contribs
    hbm_kernels = {}
    names = phase_names(fused)
    for ph in ((0, 1, 3, 5) if fused else (0, 1, 3, 5, 6)):
        b = algorithmic_bytes(ph, args.n, visible, pairs, pixels, tiles)
        if fused and ph == 5:
            b += algorithmic_bytes(6, args.n, visible, pairs, pixels, tiles)
        gbs = b / (phase_avg[ph] * 1e-3) / 1e9
        hbm_kernels[names[ph]] = {"ms": phase_avg[ph], "algorithmic_MB": b / 1e6, "GB/s": gbs,
                                  "frac": gbs / hbm_peak}
        ib = implementation_bytes(ph, args.n, visible, pairs, pixels, fused)
        if ib is not None:
            hbm_kernels[names[ph]]["implementation_min_MB"] = ib / 1e6
            hbm_kernels[names[ph]]["implementation_frac"] = ib / (phase_avg[ph] * 1e-3) / 1e9 / hbm_peak

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, params, cam, gt8, extent)

    line = {
        "metric": METRIC,
        "value": world * 1000.0 / ms,
        "unit": "iter/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": DATA,
        "config": bench_config(args, world),
        # raster forward = K1..K6, raster backward = K8 + K9 (pixels / s)
        "raster_fwd_mpix_s": pixels / ((phase_avg[0] + phase_avg[1] + phase_avg[2]) * 1e-3) / 1e6,
        "raster_bwd_mpix_s": pixels / ((phase_avg[4] + phase_avg[5]) * 1e-3) / 1e6,
        "phase_ms": {nm: round(x, 4) for nm, x, ph in zip(names, phase_avg, range(7)) if not (fused and ph == 6)},
        "tile_pairs": pairs,
        "visible": visible,
        "workload_units": {"start": dict(zip(("visible", "pge_visited", "pge_contributing"), start_units)),
                           "end": dict(zip(("visible", "pge_visited", "pge_contributing"), end_units)),
                           "tile_pairs_first_last": [rows[0]["tile_pairs"], rows[-1]["tile_pairs"]] if rows else None},
        "loss_last": rows[-1]["loss"] if rows else None,
        "roofline": roofline,
        "roofline_fp32": roofline_fp32,
        "hbm_kernels": hbm_kernels,
        "e2e": {"value": world * 1000.0 / e2e_ms, "unit": "iter/s", "h2d_bytes_per_step": int(gt8.size),
                "d2h_bytes_per_step": 44, "ms_per_step": e2e_ms},
        "gpu_launches": launches,
        "graph_steps": graph_steps,  # timed steps launched as the captured CUDA graph (the rest: plain launches)
        "clocks": clocks,
        "cpu_baseline": cpu,
        "event": event,
    }
    print(json.dumps(line), flush=True)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False

    def summary(self):
        return {}


def cpu_baseline(args, params, cam, gt8, extent):
    """The restated reference (oracle) on the host cores: one warm-up
    iteration on a throw-away trainer, then iterations 1..k from the initial
    scene (our arm's start state), bounded to ~12 s."""
    try:
        from oracle import oracle as orc
        cores = os.cpu_count() or 1
        cfg = train_config(orc.default_config)
        cfg.workers = cores
        orc.ViewTrainer(params, 3, cam, gt8, cfg, extent).run(1)  # warm-up (allocations, page-in)
        tr = orc.ViewTrainer(params, 3, cam, gt8, cfg, extent)
        secs = []
        while not secs or (sum(secs) < 12.0 and len(secs) < 8):
            secs.append(tr.run(1)[1])
        return {"value": len(secs) / sum(secs), "unit": "iter/s", "cores": cores, "kind": "port",
                "sample": f"{len(secs)} full config-2 training iterations (1..{len(secs)}, 1M Gaussians, 1920x1080) "
                          f"from the initial scene, oracle workers={cores}"}
    except Exception as e:  # the baseline is reported, never required
        return {"value": None, "unit": "iter/s", "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}


# ---------------------------------------------------------------------------
# config 3: the multi-view importance pass + densify / prune compaction
# ---------------------------------------------------------------------------

def measure_event(ctx, sk, torch, dist, rank, n, k, width, height, reps, warm):
    """BASELINE config 3: n Gaussians scored over K views
    (K1-K6 + K11 + K7-fwd + K12 per view, K13 scores), then K14 selection and
    K15 compaction, through Trainer::density_event (trainer.hpp:177-243).
    Scene: the GT of the GPU synthetic generator padded to SH degree 3, with
    20% of the Gaussians' DC and opacity perturbed (seed 3); accumulators
    synthetic (grad ~ U(0, 6e-4), views_seen in [1, 10]). Timed at iteration
    1000 (densify + prune) and 20000 (late prune); the scene and table are
    restored before every event. Returns the event dict (rank 0) or None."""
    t0 = time.perf_counter()
    ds, gt, _, _ = sk.Dataset.synthetic(ctx, n_gaussians=n, n_views=k, width=width, height=height, seed=1,
                                        scale_mult=(500.0 / n) ** (1.0 / 3.0) if n >= 100_000 else 1.0,
                                        focal=1.1 * height * 2.6)
    gen_s = time.perf_counter() - t0
    ds.set_train_indices(np.arange(k))  # K = all views
    p1 = gt.download()
    gt.close()
    p = np.zeros((sk.n_components(3), n), np.float32)
    p[: p1.shape[0]] = p1
    del p1
    rng = np.random.default_rng(3)
    sel = rng.random(n) < 0.2
    p[10, sel] += rng.normal(0.0, 1.0, int(sel.sum())).astype(np.float32)
    p[11:14, sel] += rng.normal(0.0, 0.5, (3, int(sel.sum()))).astype(np.float32)
    vs = rng.integers(1, 11, n).astype(np.int32)
    grad = rng.uniform(0, 6e-4, n).astype(np.float32)
    absg = rng.uniform(0, 6e-4, n).astype(np.float32)
    g3 = rng.normal(0, 1e-4, (n, 3)).astype(np.float32)
    rad = rng.uniform(0, 30, n).astype(np.float32)
    cfg = train_config(sk.default_config)
    cfg.k = k
    scene = ctx.scene(p, 3, capacity=2 * n)
    tr = sk.Trainer(ctx, scene, ds, cfg)
    if dist is not None:
        tr.set_comm(make_comm(sk, ctx, dist, rank, dist.get_world_size()))

    def restore():
        ctx.check(ctx._lib.sk_scene_upload(ctx.h, scene.h, sk._p(p), sk.C.c_int64(n)))
        scene.set_score_table(grad_norm_acc=grad * vs, abs_grad_acc=absg * vs, grad3d_acc=g3, views_seen=vs,
                              max_radius2d=rad)

    def phases():
        ms = (sk.C.c_double * 4)()
        cnt = sk.C.c_int64()
        ctx._lib.sk_ctx_get_event_timing(ctx.h, ms, sk.C.byref(cnt))
        mv = sk.C.c_double()
        ctx._lib.sk_ctx_get_compact_kernel_ms(ctx.h, sk.C.byref(mv))
        return [ms[i] / max(1, cnt.value) for i in range(4)] + [mv.value / max(1, cnt.value)]

    def timed(iteration, densify, prune):
        restore()
        ctx.check(ctx._lib.sk_ctx_reset_timing(ctx.h))
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        a = time.perf_counter()
        tr.density_event(iteration, densify, prune)
        torch.cuda.synchronize()
        ms = 1000.0 * (time.perf_counter() - a)
        if dist is not None:
            ms = allmax(dist, ms)
        return ms, scene.size, phases()

    ctx.check(ctx._lib.sk_ctx_enable_timing(ctx.h, 1))
    for _ in range(warm):
        timed(1000, True, True)
    early = [timed(1000, True, True) for _ in range(reps)]
    late = [timed(20000, False, True) for _ in range(reps)]
    ctx.check(ctx._lib.sk_ctx_enable_timing(ctx.h, 0))
    tr.close()
    scene.close()
    ds.close()
    if rank != 0:
        return None
    # the phase split reported is that of the median event (by wall time)
    e_med = sorted(early, key=lambda x: x[0])[len(early) // 2]
    l_med = sorted(late, key=lambda x: x[0])[len(late) // 2]
    hbm_peak, _, peak_kind = measured_peaks()
    comps = sk.n_components(3)

    def event_roofline(ph, n_out):
        # K13: int32 count rows (4 B x K x N) read, s_d / s_p_raw / s_p written
        # and s_p_raw re-read by the min-max pass (16 B x N).
        k13 = 4 * k * n + 16 * n
        # K14 + K15: params + m + v, 3 x 4 x 59 = 708 B read and
        # written per output Gaussian, plus the three flag bytes per input.
        k1415 = 2 * 3 * 4 * comps * n_out + 3 * n
        t13, t1415 = ph[1] * 1e-3, (ph[2] + ph[3]) * 1e-3
        # the K15 row-move kernel alone (CUDA events around it): the same
        # row bytes without the flags, the class scans and the host round
        # trip for the split normals that the phase time includes
        mv_b, t_mv = 2 * 3 * 4 * comps * n_out, ph[4] * 1e-3
        return {"phase_ms": dict(zip(["K6+K11+K12 views (+K1-K5, K7 fwd)", "K13 scores", "K14 select",
                                      "K15 compact"], [round(x, 4) for x in ph[:4]])),
                "K15 move kernel": {"ms": round(ph[4], 4), "algorithmic_MB": mv_b / 1e6,
                                    "GB/s": mv_b / t_mv / 1e9 if t_mv > 0 else None,
                                    "frac": mv_b / t_mv / 1e9 / hbm_peak if t_mv > 0 else None},
                "K13": {"algorithmic_MB": k13 / 1e6, "GB/s": k13 / t13 / 1e9, "frac": k13 / t13 / 1e9 / hbm_peak},
                "K14+K15": {"algorithmic_MB": k1415 / 1e6, "GB/s": k1415 / t1415 / 1e9,
                            "frac": k1415 / t1415 / 1e9 / hbm_peak},
                "view_ms": ph[0] / k, "peak_GB/s": hbm_peak, "peak_kind": peak_kind}
    return {
        "metric": f"density event ms (config 3: {n} Gaussians, {k} views {width}x{height}, score + select + compact)",
        "value": e_med[0], "unit": "ms/event", "higher_is_better": False, "reps": reps, "warmup": warm,
        "config": {"workload": "config3: multi-view importance pass over K views + densify/prune compaction",
                   "n_gaussians": n, "views": k, "width": width, "height": height,
                   "timing": "wall clock around Trainer::density_event with device syncs, median; phase split "
                             "(CUDA events) of that median event"},
        "early_event_ms": e_med[0], "late_event_ms": l_med[0],
        "views_scored_per_s": k / (e_med[0] * 1e-3),
        "n_after_early": e_med[1], "n_after_late": l_med[1],
        "early": event_roofline(e_med[2], e_med[1]), "late": event_roofline(l_med[2], l_med[1]),
        "generator_s": gen_s,
    }


def run_event(args, world, rank, local):
    """`--workload event`: the config-3 event alone as the JSON line."""
    import torch

    import paper_2511_04283_b200 as sk

    dist, dev = init_dist(world, local)
    ctx = sk.Context(dev)
    stream = torch.cuda.current_stream()
    ctx.check(ctx._lib.sk_ctx_set_stream(ctx.h, sk.C.c_void_p(stream.cuda_stream)))
    ev = measure_event(ctx, sk, torch, dist, rank, args.n, args.views, args.width, args.height,
                       reps=max(1, min(args.steps, 5)), warm=max(1, min(args.warmup, 2)))
    if rank != 0:
        return
    line = dict(ev, n_gpus=world, steps=ev["reps"], scaling="strong", vs_baseline=None, dtype="f32",
                data="synthetic (GPU generator, reference Rng draw order); scene restored before each event")
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    if args.workload == "event":
        run_event(args, world, rank, local)
        return
    run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
