"""Writes profiles/r1_ncu.md, profiles/r1_launches.csv and profiles/traffic.json
from one scripts/gpu_profile.sh capture (tag) plus its bench line.

    python scripts/make_profile_md.py <tag>
"""
import json
import shutil
import subprocess
import sys

tag = sys.argv[1]
g = f"gpurun_out"


def run(*a):
    return subprocess.run(["python", *a], capture_output=True, text=True, check=True).stdout


launches = run("scripts/ncu_summary.py", "launches", f"{g}/launches_{tag}.csv")
full = run("scripts/ncu_summary.py", "full", f"{g}/full_{tag}.ncu-rep")
fullb = run("scripts/ncu_summary.py", "full", f"{g}/fullb_{tag}.ncu-rep")
hb = run("scripts/ncu_lines.py", f"{g}/full_{tag}.ncu-rep", "blend_bwd", "20")
hf = run("scripts/ncu_lines.py", f"{g}/full_{tag}.ncu-rep", "blend_fwd_warp", "20")
shutil.copy(f"{g}/launches_{tag}.csv", "profiles/r1_launches.csv")
a = json.loads(run("scripts/ncu_summary.py", "traffic", f"{g}/full_{tag}.ncu-rep"))
b = json.loads(run("scripts/ncu_summary.py", "traffic", f"{g}/fullb_{tag}.ncu-rep"))
k = dict(b["kernels"])
k.update(a["kernels"])
json.dump({"source": f"full_{tag}.ncu-rep + fullb_{tag}.ncu-rep (steady state, after 150 training iterations)",
           "unit": "bytes per launch", "kernels": k}, open("profiles/traffic.json", "w"), indent=1)
d = json.load(open(f"{g}/bench_{tag}.json"))
ph = d["phase_ms"]
rf = d["roofline_fp32"]
phases = ", ".join(f"{n.split(' ', 1)[1]} {v:.3f}" for n, v in ph.items())
md = f"""# Round 1 — ncu evidence (B200, sm_100a), final state of the round

Workload: `bench.py` config 2 — 1,000,000 Gaussians (SH degree 3), one 1920×1080 view,
one training iteration (K1 preprocess … K10 Adam, 19 launches), captured at **steady state**:
after 150 training iterations, the state the bench's timed region sees (the per-step workload
drifts as the scene trains). Commands (`scripts/gpu_profile.sh {tag} tests 150`, summarised by
`scripts/make_profile_md.py {tag}`):

```
ncu --metrics gpu__time_duration.sum --clock-control none --csv -s 2850 -c 60 \\
    --log-file gpurun_out/launches_{tag}.csv python bench.py --profile --steps 2 --warmup 150
ncu --set full --import-source on --clock-control none -k regex:"blend_fwd|blend_bwd" -s 301 -c 2 \\
    -o gpurun_out/full_{tag} python bench.py --profile --steps 2 --warmup 150
ncu --set full --import-source on --clock-control none \\
    -k regex:"preprocess|duplicate|onesweep|ssim|project_bwd|adam|scan_gather|tile_ranges" -s 2110 -c 14 \\
    -o gpurun_out/fullb_{tag} python bench.py --profile --steps 1 --warmup 150
```

ncu serialises kernels and flushes caches between them, so absolute times are cold-cache; the
**shares** agree with bench.py's CUDA-event phase split of the same code (BENCH {tag}, ms:
{phases}; {d['value']:.1f} it/s device-resident, {d['e2e']['value']:.1f} it/s end to end).

## 1. Launch list of one training iteration

{launches}
## 2. Full-set metrics: blend kernels

{full}
## 3. Full-set metrics: streaming kernels

{fullb}
## 4. Where the blend kernels spend their issue slots (per CUDA line, top 20)

K8 `blend_bwd_kernel<16, 2>` (warp samples, executed warp instructions):

```
{hb}```

K6 `blend_fwd_warp_kernel<16, 2>`:

```
{hf}```

## Reading

* The blend kernels are **issue-bound** (stalls dominated by `not_selected` and fixed-latency
  `wait`) with small DRAM traffic: their roof is the FP32/ALU issue rate. Against SURVEY §8(d)'s
  algorithmic FP32 work (14 flop per visited + 9 / 52 per contributing pixel–Gaussian
  evaluation; PGE_v = {rf['pge_visited'] / 1e6:.1f}M and PGE_c = {rf['pge_contributing'] / 1e6:.1f}M measured on
  the frame), K6 reaches {rf['K6 blend fwd']['achieved']:.1f} TFLOP/s ({100 * rf['K6 blend fwd']['frac']:.0f}% of
  {rf['K6 blend fwd']['peak']:.1f}) and K8 {rf['K8 blend bwd']['achieved']:.1f} TFLOP/s
  ({100 * rf['K8 blend bwd']['frac']:.0f}%): the other issue slots go to the exactness machinery
  (non-contracted round-to-nearest q, the deterministic exp, threshold re-checks), the warp
  reduce-scatter (23 shuffles per entry pair) and lanes of partially covered 8×8 blocks.
* HBM-bound kernels: Adam ≈6.0 TB/s (≈92% of the 6.53 TB/s copy roof), preprocess ≈4.9 TB/s of
  DRAM traffic, project-backward ≈3.4 TB/s (latency-bound at 128 registers).
* The tile-id onesweep passes are `short_scoreboard`-bound: a third of their samples wait on the
  MATCH.ANY results of the stable warp ranking; they run out of L2.
"""
open("profiles/r1_ncu.md", "w").write(md)
print("ok")
