"""Summarise ncu output into the markdown tables kept under profiles/.

  python scripts/ncu_summary.py launches <launch.csv> [out.md]
      launch list of `ncu --metrics gpu__time_duration.sum --csv python bench.py --profile`
      -> per-kernel durations of the last full training iteration (preprocess .. adam)
  python scripts/ncu_summary.py full <report.ncu-rep> [out.md]
      `ncu --set full` capture -> per-kernel DRAM bytes, throughput, occupancy, top stalls

ncu times are cold-cache and serialised (one kernel at a time, caches flushed);
only each kernel's share of the step is comparable with bench.py's CUDA-event
phase times, not the absolute numbers.
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys

STALLS = ["barrier", "branch_resolving", "long_scoreboard", "short_scoreboard", "wait", "math_pipe_throttle",
          "mio_throttle", "lg_throttle", "not_selected", "no_instruction", "dispatch_stall", "membar", "drain"]


def short(name: str) -> str:
    n = name.split("(")[0].replace("void ", "")
    for p in ("sk::", "(anonymous namespace)::", "<unnamed>::", "unnamed>::"):
        n = n.replace(p, "")
    return n


def launch_avg(path: str):
    """[(kernel, us, dram_read_bytes, dram_write_bytes)] of one training
    iteration (each starts at preprocess): with several iterations captured,
    every launch position is averaged over them. Returns (list, iterations)."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[1:]:
        per.setdefault(int(r[ii]), {"k": short(r[ki])})[r[mi]] = float(r[vi].replace(",", ""))
    seq = [(d["k"], d.get("gpu__time_duration.sum", 0.0) / 1000.0, d.get("dram__bytes_read.sum"),
            d.get("dram__bytes_write.sum")) for _, d in sorted(per.items())]
    starts = [i for i, s in enumerate(seq) if s[0].startswith("preprocess")]
    steps = [seq[a:b] for a, b in zip(starts, starts[1:] + [len(seq)])]
    n = min(len(st) for st in steps)
    avg = []
    for j in range(n):
        ts = [st[j][1] for st in steps]
        rd = [st[j][2] for st in steps if st[j][2] is not None]
        wr = [st[j][3] for st in steps if st[j][3] is not None]
        avg.append((steps[0][j][0], sum(ts) / len(ts), sum(rd) / len(rd) if rd else None,
                    sum(wr) / len(wr) if wr else None))
    return avg, len(steps)


def launches(path: str) -> str:
    avg, nsteps = launch_avg(path)
    steps = range(nsteps)
    total = sum(t for _, t, _, _ in avg)
    out = [f"Average over {len(steps)} captured training iteration(s).", "",
           "| # | kernel | us | share | DRAM rd MB | DRAM wr MB |", "|---|---|---|---|---|---|"]
    f = lambda b: "" if b is None else f"{b / 1e6:.2f}"
    for j, (k, t, rd, wr) in enumerate(avg):
        out.append(f"| {j} | `{k}` | {t:.1f} | {100 * t / total:.1f}% | {f(rd)} | {f(wr)} |")
    out.append(f"| | **sum of kernels** | **{total:.1f}** | | | |")
    return "\n".join(out) + "\n"


def full(path: str) -> str:
    metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "sm__throughput.avg.pct_of_peak_sustained_elapsed",
               "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
               "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
               "smsp__issue_active.avg.pct_of_peak_sustained_active"]
    metrics += [f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio" for s in STALLS]
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    col = {m: h.index(m) for m in metrics}
    ki = h.index("Kernel Name")
    out = ["| kernel | us | DRAM rd MB | DRAM wr MB | DRAM GB/s | SM % | mem % | issue % | warps % | regs | top stalls (cycles/issue) |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    units = rows[1]
    tscale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    bscale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    for r in rows[2:]:
        t = float(r[col["gpu__time_duration.sum"]]) * tscale.get(units[col["gpu__time_duration.sum"]], 1e3)
        rd = float(r[col["dram__bytes_read.sum"]]) * bscale.get(units[col["dram__bytes_read.sum"]], 1.0)
        wr = float(r[col["dram__bytes_write.sum"]]) * bscale.get(units[col["dram__bytes_write.sum"]], 1.0)
        gbs = (rd + wr) * 1e6 / (t * 1e-6) / 1e9 if t > 0 else 0.0
        st = sorted(((float(r[col[f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"]] or 0), s)
                     for s in STALLS), reverse=True)[:3]
        stalls = ", ".join(f"{s} {v:.1f}" for v, s in st)
        out.append(f"| `{short(r[ki])}` | {t:.1f} | {rd:.1f} | {wr:.1f} | {gbs:.0f} | "
                   f"{float(r[col['sm__throughput.avg.pct_of_peak_sustained_elapsed']]):.0f} | "
                   f"{float(r[col['gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed']]):.0f} | "
                   f"{float(r[col['smsp__issue_active.avg.pct_of_peak_sustained_active']]):.0f} | "
                   f"{float(r[col['sm__warps_active.avg.pct_of_peak_sustained_active']]):.0f} | "
                   f"{r[col['launch__registers_per_thread']]} | {stalls} |")
    return "\n".join(out) + "\n"


def traffic(path: str) -> str:
    """DRAM bytes (read + write) per launch of each kernel, last capture of each."""
    import json
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    ur, uw = scale[rows[1][ri]], scale[rows[1][wi]]
    out = {}
    for r in rows[2:]:
        out[short(r[ki])] = int(float(r[ri]) * ur + float(r[wi]) * uw)
    return json.dumps({"source": path.split("/")[-1], "unit": "bytes per launch", "kernels": out}, indent=1) + "\n"


if __name__ == "__main__":
    mode, src = sys.argv[1], sys.argv[2]
    md = {"launches": launches, "full": full, "traffic": traffic}[mode](src)
    if len(sys.argv) > 3:
        open(sys.argv[3], "w").write(md)
    else:
        print(md)
