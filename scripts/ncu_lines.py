"""Per-source-line hot spots of one kernel from an ncu --set full report.

  python scripts/ncu_lines.py <report.ncu-rep> <kernel-regex> [top]
Aggregates warp-stall samples and executed instructions per CUDA source line
(the 'source' page with cuda,sass interleaved), prints the top lines.
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
fname = ""
hdr = None
total_s = total_i = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue  # sass rows carry an address; keep the per-line cuda rows
    try:
        line = int(r[0])
        s = int(r[4] or 0)
        ins = int(r[7] or 0)
    except ValueError:
        continue
    key = (fname, line)
    a = agg.setdefault(key, [0, 0, r[1]])
    a[0] += s
    a[1] += ins
    total_s += s
    total_i += ins
print(f"total samples {total_s}, warp instructions {total_i}")
for (f, ln), (s, ins, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100.0 * s / max(1, total_s):5.1f}% samp {100.0 * ins / max(1, total_i):5.1f}% inst  {f}:{ln}  {src.strip()[:90]}")
