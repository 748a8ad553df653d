"""Diagnostic: CUB (torch.sort, stable) on 7.6M 13-bit keys + int32 values,
to compare its per-pass cost with the onesweep tile sort."""
import torch
n = 7_600_000
k = torch.randint(0, 8160, (n,), dtype=torch.int32, device="cuda")
v = torch.arange(n, dtype=torch.int32, device="cuda")
for _ in range(3):
    torch.sort(k, stable=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    s, idx = torch.sort(k, stable=True)
e1.record()
torch.cuda.synchronize()
print("torch.sort stable int32 keys (+int64 indices):", e0.elapsed_time(e1) / 20, "ms")
