"""Time psa_construct (CUDA events, device-resident weights) at one size.

    python tools/time_build.py [--n 1e9] [--dist uniform|zipf] [--alpha 1.0] [--dtype float32|float64] [--reps 10]
                               [--method psa|psa_plus]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak  # noqa: E402
from paper_2106_12270_b200.pack import build_table  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=1e9)
ap.add_argument("--dist", default="uniform")
ap.add_argument("--dtype", default="float32")
ap.add_argument("--alpha", type=float, default=1.0, help="power-law exponent for --dist zipf")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--method", default="psa")
a = ap.parse_args()
N = int(a.n)
dt = torch.float32 if a.dtype == "float32" else torch.float64
r = ak.RngStream(1)
ws = ak.gen_uniform(N, r, dtype=dt) if a.dist == "uniform" else ak.gen_power_law(N, a.alpha, r, dtype=dt)
t = build_table(ws)
if a.method == "psa_plus":
    def build_table(ws, t):  # noqa: F811
        return ak.psa_plus_construct(ws)
for _ in range(3):
    build_table(ws, t)
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    build_table(ws, t)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
b = 4 if dt == torch.float32 else 8
byts = N * (2 * b + 2 * b)  # read w twice + write the row (8 B f32 / 16 B f64)
med = ts[len(ts) // 2]
dist = a.dist if a.dist == "uniform" else f"{a.dist}(alpha={a.alpha:g})"
print(f"{a.method} N={N:.0e} {dist} {a.dtype}: median {med:.3f} ms  min {ts[0]:.3f} ms  "
      f"{N / med / 1e6:.1f} G items/s  {byts / med / 1e6:.0f} GB/s algorithmic")
