"""One warm build then N profiled builds of psa_construct (for ncu).

  ncu --metrics gpu__time_duration.sum -k regex:k_b2 python tools/prof_build.py --n 1e9
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=1e9)
ap.add_argument("--dtype", default="float32")
ap.add_argument("--dist", default="uniform")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
dt = torch.float32 if a.dtype == "float32" else torch.float64
n = int(a.n)
if a.dist == "uniform":
    ws = ak.gen_uniform(n, ak.RngStream(seed=1), dtype=dt, device="cuda")
else:
    ws = ak.gen_power_law(n, 1.0, ak.RngStream(seed=1), dtype=dt, device="cuda")
t = ak.psa_construct(ws)
torch.cuda.synchronize()
for _ in range(a.reps):
    ak.pack.build_table(ws, t)
torch.cuda.synchronize()
print("done")
