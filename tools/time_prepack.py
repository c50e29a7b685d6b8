"""Time the prepack pass alone (ak_greedy_prepack_ex with clear_rows=False, as
psa_plus_construct calls it) at N=1e9 f32.  AK_LIB_PATH picks the library.

    python tools/time_prepack.py [--dist uniform|zipf] [--alpha 0.5] [--dtype float32|float64]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak  # noqa: E402
from paper_2106_12270_b200.prepack import _prepack  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=1e9)
ap.add_argument("--dist", default="uniform")
ap.add_argument("--alpha", type=float, default=0.5)
ap.add_argument("--dtype", default="float32")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
N = int(a.n)
dt = torch.float32 if a.dtype == "float32" else torch.float64
r = ak.RngStream(1)
ws = ak.gen_uniform(N, r, dtype=dt) if a.dist == "uniform" else ak.gen_power_law(N, a.alpha, r, dtype=dt)
for _ in range(3):
    out = _prepack(ws, 4096, 8, clear_rows=False)
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = _prepack(ws, 4096, 8, clear_rows=False)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"prepack N={N:.0e} {a.dist} {a.dtype}: median {ts[len(ts) // 2]:.3f} ms  min {ts[0]:.3f} ms  "
      f"residual {out[1].numel()}  written {out[3]}")
