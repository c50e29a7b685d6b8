"""Build one table (device-resident weights) and check it against the oracle's
sequential Vose; for compute-sanitizer / launch-blocking debugging.

    python tools/debug_build.py --n 1e6 --dist zipf --dtype float32
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2106_12270_b200 as ak  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=1e6)
ap.add_argument("--dist", default="zipf")
ap.add_argument("--dtype", default="float32")
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--check", type=int, default=1)
a = ap.parse_args()
N = int(a.n)
dt = torch.float32 if a.dtype == "float32" else torch.float64
r = ak.RngStream(a.seed)
ws = ak.gen_uniform(N, r, dtype=dt) if a.dist == "uniform" else ak.gen_power_law(N, 1.0, r, dtype=dt)
t = ak.psa_construct(ws)
torch.cuda.synchronize()
print("built", flush=True)
if a.check:
    w64 = ws.weights.double().cpu().numpy()
    q = O.vose_construct_quad(w64, ws.total)
    tw, al = t.to_numpy()
    bad = np.flatnonzero(al != q.alias)
    print(f"N={N} {a.dist} {a.dtype}: alias mismatches vs binary128 Vose: {bad.size}", bad[:10])
    print(ak.validate_table(t, ws, tol=1e-4 if dt == torch.float32 else 1e-9))
