"""Time naive sampling (sample_batch) on a device table: C2 = N=1e8 f32
uniform table, 1e9 draws, both RNG modes (CUDA events)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=1e8)
ap.add_argument("--m", type=float, default=1e9)
a = ap.parse_args()
N, M = int(a.n), int(a.m)
ws = ak.gen_uniform(N, ak.RngStream(1), dtype=torch.float32)
t = ak.psa_construct(ws)
out = torch.empty(M, dtype=torch.int64, device="cuda")
for mode in ("philox4x32", "reference"):
    for _ in range(2):
        ak.sample_batch(t, M, ak.RngStream(1, 7), rng=mode, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    ak.sample_batch(t, M, ak.RngStream(1, 7), rng=mode, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"naive N={N:.0e} M={M:.0e} {mode}: {ms:.3f} ms  {M / ms / 1e6:.1f} G draws/s  "
          f"{M * 16 / ms / 1e6:.0f} GB/s algorithmic (16 B/draw)")
