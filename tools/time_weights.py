"""Time make_weight_set at N=1e9 (f32 and f64; CUDA events, median of 10).
AK_LIB_PATH picks the library."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak  # noqa: E402

for dt in (torch.float32, torch.float64):
    ws = ak.gen_uniform(10**9, ak.RngStream(seed=1), dtype=dt)
    for _ in range(3):
        t = ak.make_weight_set(ws.weights)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t = ak.make_weight_set(ws.weights)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"make_weight_set N=1e9 {str(dt)[6:]}: median {ts[5]:.3f} ms  total {t.total!r}")
    del ws, t
    torch.cuda.empty_cache()
