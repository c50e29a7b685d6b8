"""make_weight_set at N=1e9 (f32 or f64) for ncu: one warm call, one profiled.

    ncu -k regex:k_pairwise_leaves -s 1 -c 1 python tools/prof_weights.py float32"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak  # noqa: E402

dt = torch.float32 if (len(sys.argv) < 2 or sys.argv[1] == "float32") else torch.float64
ws = ak.gen_uniform(10**9, ak.RngStream(seed=1), dtype=dt)
for _ in range(2):
    ak.make_weight_set(ws.weights)
torch.cuda.synchronize()
