"""partition_items on N (default 1e8) f32 weights, twice (for an ncu launch list)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
ws = ak.gen_uniform(n, ak.RngStream(seed=1), dtype=torch.float32)
for _ in range(2):
    p = ak.partition_items(ws)
torch.cuda.synchronize()
