"""One warm and one profiled psa_plus_construct at N=1e9 f32, for ncu.

    python tools/prof_psa_plus.py [uniform | zipf ALPHA]
Prints the handled fraction (the share of items the prepack pairs)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2106_12270_b200 as ak
from paper_2106_12270_b200.prepack import _prepack
r = ak.RngStream(seed=1)
if len(sys.argv) > 1 and sys.argv[1] == "zipf":
    ws = ak.gen_power_law(10**9, float(sys.argv[2]), r, dtype=torch.float32)
else:
    ws = ak.gen_uniform(10**9, r, dtype=torch.float32)
t = ak.psa_plus_construct(ws)
torch.cuda.synchronize()
t = ak.psa_plus_construct(ws)
torch.cuda.synchronize()
_, res_idx, _, nwritten = _prepack(ws, 4096, 8)
print(f"handled fraction {nwritten / ws.n:.4f}  residual {res_idx.numel()}")
