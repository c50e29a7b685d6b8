"""One warm and one profiled psa_plus_construct at N=1e9 f32 uniform, for ncu."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2106_12270_b200 as ak
ws = ak.gen_uniform(10**9, ak.RngStream(seed=1), dtype=torch.float32)
t = ak.psa_plus_construct(ws)
torch.cuda.synchronize()
t = ak.psa_plus_construct(ws)
torch.cuda.synchronize()
