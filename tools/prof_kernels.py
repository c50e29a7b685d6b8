"""Drive each hot kernel a few times for ncu (one process, one GPU).

    ncu --set full --clock-control none --import-source on \
        -k regex:'k_build|k_sample' -c 8 -o gpurun_out/prof python tools/prof_kernels.py

Workload: N (default 1e9) float32 uniform weights (gen_uniform seed 1), one
table build, one sectioned pass of ~1e9 draws (philox4x32 and reference RNG),
one naive pass of 1e8 draws.
"""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak  # noqa: E402
from paper_2106_12270_b200.sample import sectioned_sample_into  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=1e9)
ap.add_argument("--dist", default="uniform")
ap.add_argument("--dtype", default="float32")
ap.add_argument("--builds", type=int, default=2)
ap.add_argument("--draws", type=float, default=1e9)
a = ap.parse_args()
N = int(a.n)
dt = torch.float32 if a.dtype == "float32" else torch.float64
r = ak.RngStream(1)
ws = ak.gen_uniform(N, r, dtype=dt) if a.dist == "uniform" else ak.gen_power_law(N, 1.0, r, dtype=dt)
torch.cuda.synchronize()
t = None
for _ in range(a.builds):
    t = ak.psa_construct(ws)
torch.cuda.synchronize()
S = 1 << 14 if dt == torch.float32 else 1 << 13
M = int(a.draws)
asg = ak.assign_sections(N, S, M, 1, 7)
cd = torch.from_numpy(asg.counts).cuda()
od = torch.from_numpy(np.concatenate([[0], np.cumsum(asg.counts)[:-1]])).cuda()
out = torch.empty(M, dtype=torch.int64, device="cuda")
for mode in ("philox4x32", "reference"):
    sectioned_sample_into(t, asg.section_size, cd, od, 0, asg.n_sections, ak.RngStream(1, 7), out, 0, mode)
ak.sample_batch(t, min(M, 10**8), ak.RngStream(1, 8), out=out)
torch.cuda.synchronize()
print("done", N, M)
