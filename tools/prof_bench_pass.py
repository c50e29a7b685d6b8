"""One build + one sectioned sampling pass in exactly the bench.py
configuration (N=1e9 f32 gen_uniform table, M=1e11 draws, S=2^14,
RngStream(1, 7), rng=philox4x32, first pass of <= 2^30 draws), for ncu:

    ncu --set full --clock-control none --import-source on \
        -k regex:'k_build|k_sample_sectioned' -o gpurun_out/prof python tools/prof_bench_pass.py
Prints the pass's draw count and section count (the per-launch units)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak  # noqa: E402
from paper_2106_12270_b200.sample import sectioned_sample_into  # noqa: E402

N, M, S = 10**9, 10**11, 1 << 14
ws = ak.gen_uniform(N, ak.RngStream(seed=1), dtype=torch.float32)
t = ak.psa_construct(ws)
asg = ak.assign_sections(N, S, M, 1, 7)
cd = torch.from_numpy(asg.counts).cuda()
offs = np.concatenate([[0], np.cumsum(asg.counts)[:-1]])
od = torch.from_numpy(offs).cuda()
cap = 1 << 30
out = torch.empty(cap, dtype=torch.int64, device="cuda")
k, tot = 0, 0
while k < asg.n_sections and tot + int(asg.counts[k]) <= cap:
    tot += int(asg.counts[k])
    k += 1
sectioned_sample_into(t, asg.section_size, cd, od, 0, k, ak.RngStream(1, 7), out, 0, "philox4x32")
torch.cuda.synchronize()
print(f"pass: sections {k} draws {tot} table bytes {k * S * 8}")
