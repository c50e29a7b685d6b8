"""Per-stage device timeline of bench.py's e2e pipeline (one GPU): copy-in,
compute (make_weight_set -> psa_construct -> sectioned_sample) and copy-out
of each step, from CUDA events, to see what bounds the end-to-end rate.
    python tools/e2e_timeline.py [--out-dtype int32|int64] [--samples 2e9]"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12270_b200 as ak  # noqa: E402
from paper_2106_12270_b200.sample import sectioned_sample_into  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out-dtype", default="int64")
ap.add_argument("--samples", type=float, default=2e9)
ap.add_argument("--steps", type=int, default=4)
a = ap.parse_args()
N, S = 10**9, 1 << 14
Me, K = int(a.samples), a.steps
odt = getattr(torch, a.out_dtype)
dev = torch.device("cuda", 0)
ws = ak.gen_uniform(N, ak.RngStream(seed=1), dtype=torch.float32, device=dev)
w_host = ws.weights.cpu().pin_memory()
o_host = [torch.empty(Me, dtype=odt).pin_memory() for _ in range(2)]
wd = [torch.empty_like(ws.weights) for _ in range(2)]
od = [torch.empty(Me, dtype=odt, device=dev) for _ in range(2)]
s_in, s_cmp, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
E = lambda: torch.cuda.Event(enable_timing=True)
ev = {k: [E() for _ in range(K + 1)] for k in ("in0", "in1", "c0", "c1", "o0", "o1")}
host = {}


def copy_in(i):
    with torch.cuda.stream(s_in):
        if i >= 2:
            s_in.wait_event(ev["c1"][i - 2])
        ev["in0"][i].record(s_in)
        wd[i % 2].copy_(w_host, non_blocking=True)
        ev["in1"][i].record(s_in)


def compute(i):
    with torch.cuda.stream(s_cmp):
        s_cmp.wait_event(ev["in1"][i])
        if i >= 2:
            s_cmp.wait_event(ev["o1"][i - 2])
        ev["c0"][i].record(s_cmp)
        t0 = time.perf_counter()
        wse = ak.make_weight_set(wd[i % 2])
        t1 = time.perf_counter()
        te = ak.psa_construct(wse)
        asg = ak.assign_sections(N, S, Me, 1, 7 + i)
        t2 = time.perf_counter()
        cd = torch.from_numpy(asg.counts).to(dev, non_blocking=True)
        odf = torch.from_numpy(np.concatenate([[0], np.cumsum(asg.counts)[:-1]])).to(dev, non_blocking=True)
        sectioned_sample_into(te, asg.section_size, cd, odf, 0, asg.n_sections, ak.RngStream(1, 7 + i),
                              od[i % 2], 0, "philox4x32", n_out=Me)
        ev["c1"][i].record(s_cmp)
        host[i] = (t1 - t0, t2 - t1, time.perf_counter() - t2)


def copy_out(i):
    with torch.cuda.stream(s_out):
        s_out.wait_event(ev["c1"][i])
        ev["o0"][i].record(s_out)
        o_host[i % 2].copy_(od[i % 2], non_blocking=True)
        ev["o1"][i].record(s_out)


copy_in(0)
compute(0)
copy_out(0)
torch.cuda.synchronize()
w0 = time.perf_counter()
copy_in(1)
for i in range(1, K + 1):
    if i + 1 <= K:
        copy_in(i + 1)
    compute(i)
    copy_out(i)
torch.cuda.synchronize()
wall = time.perf_counter() - w0
print(f"{a.out_dtype} Me={Me:.0e}: wall {wall:.3f} s for {K} steps = {Me * K / wall:.3e} samples/s")
base = ev["in0"][1]
for i in range(1, K + 1):
    f = lambda e: base.elapsed_time(e) / 1e3
    print(f"step {i}: in [{f(ev['in0'][i]):.3f},{f(ev['in1'][i]):.3f}]  cmp [{f(ev['c0'][i]):.3f},{f(ev['c1'][i]):.3f}]  "
          f"out [{f(ev['o0'][i]):.3f},{f(ev['o1'][i]):.3f}]  host mws {host[i][0]*1e3:.1f} ms, build+assign {host[i][1]*1e3:.1f} ms, rest {host[i][2]*1e3:.1f} ms")
