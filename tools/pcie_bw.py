"""Host<->device copy bandwidth on the box (pinned memory, CUDA events): H2D
alone, D2H alone, and both at once on two streams — the ceiling of bench.py's
e2e leg.  python tools/pcie_bw.py [--gb 8]"""
import argparse
import json
import time

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--gb", type=float, default=8.0)
a = ap.parse_args()
nb = int(a.gb * 1e9) // 8 * 8
h_in = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
h_out = torch.empty(nb // 8, dtype=torch.int64).pin_memory()
d_in = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
d_out = torch.empty(nb // 8, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if h2d:
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


t_h = run(True, False)
t_d = run(False, True)
t_b = run(True, True)
print(json.dumps({"bytes_each_way": nb, "h2d_GBps": nb / t_h / 1e9, "d2h_GBps": nb / t_d / 1e9,
                  "both_s": t_b, "both_aggregate_GBps": 2 * nb / t_b / 1e9,
                  "duplex_gain": (t_h + t_d) / t_b}))
