"""Development check of the fused builder (psa_construct) on a GPU box.

Compares the device table with the oracle's exact fixed-point Vose
(ako_vose_fixed: the arithmetic the builder implements) on many inputs —
alias bit-exact, f64 thresholds bit-exact, f32 thresholds equal to the f32
rounding rule — then times the build at large N.

  python tools/check_build.py [--quick] [--time-n 1e9]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2106_12270_b200 as ak  # noqa: E402


def f32_rule(tw64: np.ndarray, avg: float) -> np.ndarray:
    f = tw64.astype(np.float32)
    cap = np.float32(avg)
    while float(cap) > avg:
        cap = np.nextafter(cap, np.float32(0))
    return np.where(f.astype(np.float64) > avg, cap, f)


def inputs(rng, quick):
    ns = [1, 2, 3, 7, 511, 512, 513, 1000, 4096, 8191, 100_000, 1_000_003]
    if not quick:
        ns += [3_000_017, 10_000_000]
    for n in ns:
        yield f"uniform{n}", rng.random(n) + 1e-12
        if n >= 100:
            yield f"zipf{n}", (1.0 / np.arange(1, n + 1))[rng.permutation(n)]
            yield f"pareto{n}", rng.pareto(1.1, n) + 1e-6
            yield f"ints{n}", rng.integers(1, 5, n).astype(np.float64)
            w = rng.random(n) + 0.5
            w[rng.integers(0, n)] = 1e6 * n  # one giant (wide excess)
            yield f"giant{n}", w
            w = rng.random(n)
            w[w < 0.3] = 1e-30  # tiny lights (rounded fixed-point values)
            yield f"tiny{n}", w + 1e-300
            yield f"sorted_up{n}", np.sort(rng.random(n) + 1e-9)
            yield f"sorted_dn{n}", np.sort(rng.random(n) + 1e-9)[::-1].copy()
            yield f"equal{n}", np.full(n, 0.3)


def check(name, w64, dtype):
    w = w64.astype(np.float32).astype(np.float64) if dtype == torch.float32 else w64
    ws = ak.make_weight_set(torch.from_numpy(w).to("cuda", dtype))
    t = ak.psa_construct(ws)
    tw, al = t.to_numpy()
    ref = O.vose_construct_fixed(w, ws.total)
    avg = ws.average
    bad_al = int((al != ref.alias).sum())
    want_tw = f32_rule(ref.tw, avg).astype(np.float64) if dtype == torch.float32 else ref.tw
    bad_tw = int((tw != want_tw).sum())
    ok = bad_al == 0 and bad_tw == 0
    if not ok:
        i = np.flatnonzero((al != ref.alias) | (tw != want_tw))[:5]
        print(f"FAIL {name} {dtype}: alias {bad_al} tw {bad_tw}; first {i.tolist()} "
              f"got {al[i].tolist()} {tw[i].tolist()} want {ref.alias[i].tolist()} {want_tw[i].tolist()}",
              flush=True)
    return ok


def timing(n, dtype, dist, reps=5):
    g = ak.gen_uniform if dist == "uniform" else (lambda n, r, dtype, device: ak.gen_power_law(n, 1.0, r, dtype=dtype, device=device))
    ws = g(n, ak.RngStream(seed=1), dtype=dtype, device="cuda")
    t = ak.psa_construct(ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ak.pack.build_table(ws, t)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    bw = 4 if dtype == torch.float32 else 8
    br = 8 if dtype == torch.float32 else 16
    ms = min(ts)
    gbs = n * (2 * bw + br) / ms / 1e6
    print(f"time {dist} n={n:.0e} {dtype}: {ms:.3f} ms (median {sorted(ts)[len(ts)//2]:.3f}) "
          f"{gbs:.0f} GB/s algorithmic = {gbs/6536:.3f} of 6536", flush=True)
    return t, ws


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--time-n", type=float, default=0)
    ap.add_argument("--no-check", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    rng = np.random.default_rng(2106)
    nfail = 0
    if not a.no_check:
        t0 = time.time()
        for name, w in inputs(rng, a.quick):
            for dt in (torch.float64, torch.float32):
                print(f"check {name} {dt} ...", end=" ", flush=True)
                ok = check(name, w, dt)
                print("ok" if ok else "FAIL", flush=True)
                nfail += not ok
        print(f"checks done in {time.time() - t0:.1f}s, failures {nfail}", flush=True)
    if a.time_n:
        n = int(a.time_n)
        for dt in (torch.float32, torch.float64):
            for dist in ("uniform", "powerlaw"):
                timing(n, dt, dist)
    return 1 if nfail else 0


if __name__ == "__main__":
    sys.exit(main())
