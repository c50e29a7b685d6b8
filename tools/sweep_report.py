"""Throughput sweeps on one B200 beside the CPU reference path (oracle C port,
all host cores), for profiles/r2_sweeps.md:

  * PSA construction vs N (uniform / Zipf-1, f32 / f64), device-resident weights;
  * sectioned sampling vs section size S and vs N (philox4x32, f32 / f64 tables);
  * naive sampling vs N (philox4x32 and reference RNG);
  * the oracle's PSA construction and naive sampling on the same weights (N <= 1e8).

Device times: CUDA events, median of 5 after 2 warm-ups.  Algorithmic bytes as
in SURVEY.md §8d; peak = MEASURED_PEAKS.json hbm_gbs.

    python tools/sweep_report.py [--json out.json] [--no-cpu]
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2106_12270_b200 as ak  # noqa: E402
from paper_2106_12270_b200.pack import build_table  # noqa: E402
from paper_2106_12270_b200.sample import sectioned_sample_into  # noqa: E402

PEAK = 6453.4
if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")):
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]


def dev_time(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return statistics.median(ts)


def weights(n, dist, dt):
    r = ak.RngStream(seed=1)
    return ak.gen_uniform(n, r, dtype=dt) if dist == "uniform" else ak.gen_power_law(n, 1.0, r, dtype=dt)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json")
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    rows = []

    def emit(d):
        rows.append(d)
        print(json.dumps(d), flush=True)

    # construction vs N
    for dt in (torch.float32, torch.float64):
        bw = 4 if dt == torch.float32 else 8
        br = 8 if dt == torch.float32 else 16
        for dist in ("uniform", "zipf"):
            for n in (10**5, 10**6, 10**7, 10**8, 5 * 10**8, 10**9):
                ws = weights(n, dist, dt)
                t = ak.psa_construct(ws)
                s = dev_time(lambda: build_table(ws, t))
                by = n * (2 * bw + br)
                emit({"what": "psa_construct", "dtype": str(dt)[6:], "dist": dist, "n": n, "ms": s * 1e3,
                      "items_per_s": n / s, "gbs": by / s / 1e9, "frac": by / s / 1e9 / PEAK})
                del ws, t
                torch.cuda.empty_cache()
    # sectioned sampling vs S (N=1e9) and vs N (S=2^14): one pass of <= 2^30 draws
    def sectioned(n, S, dt, rng="philox4x32"):
        ws = weights(n, "uniform", dt)
        t = ak.psa_construct(ws)
        del ws
        # the bench's M = 1e11 at N = 1e9; smaller tables get M = 2^30 so the
        # first pass holds every section (1e11 would give one section > 2^30)
        M = 10**11 if n >= 10**9 else 1 << 30
        asg = ak.assign_sections(n, S, M, 1, 7)
        cnt = asg.counts
        k, tot = 0, 0
        while k < len(cnt) and tot + int(cnt[k]) <= (1 << 30):
            tot += int(cnt[k])
            k += 1
        cd = torch.from_numpy(cnt).cuda()
        od = torch.from_numpy(np.concatenate([[0], np.cumsum(cnt)[:-1]])).cuda()
        out = torch.empty(tot, dtype=torch.int64, device="cuda")
        r = ak.RngStream(1, 7)
        s = dev_time(lambda: sectioned_sample_into(t, asg.section_size, cd, od, 0, k, r, out, 0, rng, n_out=tot))
        br = 8 if dt == torch.float32 else 16
        by = tot * 8 + k * asg.section_size * br
        d = {"what": "sectioned", "rng": rng, "dtype": str(dt)[6:], "n": n, "S": asg.section_size,
             "draws": tot, "ms": s * 1e3, "samples_per_s": tot / s, "gbs": by / s / 1e9,
             "frac": by / s / 1e9 / PEAK}
        del t, out
        torch.cuda.empty_cache()
        return d
    for S in (1 << 10, 1 << 12, 1 << 13, 1 << 14, 1 << 15):
        emit(sectioned(10**9, S, torch.float32))
    for n in (10**6, 10**7, 10**8, 10**9):
        emit(sectioned(n, 1 << 14, torch.float32))
        emit(sectioned(n, 1 << 14, torch.float64))
    emit(sectioned(10**9, 1 << 14, torch.float32, "reference"))
    # naive sampling vs N
    for n in (10**5, 10**6, 10**7, 10**8, 10**9):
        ws = weights(n, "uniform", torch.float32)
        t = ak.psa_construct(ws)
        del ws
        m = 10**9
        out = torch.empty(m, dtype=torch.int64, device="cuda")
        for rng in ("philox4x32", "reference"):
            s = dev_time(lambda: ak.sample_batch(t, m, ak.RngStream(1, 8), rng=rng, out=out))
            by = m * (8 + 8)
            emit({"what": "naive", "rng": rng, "dtype": "float32", "n": n, "draws": m, "ms": s * 1e3,
                  "samples_per_s": m / s, "gbs": by / s / 1e9, "frac": by / s / 1e9 / PEAK})
        del t, out
        torch.cuda.empty_cache()
    # the CPU reference path on the same weights (oracle C port, all cores)
    if not a.no_cpu:
        import oracle as O
        thr = os.cpu_count() or 1
        for n in (10**5, 10**6, 10**7, 10**8):
            w = weights(n, "uniform", torch.float32).weights.double().cpu().numpy()
            _, tot = O.make_weight_set(w)
            t0 = time.perf_counter()
            tab = O.psa_construct(w, tot, s=max(64, n // 65536), workers=thr)
            tb = time.perf_counter() - t0
            m = min(10**8, 10 * n)
            t0 = time.perf_counter()
            O.sample_batch(tab, m, 1, 8, 0, workers=min(thr, 16))
            tn = time.perf_counter() - t0
            emit({"what": "cpu_reference", "n": n, "cores": thr, "build_items_per_s": n / tb,
                  "naive_samples_per_s": m / tn, "naive_draws": m})
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
