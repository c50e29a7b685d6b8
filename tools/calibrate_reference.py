"""Calibrate the reference arm: the reference package itself (numba, imported
from /root/reference — this container only) against the oracle's C port that
bench.py --impl reference runs, same inputs, same host, 8 workers.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tools/calibrate_reference.py
"""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
from aliaskit import make_weight_set, psa_construct, sample_batch, sectioned_sample, RngStream
N, M = 10**7, 10**7
r = np.random.default_rng(1)
w = r.random(N).astype(np.float32).astype(np.float64)
w[w == 0.0] = 0.5
ws = make_weight_set(w)
# warm numba
t = psa_construct(make_weight_set(w[:10000]), s=64, workers=8)
sample_batch(t, 1000, RngStream(1, 7), workers=8); sectioned_sample(t, 1 << 14, 1000, RngStream(1, 7))
res = {}
t0 = time.perf_counter(); t = psa_construct(ws, s=max(64, N // 65536), workers=8); res["ref_build_s"] = time.perf_counter() - t0
t0 = time.perf_counter(); sample_batch(t, M, RngStream(1, 7), workers=8); res["ref_naive_s"] = time.perf_counter() - t0
t0 = time.perf_counter(); sectioned_sample(t, 1 << 14, M, RngStream(1, 7)); res["ref_sectioned_s"] = time.perf_counter() - t0
_, tot = O.make_weight_set(w)
t0 = time.perf_counter(); to = O.psa_construct(w, tot, s=max(64, N // 65536), workers=8); res["port_build_s"] = time.perf_counter() - t0
t0 = time.perf_counter(); O.sample_batch(to, M, 1, 7, 0, workers=8); res["port_naive_s"] = time.perf_counter() - t0
t0 = time.perf_counter(); O.sectioned_sample(to, 1 << 14, M, 1, 7, 0); res["port_sectioned_s"] = time.perf_counter() - t0
for k, v in res.items(): print(f"{k:20s} {v:8.3f} s")
