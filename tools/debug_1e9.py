"""Worst heavy-threshold gaps between the device table and the oracle's PSA
at N=1e9 (f32 or f64 uniform, gen_uniform seed 1), with the binary128 Vose
as the arbiter.  python tools/debug_1e9.py [f32|f64] [n]"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_2106_12270_b200 as ak
dt = torch.float32 if (len(sys.argv) < 2 or sys.argv[1] == "f32") else torch.float64
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**9
ws = ak.gen_uniform(n, ak.RngStream(seed=1), dtype=dt)
t = ak.psa_construct(ws)
tw, al = t.to_numpy()
w64 = ws.weights.double().cpu().numpy()
avg = ws.total / n
t0 = time.time()
ref = O.psa_construct(w64, ws.total, s=n // 1024, workers=os.cpu_count())
print("psa oracle", time.time() - t0, flush=True)
light = w64 <= avg
d = np.abs(tw - ref.tw) / avg
d[light] = 0
worst = np.argsort(d)[-8:][::-1]
print("alias flips", int((al != ref.alias).sum()))
print("rows > 1e-6:", int((d > 1e-6).sum()), "first:", np.flatnonzero(d > 1e-6)[:10])
t0 = time.time()
q = O.vose_construct_quad(w64, ws.total)
print("quad", time.time() - t0, flush=True)
for i in worst:
    print(i, "w", w64[i], "dev", tw[i], "psa", ref.tw[i], "quad", q.tw[i], "al", al[i], ref.alias[i], q.alias[i])
dq = np.abs(tw - q.tw) / avg; dq[light] = 0
dp = np.abs(ref.tw - q.tw) / avg; dp[light] = 0
print("dev vs quad max", dq.max(), "psa vs quad max", dp.max(), "alias dev!=quad", int((al != q.alias).sum()), "psa!=quad", int((ref.alias != q.alias).sum()))
