"""Debug aid: rows of psa_construct that differ from the binary128 Vose, with
their exact (long double) keys and the nearest keys of the other class."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2106_12270_b200 as ak  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
dist = sys.argv[2] if len(sys.argv) > 2 else "uniform"
r = ak.RngStream(seed=1)
ws = ak.gen_uniform(n, r, dtype=torch.float32) if dist == "uniform" else ak.gen_power_law(n, 1.0, r, dtype=torch.float32)
t = ak.psa_construct(ws)
w = ws.weights.double().cpu().numpy()
tw, al = t.to_numpy()
q = O.vose_construct_quad(w, ws.total)
bad = np.nonzero(al != q.alias)[0]
print("differing rows:", bad.size, bad[:10])
avg = ws.total / n
light = w <= avg
L = np.nonzero(light)[0]
H = np.nonzero(~light)[0]
dl = np.concatenate([[0], np.cumsum((avg - w[L]).astype(np.longdouble))])[:-1]
dh = np.cumsum((w[H] - avg).astype(np.longdouble))
for i in bad[:5]:
    print(f"item {i} ({'light' if light[i] else 'heavy'}) tile {i // 2048} chunk {(i % 2048) // 256} lane {(i % 256) // 8} q {i % 8}")
    print(f"   ours alias {al[i]} tw {tw[i]!r}   quad alias {q.alias[i]} tw {q.tw[i]!r}")
    if light[i]:
        k = np.searchsorted(L, i)
        key = dl[k]
        j = np.searchsorted(dh, key, side="right")
        print(f"   light rank {k} key/avg {float(key / avg)!r}; heavies around: ranks {j - 1},{j} keys/avg "
              f"{float(dh[j - 1] / avg)!r} {float(dh[j] / avg) if j < dh.size else None!r} items {H[j - 1]} {H[j] if j < H.size else None}")
        print(f"   margin/avg {float(min(abs(dh[j - 1] - key), abs(dh[j] - key) if j < dh.size else 1e9) / avg)!r}")
    else:
        j = np.searchsorted(H, i)
        key = dh[j]
        k = np.searchsorted(dl, key, side="left")
        print(f"   heavy rank {j} key/avg {float(key / avg)!r}; lights around ranks {k - 1},{k} keys/avg "
              f"{float(dl[k - 1] / avg)!r} {float(dl[k] / avg) if k < dl.size else None!r}")

import math
for i in bad[:2]:
    if not light[i]:
        continue
    k = int(np.searchsorted(L, i))
    DLk = math.fsum(np.concatenate([np.full(k, avg), -w[L[:k]]]).tolist())
    j = int(np.searchsorted(dh, dl[k], side="right"))
    for jj in (j - 2, j - 1, j):
        DHj = math.fsum(np.concatenate([w[H[: jj + 1]], np.full(jj + 1, -avg)]).tolist())
        m = math.fsum(np.concatenate([w[H[: jj + 1]], np.full(jj + 1 + k, -avg), w[L[:k]]]).tolist())
        print(f"   exact: DL(k)={DLk / avg!r} DH({jj})={DHj / avg!r} margin DH-DL (one rounding)/avg={m / avg!r} item {H[jj]}")
    print("   f64 reference alias:", O.vose_construct(w, ws.total).alias[i])
