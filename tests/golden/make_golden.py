"""Generate the golden fixtures from the reference itself.

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/golden.npz (reference outputs on seeded inputs) and
tests/golden/hand_vectors.json (the reference tests' hand vectors and the
Random123 Philox2x64-10 known-answer vectors).  The GPU box has no
/root/reference, so these committed files are what the oracle and the CUDA
path are pinned against there.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

ref_src = os.environ.get("ALIASKIT_REF", "/root/reference/pkg/src")
sys.path.insert(0, ref_src)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import aliaskit as A  # noqa: E402
from aliaskit import rng as R  # noqa: E402
from aliaskit import sample as SM  # noqa: E402
from aliaskit import split as SP  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def weights(rng, n, kind):
    if kind == 0:
        return rng.random(n) + 1e-9
    if kind == 1:
        return rng.pareto(1.1, n) + 1e-6
    if kind == 2:
        return np.exp(rng.normal(0.0, 3.0, n))
    if kind == 3:
        return rng.integers(1, 6, n).astype(np.float64)
    w = np.arange(1, n + 1, dtype=np.float64) ** -1.0
    rng.shuffle(w)
    return w


def main():
    rng = np.random.default_rng(0x601DE7)
    out = {}
    sizes = [1, 2, 3, 4, 17, 64, 100, 257, 1000, 1999, 2048, 4097]
    cases = []
    for ci, n in enumerate(sizes):
        kind = ci % 5
        w = weights(rng, n, kind)
        ws = A.make_weight_set(w)
        key = f"c{ci}_"
        out[key + "weights"] = ws.weights
        out[key + "total"] = np.array([ws.total])
        v = A.vose_construct(ws)
        out[key + "vose_tw"] = v.tw
        out[key + "vose_alias"] = v.alias
        p = A.partition_items(ws)
        for f in ("l_index", "l_weight", "h_index", "h_weight", "lprefix", "hprefix"):
            out[key + f] = getattr(p, f)
        for s in (1, 2, 7, 64):
            if s > n:
                continue
            plan = A.compute_split_plan(p, s)
            out[key + f"plan{s}_l"] = plan.lcounts
            out[key + f"plan{s}_h"] = plan.hcounts
            out[key + f"plan{s}_sp"] = plan.spills
            t = A.psa_construct(ws, s=s, workers=1)
            out[key + f"psa{s}_tw"] = t.tw
            out[key + f"psa{s}_alias"] = t.alias
        seed = int(rng.integers(2**63))
        out[key + "seed"] = np.array([seed], dtype=np.uint64)
        out[key + "naive"] = A.sample_batch(v, 2000, A.RngStream(seed, 3, 11))
        out[key + "sectioned16"] = A.sectioned_sample(v, 16, 3000, A.RngStream(seed, 5, 7))
        pre = A.greedy_prepack(ws, block_size=64, min_pair_threshold=4)
        out[key + "pre_tw"] = pre.tw
        out[key + "pre_alias"] = pre.alias
        out[key + "pre_res_l"] = pre.residual.l_index
        out[key + "pre_res_h"] = pre.residual.h_index
        out[key + "pre_res_hw"] = pre.residual.h_weight
        out[key + "pre_handled"] = np.array([pre.handled_fraction])
        rep = A.validate_table(v, ws)
        out[key + "vose_valid"] = np.array([rep.worst_rel_error, rep.worst_item, float(rep.ok)])
        cases.append(n)
    out["sizes"] = np.array(sizes)
    # uniform streams, including the 2^64 counter wrap
    out["ub_a"] = A.rng.uniform_block(A.RngStream(20260815, 0, 0), 1000)
    out["ub_b"] = A.rng.uniform_block(A.RngStream(7, 3, (1 << 64) - 5), 16)
    # section assignments (deep trees, both binomial branches)
    asg = []
    for (nr, S, M, seed, st) in [(10**6, 2**14, 10**9, 5, 0), (12345, 7, 999, 77, 4),
                                 (2**20, 2**14, 80, 11, 0), (10**9, 2**14, 10**11, 1, 7),
                                 (100, 10, 0, 3, 0), (7, 99, 1234, 3, 0)]:
        c = A.assign_sections(nr, S, M, seed, stream=st).counts
        out[f"asg_{len(asg)}"] = c
        asg.append([nr, S, M, seed, st])
    out["asg_params"] = np.array(asg, dtype=np.float64)
    # partial p-ary search
    hay = np.sort(rng.normal(0, 10, 5000))
    q = np.sort(rng.normal(0, 12, 300))
    out["pary_hay"] = hay
    out["pary_q"] = q
    for pp in (3, 8, 32):
        out[f"pary_{pp}"] = A.partial_pary_search(hay, q, p=pp)
        out[f"pary_contract_{pp}"] = np.array(SP._contract_range(hay, float(q[0]), float(q[-1]), pp))
    # binomial draws on both branches
    bd = []
    for m, qq, u in [(3, 0.5, 0.1), (3, 0.5, 0.2), (3, 0.5, 0.6), (3, 0.5, 0.9), (99, 0.3, 0.5),
                     (100, 0.3, 0.5), (10**6, 0.25, 1e-5), (10**9, 0.5, 0.99999),
                     (10**11, 0.4999, 0.02), (57, 0.999, 0.001)]:
        bd.append([m, qq, u, SM._binom_draw(m, qq, u)])
    out["binom"] = np.array(bd, dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)

    def hexw(x):
        return f"{x:016x}"

    kat = []
    for ctr, key in [((0, 0), 0), (((1 << 64) - 1, (1 << 64) - 1), (1 << 64) - 1),
                     ((0x243F6A8885A308D3, 0x13198A2E03707344), 0xA4093822299F31D0)]:
        kat.append({"ctr": [hexw(ctr[0]), hexw(ctr[1])], "key": hexw(key),
                    "w0": hexw(R._philox_py(ctr[0], ctr[1], key))})
    hv = {
        "philox2x64_10_kat": kat,
        "philox2x64_10_kat_w1_random123": ["66c24222c9a845b5", "4d02f3222f86df20", "b0f883d38000de5d"],
        "uniform_py_0_0_0": R.uniform_py(0, 0, 0),
        "table4": {"w": [3.0, 1.0, 2.0, 2.0], "tw": [2.0, 1.0, 2.0, 2.0], "alias": [1, 1, 3, 4]},
        "single": {"w": [5.0], "tw": [5.0], "alias": [1]},
        "two": {"w": [3.0, 1.0], "tw": [2.0, 1.0], "alias": [1, 1]},
        "all_equal": {"w": [1.0, 1.0, 1.0, 1.0], "alias": [1, 2, 3, 4]},
        "partition4": {"l": [[2, 1.0], [3, 2.0], [4, 2.0]], "h": [[1, 3.0]],
                       "lprefix": [0.0, 1.0, 3.0, 5.0], "hprefix": [0.0, 3.0]},
        "plan4_s2": [[0, 0, 0.0], [1, 1, 0.0], [3, 1, 0.0]],
        "plan_equal12_s4_l": [0, 3, 6, 9, 12],
        "rule4": [[0.3, 2], [0.4, 1], [0.0, 1], [0.999999, 4]],
        "pary_hand": {"hay": [1, 3, 5, 7, 9, 11, 13, 15], "q": [4, 10], "p": 4, "out": [2, 5]},
        "pary_ties": {"hay": [1.0, 2.0, 2.0, 2.0, 3.0], "q": [2.5, 3.0, 99.0], "out": [4, 4, 5]},
        "binom_steps": [[3, 0.5, 0.1, 0], [3, 0.5, 0.2, 1], [3, 0.5, 0.6, 2], [3, 0.5, 0.9, 3]],
    }
    with open(os.path.join(HERE, "hand_vectors.json"), "w") as f:
        json.dump(hv, f, indent=1)
    print("wrote", sorted(out)[:5], "...", len(out), "arrays")


if __name__ == "__main__":
    main()
