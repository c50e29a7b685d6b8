"""Quick end-to-end exercise of every device entry point against the oracle.

Development aid (the formal parity suite is tests/); prints one line per
check and a summary.  Run on a GPU box:  python tools/gpu_quick.py
"""

import os
import sys
import time
import traceback

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2106_12270_b200 as ak  # noqa: E402

results = []


def check(name, fn):
    t0 = time.time()
    try:
        msg = fn()
        results.append((name, True))
        print(f"PASS {name} ({time.time() - t0:.2f}s) {msg or ''}", flush=True)
    except Exception:
        results.append((name, False))
        print(f"FAIL {name}\n{traceback.format_exc()}", flush=True)


rng = np.random.default_rng(7)


def weights(n, kind):
    if kind == 0:
        return rng.random(n) + 1e-9
    if kind == 1:
        return rng.pareto(1.1, n) + 1e-6
    if kind == 2:
        return np.exp(rng.normal(0, 3, n))
    if kind == 3:
        return rng.integers(1, 6, n).astype(np.float64)
    w = np.arange(1, n + 1, dtype=np.float64) ** -1.0
    rng.shuffle(w)
    return w


def t_uniform():
    r = ak.RngStream(seed=123, stream=5, counter=(1 << 64) - 3)
    u = ak.uniform_block(r, 1000).cpu().numpy()
    want = O.uniform_block(123, 5, (1 << 64) - 3, 1000)
    assert np.array_equal(u, want)
    assert r.counter == (1 << 64) - 3 + 1000


def t_total():
    bad = 0
    for n in (1, 7, 8, 9, 127, 128, 129, 1000, 4097, 100_003, 3_000_001):
        w = weights(n, n % 5)
        ws = ak.make_weight_set(w)
        if ws.total != float(np.sum(w)):
            bad += 1
        ws32 = ak.make_weight_set(torch.tensor(w, dtype=torch.float32, device="cuda"))
        if ws32.total != float(np.sum(w.astype(np.float32).astype(np.float64))):
            bad += 1
    assert bad == 0, bad
    try:
        ak.make_weight_set([1.0, 0.0, 2.0])
        raise AssertionError("no raise")
    except ak.InvalidWeight as e:
        assert e.index == 2


def table_cmp(t, ref_tw, ref_alias, avg, tol):
    tw, al = t.to_numpy()
    am = int(np.count_nonzero(al != ref_alias))
    gap = float(np.max(np.abs(tw - ref_tw))) / avg if tw.size else 0.0
    return am, gap


def t_build():
    worst = 0.0
    bad = 0
    for trial in range(60):
        n = int(np.exp(rng.uniform(0, np.log(300_000)))) + 1
        w = weights(n, trial % 5)
        ws = ak.make_weight_set(w)
        ref = O.vose_construct(w, ws.total)
        t = ak.psa_construct(ws)
        am, gap = table_cmp(t, ref.tw, ref.alias, ws.average, 1e-9)
        worst = max(worst, gap)
        if am or gap > 1e-9:
            bad += 1
            print(f"   build mismatch n={n} kind={trial % 5} alias_mismatch={am} gap={gap:.3e}")
    for w in ([3.0, 1.0, 2.0, 2.0], [5.0], [1.0] * 4, [3.0, 1.0], [2.0000000001, 1.9999999999] * 50):
        ws = ak.make_weight_set(w)
        ref = O.vose_construct(w, ws.total)
        t = ak.psa_construct(ws)
        am, gap = table_cmp(t, ref.tw, ref.alias, ws.average, 1e-9)
        if am or gap > 1e-9:
            bad += 1
            print("   hand mismatch", w[:4], t.to_numpy(), ref.tw, ref.alias)
    assert bad == 0
    return f"worst gap {worst:.2e}"


def t_build_f32():
    bad = 0
    for trial in range(20):
        n = int(np.exp(rng.uniform(0, np.log(500_000)))) + 1
        w = weights(n, trial % 5).astype(np.float32)
        ws = ak.make_weight_set(torch.from_numpy(w).cuda())
        w64 = w.astype(np.float64)
        ref = O.vose_construct(w64, ws.total)
        t = ak.psa_construct(ws)
        am, gap = table_cmp(t, ref.tw, ref.alias, ws.average, 1e-6)
        rep = ak.validate_table(t, ws, tol=1e-4)
        if am or not rep.ok:
            bad += 1
            print(f"   f32 n={n} am={am} gap={gap:.2e} rep={rep}")
    assert bad == 0


def t_partition_plan_pack():
    bad = 0
    for trial in range(30):
        n = int(np.exp(rng.uniform(np.log(2), np.log(20000))))
        w = weights(n, trial % 5)
        ws = ak.make_weight_set(w)
        p = ak.partition_items(ws)
        po = O.partition_items(w, ws.total)
        if not (np.array_equal(p.l_index.cpu().numpy(), po["l_index"]) and
                np.array_equal(p.h_index.cpu().numpy(), po["h_index"])):
            bad += 1
            print("   partition idx mismatch", n)
        lp = p.lprefix.cpu().numpy()
        d = np.abs(lp - po["lprefix"])
        ulp = np.spacing(np.maximum(np.abs(po["lprefix"]), 1e-300))
        if np.any(d > 4 * ulp):
            bad += 1
            print("   lprefix off", n, float(np.max(d / ulp)))
        # plan on the reference's own prefix arrays: bit-exact
        ref_lp = torch.from_numpy(po["lprefix"]).cuda()
        ref_hp = torch.from_numpy(po["hprefix"]).cuda()
        p2 = ak.LightHeavyPartition(
            torch.from_numpy(po["l_index"]).cuda(), torch.from_numpy(po["l_weight"]).cuda(),
            torch.from_numpy(po["h_index"]).cuda(), torch.from_numpy(po["h_weight"]).cuda(),
            ref_lp, ref_hp, po["avg"])
        for s in (1, 2, 7, 64, 1000):
            if s > n:
                continue
            lc, hc, sp = O.compute_split_plan(po["lprefix"], po["hprefix"], po["h_weight"], n, s,
                                              po["avg"])
            for method in ("binary", "batched"):
                plan = ak.compute_split_plan(p2, s, method=method)
                if not (np.array_equal(plan.lcounts.cpu().numpy(), lc) and
                        np.array_equal(plan.hcounts.cpu().numpy(), hc) and
                        np.array_equal(plan.spills.cpu().numpy(), sp)):
                    bad += 1
                    print(f"   plan mismatch n={n} s={s} {method}")
            # pack all sections with the reference plan: bit-exact table
            plan = ak.compute_split_plan(p2, s, method="binary")
            for cap in (0, 2, 64):
                out = ak.AliasTable.blank(n, ws.total)
                ak.pack.pack_all(p2, plan, out, cap)
                tw, al = out.to_numpy()
                tw_o = np.zeros(n)
                al_o = np.zeros(n, dtype=np.int64)
                O.pack_sections(po, lc, hc, sp, 1, s, tw_o, al_o, cap)
                if not (np.array_equal(tw, tw_o) and np.array_equal(al, al_o)):
                    bad += 1
                    print(f"   pack mismatch n={n} s={s} cap={cap}")
    assert bad == 0, bad


def t_pary():
    bad = 0
    for _ in range(200):
        n = int(rng.integers(0, 4000))
        hay = np.sort(rng.normal(0, 10, n))
        q = np.sort(rng.normal(0, 12, int(rng.integers(0, 80))))
        for p in (3, 8, 32, 33, 100):
            got = ak.partial_pary_search(hay, q, p=p).cpu().numpy()
            if not np.array_equal(got, np.searchsorted(hay, q, side="left")):
                bad += 1
    assert bad == 0, bad
    try:
        ak.partial_pary_search([3.0, 1.0], [1.0])
        raise AssertionError("no raise")
    except ak.UnsortedInput:
        pass


def t_sample():
    bad = 0
    for trial in range(20):
        n = int(np.exp(rng.uniform(0, np.log(100_000)))) + 1
        w = weights(n, trial % 5)
        ws = ak.make_weight_set(w)
        ref = O.vose_construct(w, ws.total)
        t = ak.AliasTable.from_numpy(ref.tw, ref.alias, n, ws.total)
        seed = int(rng.integers(2**63))
        got = ak.sample_batch(t, 20000, ak.RngStream(seed, 3, 17)).cpu().numpy()
        want = O.sample_batch(ref, 20000, seed, 3, 17)
        if not np.array_equal(got, want):
            bad += 1
            print("   naive mismatch", n)
        for S in (1, 7, 64, 1 << 14, 10**9):
            got = ak.sectioned_sample(t, S, 30000, ak.RngStream(seed, 9, 5)).cpu().numpy()
            want = O.sectioned_sample(ref, S, 30000, seed, 9, 5)
            if not np.array_equal(got, want):
                bad += 1
                print("   sectioned mismatch", n, S)
        # f32 table vs rule on upcast table
        t32 = ak.AliasTable.from_numpy(ref.tw, ref.alias, n, ws.total, dtype=torch.float32)
        tw32, al32 = t32.to_numpy()
        u = O.uniform_block(seed, 4, 0, 5000)
        got = ak.sample_from_uniforms(t32, u).cpu().numpy()
        want = O.rule(tw32, al32, ws.average, u)
        if not np.array_equal(got, want):
            bad += 1
            print("   f32 rule mismatch", n)
        got = ak.sample_batch(t32, 5000, ak.RngStream(seed, 4, 0)).cpu().numpy()
        if not np.array_equal(got, want):
            bad += 1
            print("   f32 naive mismatch", n)
    assert bad == 0, bad


def t_assign():
    bad = 0
    for _ in range(300):
        n = int(rng.integers(1, 2_000_000))
        S = int(rng.integers(1, n + 10))
        M = int(rng.integers(0, 10**9))
        seed = int(rng.integers(2**63))
        a = ak.assign_sections(n, S, M, seed, stream=3).counts
        b = O.assign_sections(n, S, M, seed, 3)
        if not np.array_equal(a, b):
            bad += 1
    assert bad == 0


def t_fast_rng_chi2():
    n = 1000
    w = rng.random(n) + 1e-9
    ws = ak.make_weight_set(w)
    t = ak.psa_construct(ws)
    probs = w / w.sum()
    fails = 0
    for seed in range(10):
        x = ak.sample_batch(t, 10**7, ak.RngStream(seed, 1), rng="philox4x32")
        _, _, ok = ak.chi_square_test(ak.frequency_counts(x, n), probs)
        fails += not ok
        x = ak.sectioned_sample(t, 64, 10**7, ak.RngStream(seed, 2), rng="philox4x32")
        _, _, ok = ak.chi_square_test(ak.frequency_counts(x, n), probs)
        fails += not ok
    assert fails <= 1, fails


def t_validate():
    w = weights(100_000, 1)
    ws = ak.make_weight_set(w)
    t = ak.psa_construct(ws)
    rep = ak.validate_table(t, ws)
    tw, al = t.to_numpy()
    ro = O.validate_table(tw, al, w, ws.total)
    assert rep.ok, rep
    return f"{rep} oracle {ro}"


def t_big():
    for n, kind, dt in ((10**7, 0, torch.float32), (10**7, 4, torch.float32), (10**7, 0, torch.float64)):
        w = weights(n, kind)
        wd = torch.from_numpy(w).cuda().to(dt)
        ws = ak.make_weight_set(wd)
        w64 = wd.double().cpu().numpy()
        ref = O.vose_construct(w64, ws.total)
        torch.cuda.synchronize()
        t0 = time.time()
        t = ak.psa_construct(ws)
        torch.cuda.synchronize()
        dt_s = time.time() - t0
        am, gap = table_cmp(t, ref.tw, ref.alias, ws.average, 1e-9)
        rep = ak.validate_table(t, ws, tol=1e-4 if dt == torch.float32 else 1e-9, row_tol=20 * n * 2.0**-53)
        print(f"   n={n} kind={kind} {dt}: alias mismatches {am}, gap {gap:.2e}, {rep}, {dt_s*1e3:.1f} ms")
        assert rep.ok


for name, fn in [("uniform", t_uniform), ("total", t_total), ("assign", t_assign),
                 ("pary", t_pary), ("partition_plan_pack", t_partition_plan_pack),
                 ("build_f64", t_build), ("build_f32", t_build_f32), ("sample", t_sample),
                 ("validate", t_validate), ("fast_rng_chi2", t_fast_rng_chi2), ("big", t_big)]:
    check(name, fn)
print("SUMMARY", sum(ok for _, ok in results), "/", len(results))
