"""Pin the CPU oracle (test infrastructure) before trusting it.

Checked against (1) the Random123 Philox2x64-10 known-answer vectors, (2) the
reference tests' hand vectors, (3) golden fixtures generated from the
reference itself (tests/golden/make_golden.py), and (4) when the reference
is importable (build container), the live reference on fresh random inputs.
"""

import numpy as np
import pytest

import oracle as O
from conftest import golden_cases, random_weights


def test_philox_random123_kats(hand):
    for kat, w1 in zip(hand["philox2x64_10_kat"], hand["philox2x64_10_kat_w1_random123"]):
        c0, c1 = (int(x, 16) for x in kat["ctr"])
        key = int(kat["key"], 16)
        a, b = O.philox_both(c0, c1, key)
        assert a == int(kat["w0"], 16)
        assert b == int(w1, 16)
    assert O.uniform(0, 0, 0) == hand["uniform_py_0_0_0"]


def test_uniform_streams(golden):
    assert np.array_equal(O.uniform_block(20260815, 0, 0, 1000), golden["ub_a"])
    assert np.array_equal(O.uniform_block(7, 3, (1 << 64) - 5, 16), golden["ub_b"])


def test_hand_tables(hand):
    for key in ("table4", "single", "two"):
        c = hand[key]
        w, tot = O.make_weight_set(c["w"])
        t = O.vose_construct(w, tot)
        assert t.tw.tolist() == c["tw"] and t.alias.tolist() == c["alias"]
    w, tot = O.make_weight_set(hand["all_equal"]["w"])
    assert O.vose_construct(w, tot).alias.tolist() == hand["all_equal"]["alias"]
    p = O.partition_items([3.0, 1.0, 2.0, 2.0], 8.0)
    assert list(zip(p["l_index"].tolist(), p["l_weight"].tolist())) == [tuple(x) for x in hand["partition4"]["l"]]
    assert p["lprefix"].tolist() == hand["partition4"]["lprefix"]
    lc, hc, sp = O.compute_split_plan(p["lprefix"], p["hprefix"], p["h_weight"], 4, 2, 2.0)
    assert [list(x) for x in zip(lc.tolist(), hc.tolist(), sp.tolist())] == hand["plan4_s2"]
    t = O.vose_construct([3.0, 1.0, 2.0, 2.0], 8.0)
    for u, want in hand["rule4"]:
        assert O.rule(t.tw, t.alias, 2.0, [u])[0] == want
    for m, q, u, k in hand["binom_steps"]:
        assert O.binom_draw(m, q, u) == k


@pytest.mark.parametrize("ci", range(12))
def test_golden_tables(golden, ci):
    k = f"c{ci}_"
    w = golden[k + "weights"]
    tot = float(golden[k + "total"][0])
    w2, tot2 = O.make_weight_set(w)
    assert tot2 == tot  # np.sum's pairwise tree, restated
    v = O.vose_construct(w, tot)
    assert np.array_equal(v.tw, golden[k + "vose_tw"]) and np.array_equal(v.alias, golden[k + "vose_alias"])
    p = O.partition_items(w, tot)
    for f in ("l_index", "l_weight", "h_index", "h_weight", "lprefix", "hprefix"):
        assert np.array_equal(p[f], golden[k + f]), f
    n = w.size
    for s in (1, 2, 7, 64):
        if s > n:
            continue
        lc, hc, sp = O.compute_split_plan(p["lprefix"], p["hprefix"], p["h_weight"], n, s, p["avg"])
        assert np.array_equal(lc, golden[k + f"plan{s}_l"])
        assert np.array_equal(hc, golden[k + f"plan{s}_h"])
        assert np.array_equal(sp, golden[k + f"plan{s}_sp"])
        t = O.psa_construct(w, tot, s=s)
        assert np.array_equal(t.tw, golden[k + f"psa{s}_tw"])
        assert np.array_equal(t.alias, golden[k + f"psa{s}_alias"])
    seed = int(golden[k + "seed"][0])
    assert np.array_equal(O.sample_batch(v, 2000, seed, 3, 11), golden[k + "naive"])
    assert np.array_equal(O.sectioned_sample(v, 16, 3000, seed, 5, 7), golden[k + "sectioned16"])
    pre = O.greedy_prepack(w, tot, 64, 4)
    assert np.array_equal(pre["tw"], golden[k + "pre_tw"])
    assert np.array_equal(pre["alias"], golden[k + "pre_alias"])
    assert pre["nwritten"] / n == float(golden[k + "pre_handled"][0])
    ok, worst, item = O.validate_table(v.tw, v.alias, w, tot)
    g = golden[k + "vose_valid"]
    assert worst == g[0] and item == int(g[1])


def test_golden_assign_pary_binom(golden):
    params = golden["asg_params"]
    for i, (nr, S, M, seed, st) in enumerate(params):
        if int(nr) >= 10**9:
            continue  # 61k-section case: covered by the C++ product tests
        got = O.assign_sections(int(nr), int(S), int(M), int(seed), int(st))
        assert np.array_equal(got, golden[f"asg_{i}"])
    hay, q = golden["pary_hay"], golden["pary_q"]
    for p in (3, 8, 32):
        assert np.array_equal(O.partial_pary_search(hay, q, p), golden[f"pary_{p}"])
        assert list(O.contract_range(hay, q[0], q[-1], p)) == golden[f"pary_contract_{p}"].tolist()
    for m, q_, u, k in golden["binom"]:
        assert O.binom_draw(int(m), float(q_), float(u)) == int(k)


def test_pairwise_sum_matches_numpy(rng):
    for n in (0, 1, 7, 8, 9, 127, 128, 129, 1000, 65537, 1_000_003):
        a = rng.pareto(1.1, n) + 1e-6
        assert O.pairwise_sum(a) == float(np.sum(a))


# ---- live reference (build container only) --------------------------------

def test_live_reference_tables_and_samplers(reference, rng):
    A = reference
    for trial in range(40):
        n = int(rng.integers(1, 3000))
        w = random_weights(rng, n, trial % 5)
        ws = A.make_weight_set(w)
        _, tot = O.make_weight_set(w)
        assert tot == ws.total
        v, vo = A.vose_construct(ws), O.vose_construct(w, tot)
        assert np.array_equal(v.tw, vo.tw) and np.array_equal(v.alias, vo.alias)
        for s, ch, cap in ((7, False, 0), (64, True, 2), (3, True, 64)):
            if s > n:
                continue
            t = A.psa_construct(ws, s=s, workers=3, chunked=ch, chunk_capacity=max(cap, 2))
            to = O.psa_construct(w, tot, s=s, workers=3, chunked=ch, chunk_capacity=max(cap, 2))
            assert np.array_equal(t.tw, to.tw) and np.array_equal(t.alias, to.alias)
        seed = int(rng.integers(2**63))
        a = A.sample_batch(v, 700, A.RngStream(seed, 2, 9), workers=4)
        assert np.array_equal(a, O.sample_batch(vo, 700, seed, 2, 9, workers=4))
        b = A.sectioned_sample(v, 8, 900, A.RngStream(seed, 4, 1))
        assert np.array_equal(b, O.sectioned_sample(vo, 8, 900, seed, 4, 1))


def test_live_reference_assignment(reference, rng):
    A = reference
    for _ in range(300):
        n = int(rng.integers(1, 500_000))
        S = int(rng.integers(1, n + 10))
        M = int(rng.integers(0, 10**8))
        seed = int(rng.integers(2**63))
        assert np.array_equal(A.assign_sections(n, S, M, seed, stream=2).counts,
                              O.assign_sections(n, S, M, seed, 2))


def test_decision_margins_pinned(rng):
    """The O(N) exact margins (oracle decision_margins, fixed-point keys)
    equal the exact fsum-based nearest-key distances of conftest."""
    from conftest import near_tie_margins

    for n, kind in ((40, 3), (300, 0), (1500, 1), (900, 2)):
        w = random_weights(rng, n, kind)
        _, total = O.make_weight_set(w)
        rows = np.arange(1, n + 1)
        a = O.decision_margins(w, total, rows)
        b = np.array(near_tie_margins(w, total, rows))
        assert np.max(np.abs(a - b)) < 1e-10
