"""GPU parity: RNG, make_weight_set, validate_table, partition, split plan,
pack sweep, partial p-ary search — each against the golden fixtures (made
from the reference) and the oracle, through the C-ABI library."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2106_12270_b200 as ak
from paper_2106_12270_b200 import _lib
from paper_2106_12270_b200.pack import pack_all
from conftest import random_weights

pytestmark = pytest.mark.gpu
DEV = "cuda"


# ---- rng --------------------------------------------------------------------

def test_philox_kats_on_device(hand):
    kats = hand["philox2x64_10_kat"]
    s64 = lambda x: x - (1 << 64) if x >= (1 << 63) else x
    col = lambda vals: torch.tensor([s64(v) for v in vals], dtype=torch.int64, device=DEV)
    ctr = col([int(k["ctr"][0], 16) for k in kats])
    strm = col([int(k["ctr"][1], 16) for k in kats])
    key = col([int(k["key"], 16) for k in kats])
    w0 = torch.empty(3, dtype=torch.int64, device=DEV)
    w1 = torch.empty(3, dtype=torch.int64, device=DEV)
    _lib.check(_lib.lib().ak_philox2x64(ctr.data_ptr(), strm.data_ptr(), key.data_ptr(), 3,
                                        w0.data_ptr(), w1.data_ptr(), _lib.stream_ptr()))
    got0 = [x & (2**64 - 1) for x in w0.cpu().tolist()]
    got1 = [x & (2**64 - 1) for x in w1.cpu().tolist()]
    assert got0 == [int(k["w0"], 16) for k in kats]
    assert got1 == [int(x, 16) for x in hand["philox2x64_10_kat_w1_random123"]]


def philox4x32_np(c, k):
    """Philox4x32-10 (Random123 constants), the restatement the KATs pin."""
    M0, M1, W0, W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85
    c, k = list(c), list(k)
    for _ in range(10):
        p0, p1 = M0 * c[0], M1 * c[2]
        c = [(p1 >> 32) ^ c[1] ^ k[0], p1 & 0xFFFFFFFF, (p0 >> 32) ^ c[3] ^ k[1], p0 & 0xFFFFFFFF]
        k = [(k[0] + W0) & 0xFFFFFFFF, (k[1] + W1) & 0xFFFFFFFF]
    return c


# Random123 known-answer vectors for philox4x32_10 (kat_vectors)
PHILOX4X32_KATS = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def test_philox4x32_kats_on_device(rng):
    """The GPU-native RNG (rng="philox4x32") against Random123's published
    answers, through all three formulations the samplers compile (generic
    loop, inline round keys, round-key table), plus random inputs against
    the restatement."""
    ins = [(c, k) for c, k, _ in PHILOX4X32_KATS]
    for _ in range(200):
        ins.append((tuple(int(x) for x in rng.integers(0, 2**32, 4)), tuple(int(x) for x in rng.integers(0, 2**32, 2))))
    m = len(ins)
    as_i32 = lambda xs: torch.tensor([x - (1 << 32) if x >= (1 << 31) else x for x in xs], dtype=torch.int32, device=DEV)
    ctr = as_i32([x for c, _ in ins for x in c])
    key = as_i32([x for _, k in ins for x in k])
    out = torch.empty(12 * m, dtype=torch.int32, device=DEV)
    _lib.check(_lib.lib().ak_philox4x32(ctr.data_ptr(), key.data_ptr(), m, out.data_ptr(), _lib.stream_ptr()))
    got = [x & 0xFFFFFFFF for x in out.cpu().tolist()]
    for i, (c, k) in enumerate(ins):
        want = list(PHILOX4X32_KATS[i][2]) if i < 3 else philox4x32_np(c, k)
        assert philox4x32_np(c, k) == want  # the restatement reproduces the KATs
        for v in range(3):
            assert got[12 * i + 4 * v:12 * i + 4 * v + 4] == want, (i, v)


def test_uniform_block_golden_and_wrap(golden):
    r = ak.RngStream(20260815)
    assert np.array_equal(ak.uniform_block(r, 1000).cpu().numpy(), golden["ub_a"])
    assert r.counter == 1000
    r = ak.RngStream(7, 3, (1 << 64) - 5)
    assert np.array_equal(ak.uniform_block(r, 16).cpu().numpy(), golden["ub_b"])


def test_uniform_block_resume(rng):
    r = ak.RngStream(seed=7, stream=3, counter=50)
    a = ak.uniform_block(r, 10)
    b = ak.uniform_block(r, 10)
    both = ak.uniform_block(ak.RngStream(7, 3, 50), 20)
    assert torch.equal(torch.cat([a, b]), both)
    big = ak.uniform_block(ak.RngStream(99, 1, 123), 1_000_003).cpu().numpy()
    assert np.array_equal(big, O.uniform_block(99, 1, 123, 1_000_003))


# ---- make_weight_set / validate_table ---------------------------------------

def test_weight_set_totals_bit_identical_to_np_sum(golden, rng):
    for ci in range(len(golden["sizes"])):
        w = golden[f"c{ci}_weights"]
        assert ak.make_weight_set(w).total == float(golden[f"c{ci}_total"][0])
    for n in (1, 6, 7, 8, 9, 127, 128, 129, 1000, 2049, 65_537, 100_003, 3_000_001, 10_000_019):
        w = random_weights(rng, n, n % 5)
        assert ak.make_weight_set(w).total == float(np.sum(w))
        w32 = w.astype(np.float32)
        ws = ak.make_weight_set(torch.from_numpy(w32).to(DEV))
        assert ws.dtype == torch.float32
        assert ws.total == float(np.sum(w32.astype(np.float64)))


def test_weight_set_totals_sweep_tree_shapes(rng):
    """np.sum's pairwise tree at 48 log-uniform sizes up to 1e8: the cut
    nodes (about 1025..2048 values) reach leaves of <= 128 values at depth 4
    or 5 depending on n, and the device walks each node's leaf list."""
    sizes = sorted({int(x) for x in np.exp(rng.uniform(np.log(3e3), np.log(1e8), 48))})
    for n in sizes:
        for dt in (torch.float64, torch.float32):
            w = (torch.rand(n, dtype=torch.float64, device=DEV) + 1e-3).to(dt)
            expect = float(np.sum(w.cpu().numpy().astype(np.float64)))
            assert ak.make_weight_set(w).total == expect, (n, dt)


@pytest.mark.parametrize("bad,idx", [([1.0, 0.0, 2.0], 2), ([1.0, -3.0], 2),
                                     ([float("nan"), 1.0], 1), ([1.0, float("inf")], 2)])
def test_invalid_weight_reports_1based_index(bad, idx):
    with pytest.raises(ak.InvalidWeight) as e:
        ak.make_weight_set(bad)
    assert e.value.index == idx


def test_invalid_weight_first_bad_wins_at_scale():
    w = torch.rand(5_000_000, dtype=torch.float64, device=DEV) + 0.5
    w[4_000_001] = -1.0
    w[3_999_999] = float("nan")
    with pytest.raises(ak.InvalidWeight) as e:
        ak.make_weight_set(w)
    assert e.value.index == 4_000_000


def test_invalid_weight_in_leaf_tails():
    # bad values in a leaf's tail (n % 8 != 0) and in accumulator lanes
    for n, pos in ((1_000_003, 1_000_002), (1_000_003, 999_999), (4099, 4098), (130, 129), (5, 3)):
        w = torch.ones(n, dtype=torch.float32, device=DEV)
        w[pos] = float("nan")
        with pytest.raises(ak.InvalidWeight) as e:
            ak.make_weight_set(w)
        assert e.value.index == pos + 1


def test_empty_and_shape():
    with pytest.raises(ak.EmptyInput):
        ak.make_weight_set([])
    with pytest.raises(ValueError):
        ak.make_weight_set(np.ones((2, 2)))


def test_validate_table_matches_oracle(golden, rng):
    for ci in range(len(golden["sizes"])):
        w = golden[f"c{ci}_weights"]
        ws = ak.make_weight_set(w)
        t = ak.AliasTable.from_numpy(golden[f"c{ci}_vose_tw"], golden[f"c{ci}_vose_alias"], ws.n, ws.total)
        rep = ak.validate_table(t, ws)
        g = golden[f"c{ci}_vose_valid"]
        assert rep.ok == bool(g[2])
        assert abs(rep.worst_rel_error - g[0]) <= 1e-15 + 1e-6 * g[0]
    ws = ak.make_weight_set([3.0, 1.0, 2.0, 2.0])
    bad = ak.AliasTable.from_numpy([2.0, 2.0, 2.0, 2.0], [1, 1, 3, 4], 4, 8.0)
    rep = ak.validate_table(bad, ws)
    assert not rep.ok and rep.worst_item in (1, 2)
    over = ak.AliasTable.from_numpy([1.5, 0.5], [1, 1], 2, 2.0)
    assert not ak.validate_table(over, ak.make_weight_set([1.0, 1.0])).ok
    with pytest.raises(ak.SizeMismatch):
        ak.validate_table(ak.AliasTable.from_numpy(np.ones(3), np.ones(3), 3, 3.0),
                          ak.make_weight_set([1.0, 1.0]))


# ---- partition / plan / pack -------------------------------------------------

def _ref_partition(golden, ci):
    k = f"c{ci}_"
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    w = golden[k + "weights"]
    tot = float(golden[k + "total"][0])
    return ak.LightHeavyPartition(t(golden[k + "l_index"]), t(golden[k + "l_weight"]),
                                  t(golden[k + "h_index"]), t(golden[k + "h_weight"]),
                                  t(golden[k + "lprefix"]), t(golden[k + "hprefix"]), tot / w.size)


def test_partition_matches_reference(golden, hand):
    p = ak.partition_items(ak.make_weight_set(hand["table4"]["w"]))
    assert p.l == [tuple(x) for x in hand["partition4"]["l"]]
    assert p.h == [tuple(x) for x in hand["partition4"]["h"]]
    assert p.lprefix.tolist() == hand["partition4"]["lprefix"]
    for ci in range(len(golden["sizes"])):
        k = f"c{ci}_"
        p = ak.partition_items(ak.make_weight_set(golden[k + "weights"]))
        for f in ("l_index", "l_weight", "h_index", "h_weight"):
            assert np.array_equal(getattr(p, f).cpu().numpy(), golden[k + f]), f
        for f in ("lprefix", "hprefix"):
            got, want = getattr(p, f).cpu().numpy(), golden[k + f]
            ulp = np.spacing(np.maximum(np.abs(want), 1e-300))
            assert np.all(np.abs(got - want) <= 2 * ulp), f  # dd-exact vs Neumaier


@pytest.mark.parametrize("n", [524_289, 3_000_017, 20_000_003])
def test_partition_many_chunks_vs_oracle(rng, n):
    """partition_items past one scan chunk (> 256 tiles of 2048 items): the
    chunk scans + chained carries give the oracle's order exactly and its
    Neumaier prefixes within 2 ulp (partition.py:62-131)."""
    w = rng.pareto(1.1, n) + 1e-6
    ws = ak.make_weight_set(torch.from_numpy(w).to(DEV))
    p = ak.partition_items(ws)
    po = O.partition_items(w, ws.total)
    for f in ("l_index", "l_weight", "h_index", "h_weight"):
        assert np.array_equal(getattr(p, f).cpu().numpy(), po[f]), f
    for f in ("lprefix", "hprefix"):
        got, want = getattr(p, f).cpu().numpy(), po[f]
        ulp = np.spacing(np.maximum(np.abs(want), 1e-300))
        assert np.all(np.abs(got - want) <= 2 * ulp), f


def test_prefix_sums_recover_increments(rng):
    ws = ak.make_weight_set(rng.pareto(1.1, 30000) + 1e-6)
    p = ak.partition_items(ws)
    for pre, w in ((p.lprefix, p.l_weight), (p.hprefix, p.h_weight)):
        pre, w = pre.cpu().numpy(), w.cpu().numpy()
        d = np.abs(np.diff(pre) - w)
        ulp = np.spacing(np.maximum(np.abs(pre[1:]), np.abs(pre[:-1])))
        assert np.all(d <= 4 * ulp)


@pytest.mark.parametrize("method", ["binary", "batched"])
def test_split_plan_bit_identical_on_reference_partition(golden, method):
    for ci in range(len(golden["sizes"])):
        p = _ref_partition(golden, ci)
        for s in (1, 2, 7, 64):
            if s > p.n:
                continue
            plan = ak.compute_split_plan(p, s, method=method)
            k = f"c{ci}_plan{s}_"
            assert np.array_equal(plan.lcounts.cpu().numpy(), golden[k + "l"])
            assert np.array_equal(plan.hcounts.cpu().numpy(), golden[k + "h"])
            assert np.array_equal(plan.spills.cpu().numpy(), golden[k + "sp"])


@pytest.mark.parametrize("method", ["binary", "batched"])
def test_split_plan_many_boundaries_vs_oracle(rng, method):
    for trial in range(12):
        n = int(rng.integers(2, 300_000))
        w = random_weights(rng, n, trial % 5)
        _, tot = O.make_weight_set(w)
        po = O.partition_items(w, tot)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
        p = ak.LightHeavyPartition(t(po["l_index"]), t(po["l_weight"]), t(po["h_index"]),
                                   t(po["h_weight"]), t(po["lprefix"]), t(po["hprefix"]), po["avg"])
        for s in (3, 1000, n // 7 + 1, n):
            lc, hc, sp = O.compute_split_plan(po["lprefix"], po["hprefix"], po["h_weight"], n, s, po["avg"])
            plan = ak.compute_split_plan(p, s, method=method)
            assert np.array_equal(plan.lcounts.cpu().numpy(), lc)
            assert np.array_equal(plan.hcounts.cpu().numpy(), hc)
            assert np.array_equal(plan.spills.cpu().numpy(), sp)


def test_plan_hand_and_validation(hand):
    p = ak.partition_items(ak.make_weight_set(hand["table4"]["w"]))
    assert [list(b) for b in ak.compute_split_plan(p, 2).boundaries] == hand["plan4_s2"]
    assert ak.compute_split_plan(p, 1).boundaries == [(0, 0, 0.0), (3, 1, 0.0)]
    p12 = ak.partition_items(ak.make_weight_set([2.0] * 12))
    plan = ak.compute_split_plan(p12, 4)
    assert plan.lcounts.tolist() == hand["plan_equal12_s4_l"] and plan.hcounts.tolist() == [0] * 5
    with pytest.raises(ak.InvalidSectionCount):
        ak.compute_split_plan(p, 0)
    with pytest.raises(ak.InvalidSectionCount):
        ak.compute_split_plan(p, 5)
    assert ak.binary_search_boundary(p, 0, 0.0) == (0, 0, 0.0)


def _boundary_ref(lpre, hpre, hw, n_i, cap):
    """split.py:107-137 restated over numpy arrays (the reference loop)."""
    nl, nh = lpre.size - 1, hpre.size - 1
    lo, hi = max(0, n_i - nl), min(n_i, nh)
    best, a, b = lo, lo, hi
    while a <= b:
        mid = (a + b) >> 1
        if lpre[n_i - mid] + hpre[mid] <= cap:
            best, a = mid, mid + 1
        else:
            b = mid - 1
    h, l = best, n_i - best
    taken = cap - (float(lpre[l]) + float(hpre[h]))
    spill = max(float(hw[h]) - taken, 0.0) if h < nh and taken > 0.0 else 0.0
    return l, h, spill


def test_binary_search_boundary_real_boundaries(rng):
    """a5: the scalar boundary search equals the plan kernel at every real
    boundary (n_i = floor(i N / s), cap = n_i * avg), as the reference's own
    cross-check does (tests/test_split.py:76-88), and equals the reference
    loop restated at arbitrary (n_i, cap) pairs on the same prefix arrays."""
    for trial in range(12):
        n = int(rng.integers(50, 20_000))
        w = random_weights(rng, n, trial % 5)
        p = ak.partition_items(ak.make_weight_set(w))
        s = int(rng.integers(2, min(n, 300)))
        plan = ak.compute_split_plan(p, s)
        lpre, hpre = p.lprefix.cpu().numpy(), p.hprefix.cpu().numpy()
        hw = p.h_weight.cpu().numpy()
        lc, hc, sp = O.compute_split_plan(lpre, hpre, hw, n, s, p.avg)
        for i in range(1, s):
            n_i = i * n // s
            got = ak.binary_search_boundary(p, n_i, n_i * p.avg)
            assert got == (int(lc[i]), int(hc[i]), float(sp[i])), (trial, i)
            assert got == plan.boundaries[i]
        for _ in range(40):
            n_i = int(rng.integers(0, n + 1))
            cap = float(rng.uniform(0, 1.2)) * n_i * p.avg
            assert ak.binary_search_boundary(p, n_i, cap) == _boundary_ref(lpre, hpre, hw, n_i, cap)
    with pytest.raises(ValueError):
        ak.binary_search_boundary(p, n + 1, 0.0)


@pytest.mark.parametrize("cap", [0, 2, 3, 64, 10**6])
def test_pack_sections_bit_identical(golden, cap):
    """The reference's sweep on its own partition and plan -> its psa table."""
    for ci in range(len(golden["sizes"])):
        p = _ref_partition(golden, ci)
        n = p.n
        tot = float(golden[f"c{ci}_total"][0])
        for s in (1, 2, 7, 64):
            if s > n:
                continue
            plan = ak.compute_split_plan(p, s, method="binary")
            out = ak.AliasTable.blank(n, tot)
            if cap == 0:
                for i in range(1, s + 1):
                    ak.pack_section(p, plan, i, out)
            else:
                pack_all(p, plan, out, cap)
            tw, al = out.to_numpy()
            assert np.array_equal(tw, golden[f"c{ci}_psa{s}_tw"])
            assert np.array_equal(al, golden[f"c{ci}_psa{s}_alias"])


def test_pack_section_spills_and_ownership(rng):
    for trial in range(6):
        n = int(rng.integers(4, 800))
        ws = ak.make_weight_set(random_weights(rng, n, trial % 3))
        p = ak.partition_items(ws)
        s = min(5, n)
        plan = ak.compute_split_plan(p, s)
        out = ak.AliasTable.blank(n, ws.total)
        for i in range(1, s + 1):
            before = out.tw.clone()
            got = ak.pack_section(p, plan, i, out)
            touched = torch.nonzero(out.tw != before).flatten().cpu().numpy()
            la, lb = plan.lcounts[i - 1].item(), plan.lcounts[i].item()
            ha, hb = plan.hcounts[i - 1].item(), plan.hcounts[i].item()
            owned = np.concatenate([p.l_index[la:lb].cpu().numpy(), p.h_index[ha:hb].cpu().numpy()]) - 1
            assert np.array_equal(np.sort(owned), touched)
            if i < s and plan.hcounts[i].item() < p.h_index.numel():
                assert got == pytest.approx(plan.spills[i].item(), abs=1e-9 * p.avg)
        assert ak.validate_table(out, ws).ok


def test_plan_tampering_rejected():
    ws = ak.make_weight_set([3.0, 1.0, 2.0, 2.0, 5.0, 1.0])
    p = ak.partition_items(ws)
    plan = ak.compute_split_plan(p, 2)
    out = ak.AliasTable.blank(ws.n, ws.total)
    bad = ak.SplitPlan(2, plan.lcounts.clone(), plan.hcounts.clone(), plan.spills.clone())
    bad.lcounts[-1] += 1
    with pytest.raises(ak.PlanInconsistent):
        ak.pack_section(p, bad, 1, out)
    bad2 = ak.SplitPlan(2, plan.lcounts.clone(), plan.hcounts.clone(), plan.spills.clone())
    bad2.lcounts[1] = bad2.lcounts[2] + 1
    with pytest.raises(ak.PlanInconsistent):
        ak.pack_section(p, bad2, 1, out)
    with pytest.raises(ak.PlanInconsistent):
        ak.pack_section(p, plan, 0, out)
    with pytest.raises(ak.PlanInconsistent):
        ak.pack_section(p, plan, 3, out)
    with pytest.raises(ValueError):
        ak.chunked_pack_section(p, plan, 1, 1, out)


# ---- partial p-ary search ----------------------------------------------------

def test_pary_golden_and_hand(golden, hand):
    for p in (3, 8, 32):
        got = ak.partial_pary_search(golden["pary_hay"], golden["pary_q"], p=p).cpu().numpy()
        assert np.array_equal(got, golden[f"pary_{p}"])
    h = hand["pary_hand"]
    assert ak.partial_pary_search(h["hay"], h["q"], p=h["p"]).tolist() == h["out"]
    t = hand["pary_ties"]
    assert ak.partial_pary_search(t["hay"], t["q"], p=3).tolist() == t["out"]
    assert ak.partial_pary_search([1.0, 2.0], [], p=8).tolist() == []
    assert ak.partial_pary_search([], [1.0, 2.0], p=3).tolist() == [0, 0]
    with pytest.raises(ak.UnsortedInput):
        ak.partial_pary_search([3.0, 1.0], [1.0])
    with pytest.raises(ak.UnsortedInput):
        ak.partial_pary_search([1.0, 3.0], [2.0, 1.0])
    with pytest.raises(ValueError):
        ak.partial_pary_search([1.0, 3.0], [1.0], p=2)


def test_pary_equals_searchsorted(rng):
    for i in range(300):
        n = int(rng.integers(0, 100_000))
        if i % 2:
            hay = np.sort(rng.normal(0, 10, n))
            q = np.sort(rng.normal(0, 12, int(rng.integers(0, 513))))
        else:  # long tied runs
            hay = np.sort(rng.integers(0, max(n // 4, 1), n)).astype(np.float64)
            q = np.sort(rng.integers(-2, max(n // 4, 1) + 2, int(rng.integers(0, 513)))).astype(np.float64)
        ref = np.searchsorted(hay, q, side="left")
        for p in (3, 8, 32, 100):
            assert np.array_equal(ak.partial_pary_search(hay, q, p=p).cpu().numpy(), ref)
