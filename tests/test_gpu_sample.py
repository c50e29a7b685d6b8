"""GPU parity of both samplers: bit-exact against the reference for the same
RngStream (golden fixtures + oracle), f32 tables bit-exact against the rule on
the upcast table, and chi-square goodness of fit for the GPU-native RNG."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2106_12270_b200 as ak
from paper_2106_12270_b200 import distributed as D
from conftest import random_weights

pytestmark = pytest.mark.gpu
DEV = "cuda"


def table_from_golden(golden, ci, dtype=torch.float64):
    k = f"c{ci}_"
    n = golden[k + "weights"].size
    return ak.AliasTable.from_numpy(golden[k + "vose_tw"], golden[k + "vose_alias"], n,
                                    float(golden[k + "total"][0]), dtype=dtype)


def test_rule_hand_values(hand):
    t = ak.vose_construct(ak.make_weight_set(hand["table4"]["w"]))
    for u, want in hand["rule4"]:
        assert ak.sample_from_uniforms(t, [u]).item() == want


def test_golden_samplers(golden):
    for ci in range(len(golden["sizes"])):
        t = table_from_golden(golden, ci)
        seed = int(golden[f"c{ci}_seed"][0])
        r = ak.RngStream(seed, 3, 11)
        assert np.array_equal(ak.sample_batch(t, 2000, r).cpu().numpy(), golden[f"c{ci}_naive"])
        assert r.counter == 2011
        r = ak.RngStream(seed, 5, 7)
        assert np.array_equal(ak.sectioned_sample(t, 16, 3000, r).cpu().numpy(),
                              golden[f"c{ci}_sectioned16"])
        assert r.counter == 3007


def test_batch_is_sequence_of_single_draws():
    t = ak.vose_construct(ak.make_weight_set([3.0, 1.0, 2.0, 2.0]))
    r1, r2 = ak.RngStream(42), ak.RngStream(42)
    batch = ak.sample_batch(t, 64, r1)
    assert batch.tolist() == [ak.sample_one(t, r2) for _ in range(64)]
    assert r1.counter == r2.counter == 64


def test_empty_and_args():
    t = ak.vose_construct(ak.make_weight_set([3.0, 1.0]))
    r = ak.RngStream(1, 1)
    assert ak.sample_batch(t, 0, r).numel() == 0 and r.counter == 0
    assert ak.sectioned_sample(t, 2, 0, r).numel() == 0 and r.counter == 0
    with pytest.raises(ValueError):
        ak.sample_batch(t, -1, r)
    with pytest.raises(ak.InvalidSectionSize):
        ak.sectioned_sample(t, 0, 5, r)
    with pytest.raises(ValueError):
        ak.sample_batch(t, 5, r, rng="mt19937")


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_random_tables_bit_exact(rng, dtype):
    for trial in range(16):
        n = int(np.exp(rng.uniform(0, np.log(300_000)))) + 1
        w = random_weights(rng, n, trial % 5)
        if dtype == torch.float32:
            w = w.astype(np.float32).astype(np.float64)
        _, tot = O.make_weight_set(w)
        ref = O.vose_construct(w, tot)
        t = ak.AliasTable.from_numpy(ref.tw, ref.alias, n, tot, dtype=dtype)
        tw, al = t.to_numpy()  # the device table as the reference would see it
        rt = O.Table(tw, al, n, tot)
        seed = int(rng.integers(2**63))
        ctr = int(rng.integers(2**64, dtype=np.uint64)) if trial % 4 == 0 else int(rng.integers(1000))
        got = ak.sample_batch(t, 50_000, ak.RngStream(seed, 3, ctr)).cpu().numpy()
        assert np.array_equal(got, O.sample_batch(rt, 50_000, seed, 3, ctr))
        for S in (1, 7, 64, 1000, 1 << 13, 1 << 14, 10**9):
            got = ak.sectioned_sample(t, S, 40_000, ak.RngStream(seed, 9, ctr)).cpu().numpy()
            assert np.array_equal(got, O.sectioned_sample(rt, S, 40_000, seed, 9, ctr)), S
        u = O.uniform_block(seed, 4, 0, 10_000)
        assert np.array_equal(ak.sample_from_uniforms(t, u).cpu().numpy(),
                              O.rule(tw, al, tot / n, u))


def test_sectioned_row_provenance(rng):
    w = rng.random(300_000) + 0.01
    ws = ak.make_weight_set(w)
    t = ak.vose_construct(ws)
    tw, al = t.to_numpy()
    S, M = 1 << 14, 2_000_000
    out = ak.sectioned_sample(t, S, M, ak.RngStream(31, 6)).cpu().numpy()
    asg = ak.assign_sections(t.n, S, M, 31, 6)
    off = 0
    for j in range(asg.n_sections):
        mj = int(asg.counts[j])
        lo = j * asg.section_size
        span = min(lo + asg.section_size, t.n) - lo
        strm = O.derive_stream(31, 6, j, O.SALT_SECTION)
        u = O.uniform_block(31, strm, 0, mj)
        assert np.array_equal(out[off:off + mj], O.rule(tw, al, t.average, u, lo, span))
        off += mj
    assert off == M


def test_shards_reassemble_single_gpu_output():
    """Every rank's slice (naive counter blocks, sectioned section runs)
    concatenates to the single-GPU output (the multi-GPU sharding, run here
    rank by rank on one device)."""
    ws = ak.gen_uniform(1_000_000, ak.RngStream(5), dtype=torch.float32)
    t = ak.psa_construct(ws)
    M = 3_000_001
    full = ak.sample_batch(t, M, ak.RngStream(9, 1, 77))
    for world in (2, 4, 8):
        parts = [D.sample_batch_shard(t, M, ak.RngStream(9, 1, 77), g, world) for g in range(world)]
        assert torch.equal(torch.cat(parts), full)
    S = 1 << 14
    fulls = ak.sectioned_sample(t, S, M, ak.RngStream(9, 2, 5))
    for world in (2, 4, 8):
        out = torch.full((M,), -1, dtype=torch.int64, device=DEV)
        for g in range(world):
            plan = D.ShardedSectioned(t, S, M, ak.RngStream(9, 2, 5), g, world)
            piece = torch.empty(plan.draws, dtype=torch.int64, device=DEV)
            plan.run(t, ak.RngStream(9, 2, 5), piece)
            out[plan.out_off:plan.out_off + plan.draws] = piece
        assert torch.equal(out, fulls)


@pytest.mark.parametrize("rng_mode", ["reference", "philox4x32"])
def test_chi_square_gate(rng_mode, acceptance):
    """The reference's c5 protocol exactly (test_acceptance.py:157-188):
    n = 1000, 1e7 draws, 100 seeds per configuration, at most 2 failures at
    alpha = 0.001, for baseline and sectioned (S = 64, 2^14) sampling of a
    uniform and a power-law table — here for both RNG modes."""
    n, M = 1000, 10**7
    g = np.random.default_rng(0xACCE97 + 5)
    sets = {"uniform": g.random(n) + 1e-9, "powerlaw": np.arange(1, n + 1, dtype=np.float64) ** -1.0}
    verdicts, ok_all = [], True
    for dist, w in sets.items():
        ws = ak.make_weight_set(w)
        t = ak.vose_construct(ws)
        probs = w / ws.total
        for sampler, S in (("baseline", 0), ("sectioned", 64), ("sectioned", 2**14)):
            fails = 0
            for seed in range(100):
                r = ak.RngStream(0xACCE97 + seed, 7 * S + (dist == "powerlaw"))
                x = ak.sample_batch(t, M, r, rng=rng_mode) if S == 0 else \
                    ak.sectioned_sample(t, S, M, r, rng=rng_mode)
                _, _, passed = ak.chi_square_test(ak.frequency_counts(x, n), probs)
                fails += not passed
            verdicts.append(f"{dist}/{sampler}{'' if S == 0 else f'(S={S})'}: {fails}")
            ok_all &= fails <= 2
    acceptance(f"{'PASS' if ok_all else 'FAIL'}  chi-square ({rng_mode}) at 0.001, 1e7 draws, "
               f"100 seeds; failures per config <= 2 [{', '.join(verdicts)}]")
    assert ok_all, verdicts


def test_frequency_counts_device():
    c = ak.frequency_counts(torch.tensor([1, 3, 3, 2, 3], device=DEV), 4)
    assert c.tolist() == [1, 1, 3, 0]
    with pytest.raises(ak.IndexOutOfRange):
        ak.frequency_counts(torch.tensor([0, 1], device=DEV), 3)
    assert ak.frequency_counts(torch.empty(0, dtype=torch.int64, device=DEV), 2).tolist() == [0, 0]


def test_status_words_per_stream_threads():
    """Entry points that read a status word back (frequency_counts,
    count_unwritten, partial_pary_search) keep one scratch per (device,
    stream): calls from several host threads on their own streams, one of
    them failing, must not see each other's flags."""
    import threading

    bad = torch.tensor([0, 1], device=DEV)
    good = torch.tensor([1, 2, 2], device=DEV)
    hay = torch.arange(1000, dtype=torch.float64, device=DEV)
    errs = []

    def worker(k):
        s = torch.cuda.Stream()
        try:
            with torch.cuda.stream(s):
                for it in range(30):
                    if (k + it) % 2:
                        with pytest.raises(ak.IndexOutOfRange):
                            ak.frequency_counts(bad, 3)
                    else:
                        assert ak.frequency_counts(good, 3).tolist() == [1, 2, 0]
                    q = torch.tensor([3.5, 10.0, 999.0], dtype=torch.float64, device=DEV)
                    assert ak.partial_pary_search(hay, q, 8).tolist() == [4, 10, 999]
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs


def test_threads_share_default_stream():
    """host threads that all use the default stream must not share
    scratch.  Four threads build different tables and read status words back
    concurrently on the default stream; every result must equal the
    single-threaded one."""
    import threading

    sets = [ak.make_weight_set(random_weights(np.random.default_rng(50 + k), 200_000 + 977 * k, k % 3))
            for k in range(4)]
    want = [ak.psa_construct(ws).to_numpy() for ws in sets]
    bad = torch.tensor([0, 1], device=DEV)
    good = torch.tensor([1, 2, 2], device=DEV)
    errs = []

    def worker(k):
        try:
            for it in range(6):
                tw, al = ak.psa_construct(sets[k]).to_numpy()
                assert np.array_equal(al, want[k][1]) and np.array_equal(tw, want[k][0])
                if (k + it) % 2:
                    with pytest.raises(ak.IndexOutOfRange):
                        ak.frequency_counts(bad, 3)
                else:
                    assert ak.frequency_counts(good, 3).tolist() == [1, 2, 0]
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs


def test_out_buffer_is_checked():
    """a caller-supplied out tensor is validated before the kernel
    writes through its pointer."""
    t = ak.psa_construct(ak.make_weight_set(np.arange(1.0, 101.0)))
    r = ak.RngStream(1)
    for bad in (torch.empty(9, dtype=torch.int64, device=DEV),             # too short
                torch.empty(10, dtype=torch.int16, device=DEV),            # wrong dtype
                torch.empty(20, dtype=torch.int64, device=DEV)[::2],       # strided
                torch.empty(10, dtype=torch.int64)):                       # host
        with pytest.raises(ValueError):
            ak.sample_batch(t, 10, r, out=bad)
        with pytest.raises(ValueError):
            ak.sectioned_sample(t, 16, 10, r, out=bad)
    assert r.counter == 0  # nothing drawn
    ok = torch.empty(10, dtype=torch.int64, device=DEV)
    assert ak.sample_batch(t, 10, r, out=ok) is ok


def philox4x32_words(call: np.ndarray, strm: int, seed: int):
    """numpy Philox4x32-10 (Random123 constants) of counters (call lo, call
    hi, strm lo, strm hi) under key (seed lo, seed hi): the two 64-bit words
    of every call (the GPU-native stream of rng="philox4x32")."""
    M0, M1, W0, W1, m32 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85, 0xFFFFFFFF
    call = call.astype(np.uint64)
    c0 = call & np.uint64(m32)
    c1 = call >> np.uint64(32)
    c2 = np.full_like(c0, strm & m32)
    c3 = np.full_like(c0, strm >> 32)
    k0, k1 = seed & m32, seed >> 32
    for _ in range(10):
        p0 = c0 * np.uint64(M0)
        p1 = c2 * np.uint64(M1)
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(m32)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(m32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0
        k0, k1 = (k0 + W0) & m32, (k1 + W1) & m32
    return (c1 << np.uint64(32)) | c0, (c3 << np.uint64(32)) | c2


def fast_section_reference(tw, al, avg, lo, span, seed, strm, ctr0, m):
    v = np.uint64(ctr0) + np.arange(m, dtype=np.uint64)
    a, b = philox4x32_words(v >> np.uint64(1), strm, seed)
    word = np.where((v & np.uint64(1)) == 0, a, b)
    u = (word >> np.uint64(11)).astype(np.float64) * 2.0**-53
    return O.rule(tw, al, avg, u, lo, span)


@pytest.mark.parametrize("ctr0,m", [(0, 1), (0, 100_001), (7, 100_000), (2**33 + 3, 54_321)])
def test_fast_rng_naive_bit_exact(ctr0, m):
    """rng="philox4x32" naive draws: draw i takes word (ctr0+i)&1 of the call
    (ctr0+i)>>1 on the caller's stream, the rule over the whole table."""
    g = np.random.default_rng(m)
    w = g.random(5000) + 1e-3
    ws = ak.make_weight_set(w)
    t = ak.psa_construct(ws)
    tw, al = t.to_numpy()
    seed, stream = 0xABCDEF, 5
    want = fast_section_reference(tw, al, t.average, 0, t.n, seed, stream, ctr0, m)
    got = ak.sample_batch(t, m, ak.RngStream(seed, stream, ctr0), rng="philox4x32")
    assert np.array_equal(got.cpu().numpy(), want)


@pytest.mark.parametrize("ctr0,dtype,S,tail", [(0, torch.float32, 4096, 1000), (5, torch.float32, 4096, 1000),
                                               (2**32 - 3, torch.float32, 4096, 1000),
                                               (7, torch.float64, 1 << 14, 1000),
                                               (3, torch.float64, 4096, 1000),
                                               (1, torch.float32, 3000, 7),      # non-power-of-two sections
                                               (2, torch.float32, 4096, 2),      # a 2-row last section
                                               (4, torch.float64, 2048, 1)])     # a 1-row last section
def test_fast_rng_sectioned_bit_exact(ctr0, dtype, S, tail):
    """rng="philox4x32": the sectioned kernel (interior fast path, checked
    edges, misaligned outputs, several passes per call; f64 rows staged as
    rows (S=4096) or, for 2^14-row sections, as threshold/alias arrays)
    against a numpy restatement of the GPU-native stream."""
    g = np.random.default_rng(ctr0 + 1)
    # enough draws that even a 1- or 2-row last section runs whole CTA steps
    n, M = 3 * S + tail, (1_500_003 if tail >= 1000 else 15_000_007)
    w = (g.random(n) + 1e-3).astype(np.float32 if dtype == torch.float32 else np.float64)
    ws = ak.make_weight_set(torch.from_numpy(w).to(DEV))
    t = ak.psa_construct(ws)
    tw, al = t.to_numpy()
    seed, stream = 0x1234_5678_9ABC, 11
    asg = ak.assign_sections(n, S, M, seed, stream)
    want = np.concatenate([
        fast_section_reference(tw, al, t.average, j * S, min((j + 1) * S, n) - j * S, seed,
                               O.derive_stream(seed, stream, j, O.SALT_SECTION), ctr0,
                               int(asg.counts[j]))
        for j in range(asg.n_sections)])
    got = ak.sectioned_sample(t, S, M, ak.RngStream(seed, stream, ctr0), rng="philox4x32")
    assert np.array_equal(got.cpu().numpy(), want)
    # pass-by-pass into a buffer offset by one element (odd 8-byte alignment)
    from paper_2106_12270_b200.sample import sectioned_sample_into
    counts = torch.from_numpy(asg.counts).to(DEV)
    offs = torch.from_numpy(np.concatenate([[0], np.cumsum(asg.counts)[:-1]])).to(DEV)
    buf = torch.full((M + 1,), -1, dtype=torch.int64, device=DEV)
    for first, count in ((0, 1), (1, 2), (3, asg.n_sections - 3)):
        sectioned_sample_into(t, S, counts, offs, first, count, ak.RngStream(seed, stream, ctr0),
                              buf[1:], 0, "philox4x32")
    assert np.array_equal(buf[1:].cpu().numpy(), want)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("rng_mode", ["reference", "philox4x32"])
def test_int32_outputs_equal_int64(dtype, rng_mode):
    """out_dtype=torch.int32 (opt-in, n <= 2^31-1) writes the int64 ids
    narrowed: both samplers, both RNG modes, f32/f64 tables, fast interior and
    generic edges (section size 2^12 pow2 and 1000 non-pow2), aligned and
    misaligned output offsets."""
    g = np.random.default_rng(32)
    w = g.pareto(1.1, 300_000) + 1e-6
    t = ak.psa_construct(ak.make_weight_set(torch.tensor(w, dtype=dtype)))
    for ctr in (0, 1, 2**33 + 5):
        a = ak.sample_batch(t, 100_003, ak.RngStream(5, 1, ctr), rng=rng_mode)
        b = ak.sample_batch(t, 100_003, ak.RngStream(5, 1, ctr), rng=rng_mode, out_dtype=torch.int32)
        assert b.dtype == torch.int32 and torch.equal(a, b.long())
        for S in (1 << 12, 1000):
            a = ak.sectioned_sample(t, S, 1_000_001, ak.RngStream(5, 2, ctr), rng=rng_mode)
            b = ak.sectioned_sample(t, S, 1_000_001, ak.RngStream(5, 2, ctr), rng=rng_mode,
                                    out_dtype=torch.int32)
            assert b.dtype == torch.int32 and torch.equal(a, b.long())
    # a misaligned int32 destination (odd element offset) through the pass API
    asg = ak.assign_sections(t.n, 1 << 12, 500_000, 9, 4)
    cd = torch.from_numpy(asg.counts).to(DEV)
    od = torch.from_numpy(np.concatenate([[0], np.cumsum(asg.counts)[:-1]])).to(DEV)
    from paper_2106_12270_b200.sample import sectioned_sample_into
    ref = torch.empty(500_000, dtype=torch.int64, device=DEV)
    sectioned_sample_into(t, asg.section_size, cd, od, 0, asg.n_sections, ak.RngStream(9, 4), ref, 0,
                          rng_mode, n_out=500_000)
    buf = torch.zeros(500_001, dtype=torch.int32, device=DEV)
    sectioned_sample_into(t, asg.section_size, cd, od, 0, asg.n_sections, ak.RngStream(9, 4), buf[1:], 0,
                          rng_mode, n_out=500_000)
    assert torch.equal(buf[1:].long(), ref) and buf[0].item() == 0
