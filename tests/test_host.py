"""Host-side logic: multi-GPU sharding (with a world_size-2 gloo run on the
CPU), chi-square verification harness, weight-set argument handling."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2106_12270_b200 import distributed as D
from paper_2106_12270_b200 import errors
from paper_2106_12270_b200.stats import _chi2_quantile, _probit, chi_square_test


def test_naive_shard_matches_worker_split():
    for m in (0, 1, 5, 1000, 10**9 + 7):
        for world in (1, 2, 3, 4, 8):
            parts = [D.naive_shard(m, g, world) for g in range(world)]
            assert sum(c for _, c in parts) == m
            off = 0
            for o, c in parts:
                assert o == off or c == 0
                off += c


def test_section_shard_partitions_output(rng):
    for _ in range(50):
        ns = int(rng.integers(1, 5000))
        counts = rng.integers(0, 1000, ns)
        for world in (1, 2, 4, 8):
            runs = [D.section_shard(counts, g, world) for g in range(world)]
            nxt, out = 0, 0
            for first, cnt, off, draws in runs:
                assert first == nxt and off == out
                assert draws == int(counts[first:first + cnt].sum())
                nxt, out = first + cnt, out + draws
            assert nxt == ns and out == int(counts.sum())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    """One rank: the PRODUCT's host-side sharding (naive_shard, the host C++
    binomial assignment behind assign_sections, section_shard) plans its
    share; its draws come from the oracle sampler here, as the product's
    samplers need a GPU (tests/test_gpu_multi.py runs the same plan on the
    device through the product end to end)."""
    import paper_2106_12270_b200 as ak

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(11)
    w = rng.random(777) + 0.01
    _, tot = O.make_weight_set(w)
    t = O.vose_construct(w, tot)
    # naive: each rank draws its counter block
    m = 10_001
    off, cnt = D.naive_shard(m, rank, world)
    part = O.sample_batch(t, cnt, seed=42, stream=3, counter=100 + off)
    # sectioned: each rank recomputes the counts (product host C++) and draws
    # its section run, section by section with the reference's per-section
    # streams
    S, M = 16, 20_000
    asg = ak.assign_sections(t.n, S, M, 42, 5)
    first, count, out_off, draws = D.section_shard(asg.counts, rank, world)
    pieces = []
    for j in range(first, first + count):
        lo, hi = j * S, min((j + 1) * S, t.n)
        strm = O.derive_stream(42, 5, j, O.SALT_SECTION)
        pieces.append(O.rule(t.tw, t.alias, t.total / t.n,
                             O.uniform_block(42, strm, 9, int(asg.counts[j])), lo, hi - lo))
    mine = np.concatenate(pieces) if pieces else np.empty(0, dtype=np.int64)
    assert mine.size == draws
    # the product's host counts equal the oracle's on every rank
    assert np.array_equal(asg.counts, O.assign_sections(t.n, S, M, 42, 5))
    parts = [None] * world
    dist.all_gather_object(parts, (part.tolist(), out_off, mine.tolist()))
    if rank == 0:
        q.put(parts)
    dist.destroy_process_group()


def test_gloo_world2_shards_reassemble_single_process_output():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(11)
    w = rng.random(777) + 0.01
    _, tot = O.make_weight_set(w)
    t = O.vose_construct(w, tot)
    naive = np.concatenate([np.array(p[0], dtype=np.int64) for p in parts])
    assert np.array_equal(naive, O.sample_batch(t, 10_001, 42, 3, 100))
    sec = np.concatenate([np.array(p[2], dtype=np.int64) for p in sorted(parts, key=lambda x: x[1])])
    assert np.array_equal(sec, O.sectioned_sample(t, 16, 20_000, 42, 5, 9))


def test_chi_square_harness_hand_cases():
    stat, df, ok = chi_square_test([10.0, 0.0], [0.5, 0.5])
    assert stat == pytest.approx(10.0) and df == 1 and ok
    stat, df, ok = chi_square_test([1000, 0, 0, 0], [0.25] * 4)
    assert not ok and stat == pytest.approx(3000.0)
    stat, df, ok = chi_square_test([499, 499, 1, 1], [0.499, 0.499, 0.001, 0.001])
    assert df == 2 and ok
    with pytest.raises(errors.DegenerateBins):
        chi_square_test([2, 2], [0.5, 0.5])
    assert _probit(0.5) == 0.0
    assert _chi2_quantile(0.999, 1) == pytest.approx(10.83, rel=0.15)


def test_chi_square_matches_reference(reference):
    rng = np.random.default_rng(3)
    for _ in range(50):
        k = int(rng.integers(2, 300))
        probs = rng.random(k)
        probs /= probs.sum()
        if abs(probs.sum() - 1.0) > 1e-12:
            continue
        obs = rng.multinomial(int(rng.integers(10, 10**6)), probs)
        assert chi_square_test(obs, probs) == reference.chi_square_test(obs, probs)


# ---- CSV bench rows (aliaskit.bench schema) -------------------------------

def test_bench_config_validation_mirrors_reference():
    from paper_2106_12270_b200.bench import BenchConfig, ConfigError
    cases = [
        (dict(n=0, methods=("psa",)), "n must be at least 1"),
        (dict(dist="zipf", methods=("psa",)), "unknown distribution"),
        (dict(methods=("alias",)), "unknown method"),
        (dict(samplers=("fast",)), "unknown sampler"),
        (dict(), "nothing to benchmark"),
        (dict(methods=("psa",), repetitions=4), "at least 5 repetitions"),
        (dict(methods=("psa",), warmup=-1), "warmup"),
        (dict(methods=("psa",), splits=0), "splits and workers"),
        (dict(samplers=("baseline",), samples=0), "samples and section_size"),
        (dict(methods=("psa",), chunk_capacity=1), "chunk_capacity"),
    ]
    for kw, msg in cases:
        with pytest.raises(ConfigError, match=msg):
            BenchConfig(**kw).validate()
    BenchConfig(methods=("vose", "psa", "psa-plus"), samplers=("baseline", "sectioned")).validate()


def test_rows_to_csv_schema():
    from paper_2106_12270_b200.bench import CSV_HEADER, _rows, rows_to_csv
    rows = _rows("psa", 10, 64, 1, {"dist": "uniform", "seed": 1, "backend": "b200"}, [10, 30, 20, 40, 50], 10)
    csv = rows_to_csv(rows).splitlines()
    assert csv[0] == CSV_HEADER == "method,n,s,workers,param,repetition,wall_time_ns,throughput_per_s"
    assert len(csv) == 7 and csv[-1].startswith("psa,10,64,1,dist=uniform;seed=1;backend=b200,median,30,")
