"""The multi-GPU code path executed: two ranks (gloo, both on cuda:0 — a
single-GPU box cannot host two NCCL ranks on one device) run the product's
broadcast_table, sample_batch_shard, ShardedSectioned, validate_table_sharded,
frequency_counts_allreduce and chi_square_sharded; the parent checks that the
shards reassemble the single-GPU outputs bit for bit and that the sharded
verification equals the single-GPU one.  Under torchrun with NCCL on an 8-GPU
node the same functions run unchanged (bench.py --gpus N)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2106_12270_b200 as ak
    from paper_2106_12270_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 300_001
    t = None
    ws = ak.gen_power_law(n, 0.8, ak.RngStream(seed=3), dtype=torch.float64)
    if rank == 0:
        t = ak.psa_construct(ws)
    t = D.broadcast_table(t, 0)  # the NCCL broadcast of the rows in production
    out = {"rows": t.rows.cpu().numpy()}
    # naive sampling: counter blocks
    r = ak.RngStream(9, 2, 5)
    out["naive"] = D.sample_batch_shard(t, 1_000_003, r, rank, world).cpu().numpy()
    out["naive_counter"] = r.counter
    # sectioned sampling: communication-free section runs
    S, M = 1 << 12, 2_000_000
    plan = D.ShardedSectioned(t, S, M, ak.RngStream(9, 4, 7), rank, world)
    piece = torch.empty(plan.draws, dtype=torch.int64, device="cuda")
    plan.run(t, ak.RngStream(9, 4, 7), piece, rng="philox4x32")
    out["sec"] = (plan.out_off, piece.cpu().numpy())
    # sharded verification
    rep = D.validate_table_sharded(t, ws, tol=1e-9)
    out["validate"] = (rep.ok, rep.worst_rel_error, rep.worst_item)
    counts = D.frequency_counts_allreduce(piece, n)
    out["counts"] = counts.cpu().numpy()
    out["chi2"] = D.chi_square_sharded(counts, ws)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_reassemble_single_gpu_outputs():
    import paper_2106_12270_b200 as ak

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = 300_001
    ws = ak.gen_power_law(n, 0.8, ak.RngStream(seed=3), dtype=torch.float64)
    t = ak.psa_construct(ws)
    rows = t.rows.cpu().numpy()
    for rk in range(world):
        assert np.array_equal(res[rk]["rows"], rows)  # the broadcast replica
    naive = ak.sample_batch(t, 1_000_003, ak.RngStream(9, 2, 5)).cpu().numpy()
    assert np.array_equal(np.concatenate([res[0]["naive"], res[1]["naive"]]), naive)
    assert res[0]["naive_counter"] == res[1]["naive_counter"] == 5 + 1_000_003
    sec = ak.sectioned_sample(t, 1 << 12, 2_000_000, ak.RngStream(9, 4, 7), rng="philox4x32").cpu().numpy()
    parts = sorted((res[rk]["sec"] for rk in range(world)), key=lambda x: x[0])
    assert np.array_equal(np.concatenate([p[1] for p in parts]), sec)
    # verification: the sharded reports equal the single-GPU ones
    single = ak.validate_table(t, ws, tol=1e-9)
    for rk in range(world):
        ok, worst, item = res[rk]["validate"]
        assert ok == single.ok
        assert worst == pytest.approx(single.worst_rel_error, rel=1e-6, abs=1e-18)
    counts = ak.frequency_counts(torch.from_numpy(sec).cuda(), n).cpu().numpy()
    for rk in range(world):
        assert np.array_equal(res[rk]["counts"], counts)
        stat, df, passed = res[rk]["chi2"]
        sref, dref, pref = ak.chi_square_test(counts, ws.weights.cpu().numpy() / ws.total)
        assert df == dref and passed == pref
        assert stat == pytest.approx(sref, rel=1e-9)
