"""Multi-GPU sampling: table replication and communication-free sharding.

One process per GPU (torchrun), torch.distributed over NCCL for plumbing.
Sampling shards naturally:

* the table is replicated from rank 0 with one NCCL broadcast over NVLink
  (the only exchange of the whole job);
* naive sampling: rank g draws the counter block [ctr0 + g*ceil(M/G), ...) —
  exactly sample_batch's worker split (sample.py:133-145), so the
  concatenated output equals the single-GPU output;
* sectioned sampling: every rank recomputes the binomial section counts
  (host, bit-exact, < 1 ms for 61k sections) and takes a contiguous run of
  sections holding ~M/G draws; its output is that run's slice of the
  section-major single-GPU output.

Construction is replicas-only: it is reported at one GPU.

Verification shards too, with no host gather of samples
or tables:

* ``validate_table_sharded``: rank g validates the items of its range
  (ak_validate_table_range: every row is read, its own rows' invariants and
  its items' reconstructed mass are checked); three scalars are reduced;
* ``frequency_counts_allreduce``: the per-rank histograms are summed in
  place on the devices (all-reduce);
* ``chi_square_sharded``: each rank takes a bin shard of the summed
  histogram and forms chi_square_test's sums on its device
  (ak_chi2_partial); four doubles are reduced and the verdict formed exactly
  as stats.py:84-121 does.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

import ctypes as C
import math

from . import _lib
from .errors import DegenerateBins, SizeMismatch
from .model import AliasTable, ValidationReport, WeightSet
from .rng import RngStream
from .sample import assign_sections, sample_batch, sectioned_sample_into
from .stats import _chi2_quantile, frequency_counts


def broadcast_table(t: AliasTable | None, src: int = 0, group=None, device=None) -> AliasTable:
    """Replicate rank src's table on every rank (NCCL broadcast of the rows)."""
    rank = dist.get_rank(group)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    meta = torch.zeros(3, dtype=torch.float64, device=dev)
    if rank == src:
        meta[0] = float(t.n)
        meta[1] = t.total
        meta[2] = 1.0 if t.dtype == torch.float64 else 0.0
    dist.broadcast(meta, src, group=group)
    n, total, is64 = int(meta[0].item()), float(meta[1].item()), bool(meta[2].item())
    dtype = torch.float64 if is64 else torch.float32
    if rank != src:
        t = AliasTable.empty(n, total, dtype, dev)
    dist.broadcast(t.rows, src, group=group)
    return t


def naive_shard(m: int, rank: int, world: int) -> tuple[int, int]:
    """(offset, count) of rank's draws: ceil(m/world)-sized counter blocks."""
    step = -(-m // world) if m else 0
    off = min(rank * step, m)
    return off, min(step, m - off)


def sample_batch_shard(t: AliasTable, m: int, r: RngStream, rank: int, world: int,
                       rng: str = "reference", out: torch.Tensor | None = None) -> torch.Tensor:
    """This rank's slice of sample_batch(t, m, r); r is advanced by m on
    every rank (all ranks hold the same stream state)."""
    off, cnt = naive_shard(m, rank, world)
    sub = RngStream(r.seed, r.stream, r.counter + off)
    res = sample_batch(t, cnt, sub, rng=rng, out=out)
    r.counter += m
    return res


def section_shard(counts: np.ndarray, rank: int, world: int) -> tuple[int, int, int, int]:
    """Contiguous section run of rank holding ~total/world draws:
    (first section, section count, output offset, draws)."""
    cum = np.concatenate([[0], np.cumsum(counts)])
    total = int(cum[-1])
    lo_t = (total * rank) // world
    hi_t = (total * (rank + 1)) // world
    first = int(np.searchsorted(cum, lo_t, side="right")) - 1 if rank else 0
    last = int(np.searchsorted(cum, hi_t, side="right")) - 1 if rank < world - 1 else counts.size
    first = max(0, min(first, counts.size))
    last = max(first, min(last, counts.size))
    return first, last - first, int(cum[first]), int(cum[last] - cum[first])


class ShardedSectioned:
    """Precomputed per-rank plan for repeated sectioned sampling."""

    def __init__(self, t: AliasTable, S: int, M: int, r: RngStream, rank: int, world: int):
        asg = assign_sections(t.n, S, M, r.seed, r.stream)
        self.S = asg.section_size
        self.first, self.count, self.out_off, self.draws = section_shard(asg.counts, rank, world)
        dev = t.rows.device
        offs = np.concatenate([[0], np.cumsum(asg.counts)[:-1]])
        self.counts_d = torch.from_numpy(asg.counts).to(dev)
        self.offsets_d = torch.from_numpy(offs).to(dev)
        self.counts = asg.counts
        self.offsets = offs

    def run(self, t: AliasTable, r: RngStream, out: torch.Tensor, rng: str = "reference") -> None:
        sectioned_sample_into(t, self.S, self.counts_d, self.offsets_d, self.first, self.count, r,
                              out, self.out_off, rng, n_out=self.draws)


def _shard(n: int, rank: int, world: int) -> tuple[int, int]:
    return n * rank // world, n * (rank + 1) // world


def validate_table_sharded(t: AliasTable, w: WeightSet, tol: float = 1e-9, row_tol: float = 1e-9,
                           group=None) -> ValidationReport:
    """validate_table (model.py:111-144) split over the ranks of ``group``:
    the same report on every rank, equal to the single-GPU validate_table."""
    if t.n != w.n:
        raise SizeMismatch(f"table has {t.n} rows, weight set has {w.n}")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = _shard(t.n, rank, world)
    dev = t.rows.device
    L = _lib.lib()
    ws = _lib.workspace(L.ak_validate_workspace_bytes(hi - lo), dev, "validate")
    ok, worst, item = C.c_int(0), C.c_double(0.0), C.c_int64(0)
    with torch.cuda.device(dev):
        _lib.check(L.ak_validate_table_range(_lib.ptr(t.rows), t.dtype_code, t.n, lo, hi,
                                             _lib.ptr(w.weights), _lib.dtype_code(w.weights.dtype),
                                             w.average, float(row_tol), C.byref(ok), C.byref(worst),
                                             C.byref(item), _lib.ptr(ws), ws.numel(),
                                             _lib.stream_ptr(dev)), "validate_table_range")
    werr = float(worst.value)
    if math.isnan(werr):
        werr = math.inf
    red = torch.tensor([0.0 if ok.value else 1.0, werr], dtype=torch.float64, device=dev)
    dist.all_reduce(red, op=dist.ReduceOp.MAX, group=group)
    bad, gworst = bool(red[0].item()), float(red[1].item())
    # the first item attaining the global worst error (as the single-GPU scan)
    cand = torch.tensor([item.value if werr == gworst and hi > lo else 2**62], dtype=torch.int64, device=dev)
    dist.all_reduce(cand, op=dist.ReduceOp.MIN, group=group)
    return ValidationReport(ok=not bad and gworst <= tol, worst_rel_error=gworst,
                            worst_item=int(cand.item()))


def frequency_counts_allreduce(samples: torch.Tensor, n: int, group=None) -> torch.Tensor:
    """frequency_counts (stats.py:25-32) of the union of every rank's samples,
    summed on the devices (the histogram never leaves them)."""
    counts = frequency_counts(samples, n)
    dist.all_reduce(counts, group=group)
    return counts


def chi_square_sharded(counts: torch.Tensor, w: WeightSet, significance: float = 0.001,
                       group=None) -> tuple[float, int, bool]:
    """chi_square_test (stats.py:84-121) of a summed histogram against the
    table's probabilities w / W, each rank forming the sums of one bin shard
    on its device; the same (statistic, df, pass) on every rank."""
    if counts.numel() != w.n:
        raise ValueError("observed and expected_probs must be 1-d and equal length")
    if not 0.0 < significance < 1.0:
        raise ValueError("significance must lie in (0, 1)")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = _shard(w.n, rank, world)
    dev = counts.device
    draws = float(counts.sum().item()) if world == 1 else None
    if draws is None:
        tot = counts[lo:hi].sum().reshape(1).to(torch.float64)
        dist.all_reduce(tot, group=group)
        draws = float(tot.item())
    part = torch.empty(4, dtype=torch.float64, device=dev)
    c = counts[lo:hi].contiguous()
    wv = w.weights[lo:hi]
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().ak_chi2_partial(_lib.ptr(c), _lib.ptr(wv), _lib.dtype_code(wv.dtype),
                                              hi - lo, w.total, draws, _lib.ptr(part),
                                              _lib.stream_ptr(dev)), "chi2_partial")
    dist.all_reduce(part, group=group)
    stat, kept, po, pe = (float(x) for x in part.tolist())
    small = (w.n - int(round(kept))) > 0
    bins = int(round(kept)) + (1 if small else 0)
    if bins < 2:
        raise DegenerateBins("fewer than 2 bins after pooling")
    if small:
        if pe > 0.0:
            stat += (po - pe) ** 2 / pe
        elif po > 0.0:
            stat = math.inf
    df = bins - 1
    return stat, df, stat <= _chi2_quantile(1.0 - significance, df)
