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
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .model import AliasTable
from .rng import RngStream
from .sample import assign_sections, sample_batch, sectioned_sample_into


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
