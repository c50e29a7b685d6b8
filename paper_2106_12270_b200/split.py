"""Section boundaries and batched search (mirror of aliaskit/split.py).

``compute_split_plan`` runs ak_split_plan: the boundary predicate
L[n_i - h] + H[h] <= n_i * W/N of split.py:52-88, either one binary search
per boundary or the paper's batched search (a CTA narrows the shared h-range
of a run of consecutive boundaries with 32-ary warp probes, stages the
prefix windows in shared memory and finishes every boundary there).  On the
same prefix arrays both are bit-identical to the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InvalidSectionCount, UnsortedInput
from .partition import LightHeavyPartition

__all__ = [
    "InvalidSectionCount",
    "UnsortedInput",
    "SplitPlan",
    "compute_split_plan",
    "binary_search_boundary",
    "partial_pary_search",
]


@dataclass
class SplitPlan:
    """Boundary records 0..s (split.py:36-49); device int64/f64 arrays."""

    s: int
    lcounts: torch.Tensor
    hcounts: torch.Tensor
    spills: torch.Tensor

    @property
    def boundaries(self) -> list[tuple[int, int, float]]:
        return list(zip(self.lcounts.cpu().tolist(), self.hcounts.cpu().tolist(),
                        self.spills.cpu().tolist()))


_METHODS = {"binary": 0, "batched": 1}


def compute_split_plan(p: LightHeavyPartition, s: int, method: str = "batched") -> SplitPlan:
    """Boundary states for s sections of floor-balanced item counts."""
    n = p.n
    s = int(s)
    if s < 1 or s > max(n, 1):
        raise InvalidSectionCount(f"s={s} not in [1, {max(n, 1)}]")
    dev = p.lprefix.device
    lc = torch.empty(s + 1, dtype=torch.int64, device=dev)
    hc = torch.empty(s + 1, dtype=torch.int64, device=dev)
    sp = torch.empty(s + 1, dtype=torch.float64, device=dev)
    hw = p.h_weight if p.h_weight.numel() else torch.zeros(1, dtype=p.dtype, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().ak_split_plan(
            _lib.ptr(p.lprefix), p.l_index.numel(), _lib.ptr(p.hprefix), p.h_index.numel(),
            _lib.ptr(hw), _lib.dtype_code(p.dtype), n, s, p.avg, _lib.ptr(lc), _lib.ptr(hc),
            _lib.ptr(sp), _METHODS[method], _lib.stream_ptr(dev)), "compute_split_plan")
    return SplitPlan(s=s, lcounts=lc, hcounts=hc, spills=sp)


def binary_search_boundary(p: LightHeavyPartition, n_i: int, cap: float):
    """Scalar replica of one boundary search (split.py:107-137), host side
    over the device prefix arrays; a cross-check helper."""
    nl = p.l_index.numel()
    nh = p.h_index.numel()
    if not 0 <= n_i <= nl + nh:
        raise ValueError(f"n_i={n_i} outside [0, {nl + nh}]")
    lpre = p.lprefix.cpu().numpy()
    hpre = p.hprefix.cpu().numpy()
    lo = max(0, n_i - nl)
    hi = min(n_i, nh)
    best = lo
    a, b = lo, hi
    while a <= b:
        mid = (a + b) >> 1
        if lpre[n_i - mid] + hpre[mid] <= cap:
            best = mid
            a = mid + 1
        else:
            b = mid - 1
    h = best
    l = n_i - h
    taken = cap - (float(lpre[l]) + float(hpre[h]))
    spill = 0.0
    if h < nh and taken > 0.0:
        spill = max(float(p.h_weight[h].item()) - taken, 0.0)
    return int(l), int(h), spill


def partial_pary_search(haystack, queries, p: int = 32) -> torch.Tensor:
    """Lower-bound indices of a sorted query batch in a sorted haystack
    (split.py:190-213), on the device: one warp runs the shared p-pivot
    contraction (_contract_range, split.py:157-187), then one thread per
    query binary-searches the contracted range.  Equal to searchsorted."""
    dev = _lib.require_cuda()
    hay = torch.as_tensor(haystack, dtype=torch.float64, device=dev).contiguous().reshape(-1)
    q = torch.as_tensor(queries, dtype=torch.float64, device=dev).contiguous().reshape(-1)
    if p < 3:
        raise ValueError("fanout p must be at least 3")
    out = torch.empty(q.numel(), dtype=torch.int64, device=dev)
    st = _lib.lib().ak_partial_pary_search(_lib.ptr(hay), hay.numel(), _lib.ptr(q), q.numel(),
                                           int(p), _lib.ptr(out), _lib.stream_ptr(dev))
    if st == 5:
        raise UnsortedInput("haystack or query batch is not sorted ascending")
    _lib.check(st, "partial_pary_search")
    return out
