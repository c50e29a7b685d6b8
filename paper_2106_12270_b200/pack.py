"""Bucket writing and construction (mirror of aliaskit/pack.py).

``pack_section`` / ``chunked_pack_section`` run the reference's per-section
sweep on the device (ak_pack_sections; bit-identical to pack.py:30-159 on
the same partition and plan).  ``psa_construct`` runs the fused B200
pipeline (ak_build_psa): classify + decoupled-look-back scan,
coarse boundary merge, tile-owner pack.  Its alias indices are those of the
sequential construction; thresholds are exact double-double prefix
differences rounded once, so they agree with the reference's to within its
own f64 drift.
"""

from __future__ import annotations

import torch

from . import _lib
from .errors import PlanInconsistent
from .model import AliasTable, WeightSet
from .partition import LightHeavyPartition
from .split import SplitPlan

__all__ = [
    "PlanInconsistent",
    "pack_section",
    "chunked_pack_section",
    "psa_construct",
    "psa_plus_construct",
    "build_table",
]


def _check_plan(p: LightHeavyPartition, plan: SplitPlan) -> None:
    """pack.py:166-174"""
    s = plan.s
    lc, hc = plan.lcounts, plan.hcounts
    if tuple(lc.shape) != (s + 1,) or tuple(hc.shape) != (s + 1,) or tuple(plan.spills.shape) != (s + 1,):
        raise PlanInconsistent("plan arrays must have s+1 boundary records")
    ends = torch.stack([lc[0], hc[0], lc[s], hc[s]]).cpu().tolist()
    if ends[0] != 0 or ends[1] != 0 or ends[2] != p.l_index.numel() or ends[3] != p.h_index.numel():
        raise PlanInconsistent("plan endpoints do not close over the partition")
    if s > 0 and (bool((lc[1:] < lc[:-1]).any()) or bool((hc[1:] < hc[:-1]).any())):
        raise PlanInconsistent("boundary counts must be non-decreasing")


def _pack(p, plan, i0, i1, out: AliasTable, cap: int):
    dev = out.rows.device
    if out.dtype != p.dtype:
        raise ValueError(f"table dtype {out.dtype} does not match partition dtype {p.dtype}")
    spills = torch.empty(i1 - i0 + 1, dtype=torch.float64, device=dev)
    dummy_i = torch.zeros(1, dtype=torch.int64, device=dev)
    dummy_w = torch.zeros(1, dtype=p.dtype, device=dev)
    li = p.l_index if p.l_index.numel() else dummy_i
    lw = p.l_weight if p.l_weight.numel() else dummy_w
    hi = p.h_index if p.h_index.numel() else dummy_i
    hw = p.h_weight if p.h_weight.numel() else dummy_w
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().ak_pack_sections(
            _lib.ptr(li), _lib.ptr(lw), p.l_index.numel(), _lib.ptr(hi), _lib.ptr(hw),
            p.h_index.numel(), _lib.dtype_code(p.dtype), _lib.ptr(plan.lcounts),
            _lib.ptr(plan.hcounts), _lib.ptr(plan.spills), plan.s, i0, i1, p.avg,
            _lib.ptr(out.rows), _lib.ptr(spills), int(cap), _lib.stream_ptr(dev)), "pack")
    return spills


def pack_section(p: LightHeavyPartition, plan: SplitPlan, i: int, out: AliasTable) -> float:
    """Write section i's buckets into ``out``; returns the outgoing residual
    (pack.py:201-213)."""
    _check_plan(p, plan)
    if not 1 <= i <= plan.s:
        raise PlanInconsistent(f"section {i} outside 1..{plan.s}")
    return float(_pack(p, plan, i, i, out, 0)[0].item())


def chunked_pack_section(p: LightHeavyPartition, plan: SplitPlan, i: int, chunk_capacity: int,
                         out: AliasTable) -> float:
    """Staged variant (pack.py:216-232): a warp copies light and heavy chunks
    coalesced into shared memory; same bucket output."""
    _check_plan(p, plan)
    if not 1 <= i <= plan.s:
        raise PlanInconsistent(f"section {i} outside 1..{plan.s}")
    if chunk_capacity < 2:
        raise ValueError("chunk_capacity must be at least 2")
    return float(_pack(p, plan, i, i, out, int(chunk_capacity))[0].item())


def pack_all(p: LightHeavyPartition, plan: SplitPlan, out: AliasTable, chunk_capacity: int = 0):
    """Every section of a plan in one launch (one thread or warp each)."""
    _check_plan(p, plan)
    return _pack(p, plan, 1, plan.s, out, chunk_capacity)


def build_table(w: WeightSet, out: AliasTable | None = None) -> AliasTable:
    """The fused device construction (ak_build_psa) into ``out`` (allocated
    when None).  Asynchronous on the current stream."""
    dev = w.weights.device
    dt = w.weights.dtype
    if out is None:
        out = AliasTable.empty(w.n, w.total, dt, dev)
    L = _lib.lib()
    ws = _lib.workspace(L.ak_build_workspace_bytes(w.n, _lib.dtype_code(dt)), dev, "build")
    wt = _lib.aligned32(w.weights)  # held until the call is queued
    with torch.cuda.device(dev):
        _lib.check(L.ak_build_psa(_lib.ptr(wt), _lib.dtype_code(dt), w.n, w.total,
                                  _lib.ptr(out.rows), _lib.ptr(ws), ws.numel(),
                                  _lib.stream_ptr(dev)), "build_psa")
    return out


def psa_construct(w: WeightSet, s: int = 64, workers: int = 1, chunked: bool = False,
                  chunk_capacity: int = 1024) -> AliasTable:
    """Split construction (pack.py:255-277) as the fused device pipeline.

    ``s``, ``workers``, ``chunked`` and ``chunk_capacity`` are validated as in
    the reference; the device pipeline sections the work by 512-item chunks
    itself, and (like the reference, whose output is section- and
    worker-invariant up to rounding) its table does not depend on them.
    """
    if s < 1:
        raise ValueError("section count must be positive")
    if workers < 1:
        raise ValueError("worker count must be positive")
    if chunked and chunk_capacity < 2:
        raise ValueError("chunk_capacity must be at least 2")
    return build_table(w)


def psa_plus_construct(w: WeightSet, s: int = 64, workers: int = 1, block_size: int = 4096,
                       threshold: int = 8) -> AliasTable:
    """Split construction preceded by the block-local pairing pass
    (pack.py:280-305)."""
    if s < 1:
        raise ValueError("section count must be positive")
    if workers < 1:
        raise ValueError("worker count must be positive")
    from .prepack import psa_plus_construct as _ppc

    return _ppc(w, s, block_size, threshold)
