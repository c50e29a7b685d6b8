"""PSA+ (mirror of aliaskit's greedy_prepack, partition.py:233-282, and
psa_plus_construct, pack.py:280-305) on the device.

``greedy_prepack`` runs ak_greedy_prepack: every block of ``block_size``
items pairs its lights and heavies (when it holds at least
``min_pair_threshold`` of each) in the block-local sequential order and
forwards the leftovers in item order.  ``psa_plus_construct`` then builds the
residual with the fused PSA pipeline at the global average, its rows written
straight into the table through the residual's item ids
(ak_build_psa_residual).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .errors import PlanInconsistent
from .model import AliasTable, WeightSet
from .partition import LightHeavyPartition, PrepackResult


MAX_BLOCK = 11000  # 20 bytes of shared memory per item of a block (ak_prepack.cu)


def _prepack(w: WeightSet, block_size: int, threshold: int, clear_rows: bool = True):
    if block_size < 2:
        raise ValueError("block_size must be at least 2")
    if threshold < 1:
        raise ValueError("min_pair_threshold must be at least 1")
    if block_size > MAX_BLOCK:
        # a block's lights, heavies and keys live in one CTA's shared memory
        raise ValueError(f"block_size {block_size} exceeds the device limit {MAX_BLOCK}")
    dev = w.weights.device
    n = w.n
    L = _lib.lib()
    t = AliasTable.empty(n, w.total, w.weights.dtype, dev)
    res_idx = torch.empty(n, dtype=torch.int64, device=dev)
    res_w = torch.empty(n, dtype=torch.float64, device=dev)
    ws = _lib.workspace(L.ak_prepack_workspace_bytes(n, block_size), dev, "prepack")
    nres = C.c_uint64(0)
    nw = C.c_uint64(0)
    with torch.cuda.device(dev):
        _lib.check(L.ak_greedy_prepack_ex(_lib.ptr(w.weights), _lib.dtype_code(w.weights.dtype), n,
                                          w.average, block_size, threshold, int(clear_rows),
                                          _lib.ptr(t.rows), _lib.ptr(res_idx), _lib.ptr(res_w),
                                          C.byref(nres), C.byref(nw), _lib.ptr(ws), ws.numel(),
                                          _lib.stream_ptr(dev)), "greedy_prepack")
    k = int(nres.value)
    return t, res_idx[:k], res_w[:k], int(nw.value)


def greedy_prepack(w: WeightSet, block_size: int = 4096,
                   min_pair_threshold: int = 8) -> PrepackResult:
    """Pair lights and heavies block-locally, forwarding leftovers
    (partition.py:233-282)."""
    t, res_idx, res_w, nwritten = _prepack(w, block_size, min_pair_threshold)
    tw, alias = t.tw_alias()
    light = res_w <= w.average
    li, hi = res_idx[light], res_idx[~light]
    lw, hw = res_w[light], res_w[~light]
    zero = torch.zeros(1, dtype=torch.float64, device=res_w.device)
    residual = LightHeavyPartition(
        l_index=li, l_weight=lw, h_index=hi, h_weight=hw,
        lprefix=torch.cat([zero, torch.cumsum(lw, 0)]),
        hprefix=torch.cat([zero, torch.cumsum(hw, 0)]),
        avg=w.average)
    return PrepackResult(tw=tw, alias=alias, written=alias != 0, residual=residual,
                         handled_fraction=nwritten / w.n)


def psa_plus_construct(w: WeightSet, s: int = 64, block_size: int = 4096,
                       threshold: int = 8) -> AliasTable:
    """Split construction preceded by the block-local pairing pass
    (pack.py:280-305); the residual goes through the fused PSA pipeline with
    the global average (the section count ``s`` does not change the table).

    The reference's closing check, every bucket written (pack.py:303-304),
    is made from counts instead of a pass over the table: the prepack counts
    the rows it pairs, the residual build the rows it writes through res_idx,
    and the two sets are disjoint by construction — so the table is not
    cleared first and not re-read afterwards."""
    t, res_idx, res_w, nwritten = _prepack(w, block_size, threshold, clear_rows=False)
    k = res_idx.numel()
    dev = w.weights.device
    L = _lib.lib()
    if k:
        # the residual built with the global average, its rows written
        # straight into the table through res_idx (no intermediate table)
        ws = _lib.workspace(L.ak_build_workspace_bytes(k, _lib.F64), dev, "build")
        res_w = _lib.aligned32(res_w)
        scattered = C.c_uint64(0)
        with torch.cuda.device(dev):
            _lib.check(L.ak_build_psa_residual(_lib.ptr(res_w), k, w.average, _lib.ptr(res_idx),
                                               t.dtype_code, _lib.ptr(t.rows), C.byref(scattered),
                                               _lib.ptr(ws), ws.numel(), _lib.stream_ptr(dev)),
                       "psa_plus residual build")
        nwritten += int(scattered.value)
    if nwritten != w.n:
        raise PlanInconsistent("pack left buckets unwritten")
    return t
