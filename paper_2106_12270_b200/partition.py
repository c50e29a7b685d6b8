"""Light/heavy partitioning (mirror of aliaskit/partition.py) on the device.

``partition_items`` runs ak_partition: stable classification (w <= W/N is
light) in ascending item order with co-located weights and exclusive
prefix sums, computed as exact double-double sums rounded to f64 (the
reference uses a Neumaier-compensated running sum, partition.py:62-75; both
are within an ulp or two of the exact prefix).  ``greedy_prepack`` is the
PSA+ block pairing (partition.py:134-282).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .model import WeightSet


@dataclass
class LightHeavyPartition:
    """Device index/weight arrays for both classes plus exclusive prefixes
    (partition.py:21-48).  Indices are 1-based int64; weights keep the
    weight-set dtype; prefixes are float64 of length |class|+1."""

    l_index: torch.Tensor
    l_weight: torch.Tensor
    h_index: torch.Tensor
    h_weight: torch.Tensor
    lprefix: torch.Tensor
    hprefix: torch.Tensor
    avg: float

    @property
    def n(self) -> int:
        return int(self.l_index.numel() + self.h_index.numel())

    @property
    def dtype(self) -> torch.dtype:
        return self.l_weight.dtype

    @property
    def l(self) -> list[tuple[int, float]]:
        return list(zip(self.l_index.cpu().tolist(), self.l_weight.double().cpu().tolist()))

    @property
    def h(self) -> list[tuple[int, float]]:
        return list(zip(self.h_index.cpu().tolist(), self.h_weight.double().cpu().tolist()))


@dataclass
class PrepackResult:
    """Partially written table plus the partition of leftover items
    (partition.py:51-59)."""

    tw: torch.Tensor
    alias: torch.Tensor
    written: torch.Tensor
    residual: LightHeavyPartition
    handled_fraction: float


def partition_items(w: WeightSet) -> LightHeavyPartition:
    """Split items into light/heavy arrays (ascending) with prefix sums."""
    dev = w.weights.device
    n = w.n
    dt = w.weights.dtype
    L = _lib.lib()
    l_idx = torch.empty(n, dtype=torch.int64, device=dev)
    h_idx = torch.empty(n, dtype=torch.int64, device=dev)
    l_w = torch.empty(n, dtype=dt, device=dev)
    h_w = torch.empty(n, dtype=dt, device=dev)
    lpre = torch.empty(n + 1, dtype=torch.float64, device=dev)
    hpre = torch.empty(n + 1, dtype=torch.float64, device=dev)
    ws = _lib.workspace(L.ak_partition_workspace_bytes(n), dev, "partition")
    nl = C.c_uint64(0)
    nh = C.c_uint64(0)
    with torch.cuda.device(dev):
        _lib.check(L.ak_partition(_lib.ptr(w.weights), _lib.dtype_code(dt), n, w.average,
                                  _lib.ptr(l_idx), _lib.ptr(l_w), _lib.ptr(h_idx), _lib.ptr(h_w),
                                  _lib.ptr(lpre), _lib.ptr(hpre), C.byref(nl), C.byref(nh),
                                  _lib.ptr(ws), ws.numel(), _lib.stream_ptr(dev)),
                   "partition_items")
    a, b = int(nl.value), int(nh.value)
    # exact-length views of the n-sized outputs (no copies; the unused tails
    # stay allocated with them)
    return LightHeavyPartition(
        l_index=l_idx[:a], l_weight=l_w[:a], h_index=h_idx[:b], h_weight=h_w[:b],
        lprefix=lpre[: a + 1], hprefix=hpre[: b + 1], avg=w.average,
    )


def greedy_prepack(w: WeightSet, block_size: int = 4096,
                   min_pair_threshold: int = 8) -> PrepackResult:
    """Pair lights and heavies block-locally, forwarding leftovers
    (partition.py:233-282)."""
    from .prepack import greedy_prepack as _gp

    return _gp(w, block_size, min_pair_threshold)
