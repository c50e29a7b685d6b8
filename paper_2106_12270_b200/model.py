"""Core domain types (mirror of aliaskit/model.py) with device storage.

``WeightSet`` keeps the weights in device memory (float64 like the reference,
or float32 for the device-native f32 path).  ``AliasTable`` keeps rows in the
device layout of include/aliaskit_b200.h — (f32 threshold, u32 alias) in 8
bytes or (f64 threshold, u64 alias) in 16 bytes, the ALT1 row — with
``tw``/``alias`` views and ``to_numpy()`` for the reference's SoA form
(tw f64[N], alias int64[N], model.py:66-77).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import EmptyInput, InvalidWeight, SizeMismatch
from .rng import MASK64, RngStream, uniform_py

__all__ = [
    "EmptyInput",
    "InvalidWeight",
    "SizeMismatch",
    "WeightSet",
    "AliasTable",
    "ValidationReport",
    "RngStream",
    "make_weight_set",
    "validate_table",
    "rng_uniform",
]


@dataclass(frozen=True)
class WeightSet:
    """Positive finite item weights (device tensor), their total, the count."""

    weights: torch.Tensor
    total: float
    n: int

    @property
    def average(self) -> float:
        """Bucket size W/N shared by every table row (model.py:60-63)."""
        return self.total / self.n

    @property
    def dtype(self) -> torch.dtype:
        return self.weights.dtype


@dataclass
class AliasTable:
    """N rows of (threshold, 1-based alias) plus N and W (model.py:66-85).

    ``rows`` is raw int64 storage: N words (f32 rows) or 2N words (f64 rows).
    """

    rows: torch.Tensor
    n: int
    total: float
    dtype: torch.dtype = torch.float64

    @property
    def average(self) -> float:
        return self.total / self.n

    @property
    def dtype_code(self) -> int:
        return _lib.dtype_code(self.dtype)

    @property
    def tw(self) -> torch.Tensor:
        if self.dtype == torch.float32:
            return self.rows.view(torch.float32)[0::2]
        return self.rows.view(torch.float64).view(self.n, 2)[:, 0]

    @property
    def alias(self) -> torch.Tensor:
        """1-based alias ids as int64 (a converted copy for f32 rows)."""
        if self.dtype == torch.float32:
            return self.rows.view(torch.int32)[1::2].to(torch.int64) & 0xFFFFFFFF
        return self.rows.view(self.n, 2)[:, 1]

    def tw_alias(self) -> tuple[torch.Tensor, torch.Tensor]:
        """(tw float64[N], alias int64[N]) on the device: the reference layout."""
        tw = torch.empty(self.n, dtype=torch.float64, device=self.rows.device)
        al = torch.empty(self.n, dtype=torch.int64, device=self.rows.device)
        with torch.cuda.device(self.rows.device):
            _lib.check(_lib.lib().ak_rows_to_soa(_lib.ptr(self.rows), self.dtype_code, self.n,
                                                 _lib.ptr(tw), _lib.ptr(al),
                                                 _lib.stream_ptr(self.rows.device)),
                       "rows_to_soa")
        return tw, al

    def to_numpy(self) -> tuple[np.ndarray, np.ndarray]:
        """(tw float64[N], alias int64[N]) on the host: the reference layout."""
        tw, al = self.tw_alias()
        return tw.cpu().numpy(), al.cpu().numpy()

    def count_unwritten(self) -> int:
        """Rows with alias 0 (the pack.py:275-276 check)."""
        import ctypes as C

        un = C.c_uint64(0)
        with torch.cuda.device(self.rows.device):
            _lib.check(_lib.lib().ak_count_unwritten(_lib.ptr(self.rows), self.dtype_code, self.n,
                                                     C.byref(un), _lib.stream_ptr(self.rows.device)),
                       "count_unwritten")
        return int(un.value)

    @property
    def rows_list(self) -> list[tuple[float, int]]:
        tw, al = self.to_numpy()
        return list(zip(tw.tolist(), al.tolist()))

    @classmethod
    def empty(cls, n: int, total: float, dtype=torch.float64, device=None) -> "AliasTable":
        dev = _lib.require_cuda(device)
        words = n * _lib.row_words(_lib.dtype_code(dtype))
        return cls(torch.empty(words, dtype=torch.int64, device=dev), int(n), float(total), dtype)

    @classmethod
    def blank(cls, n: int, total: float, dtype=torch.float64, device=None,
              fill_tw: float = -1.0) -> "AliasTable":
        """A table with every threshold = fill_tw and alias = 0 (unwritten)."""
        t = cls.empty(n, total, dtype, device)
        t.rows.zero_()
        t.tw.fill_(fill_tw)
        return t

    @classmethod
    def from_numpy(cls, tw, alias, n: int, total: float, dtype=torch.float64,
                   device=None) -> "AliasTable":
        dev = _lib.require_cuda(device)
        t = cls.empty(n, total, dtype, dev)
        twd = torch.as_tensor(np.ascontiguousarray(tw, dtype=np.float64), device=dev)
        ald = torch.as_tensor(np.ascontiguousarray(alias, dtype=np.int64), device=dev)
        with torch.cuda.device(dev):
            _lib.check(_lib.lib().ak_soa_to_rows(_lib.ptr(twd), _lib.ptr(ald), n, t.dtype_code,
                                                 _lib.ptr(t.rows), _lib.stream_ptr(dev)),
                       "soa_to_rows")
        return t


@dataclass(frozen=True)
class ValidationReport:
    ok: bool
    worst_rel_error: float
    worst_item: int  # 1-based


def _to_device_weights(weights, dtype, device) -> torch.Tensor:
    dev = _lib.require_cuda(device)
    if isinstance(weights, torch.Tensor):
        t = weights
        if dtype is None:
            dtype = t.dtype if t.dtype in (torch.float32, torch.float64) else torch.float64
        if t.dim() != 1:
            raise ValueError("weights must be one-dimensional")
        t = t.to(device=dev, dtype=dtype).contiguous()
    else:
        np_dtype = np.float64 if dtype in (None, torch.float64) else np.float32
        arr = np.ascontiguousarray(weights, dtype=np_dtype)
        if arr.ndim != 1:
            raise ValueError("weights must be one-dimensional")
        t = torch.from_numpy(arr).to(dev)
    if t.numel() and t.data_ptr() % 16:
        t = t.clone()
    return t


def make_weight_set(weights, dtype=None, device=None) -> WeightSet:
    """Validate weights and total them on the device (model.py:95-108).

    The total reproduces np.sum's pairwise tree exactly, so it is
    bit-identical to the reference's.  ``dtype`` defaults to float64 like the
    reference (float32 torch tensors keep float32: the f32 table path).
    """
    w = _to_device_weights(weights, dtype, device)
    n = int(w.numel())
    if n == 0:
        raise EmptyInput("at least one weight is required")
    dev = w.device
    L = _lib.lib()
    ws = _lib.workspace(L.ak_weights_workspace_bytes(n), dev, "weights")
    import ctypes as C

    total = C.c_double(0.0)
    bad = C.c_int64(-1)
    with torch.cuda.device(dev):
        st = L.ak_weights_validate_total(_lib.ptr(w), _lib.dtype_code(w.dtype), n,
                                         C.byref(total), C.byref(bad), _lib.ptr(ws), ws.numel(),
                                         _lib.stream_ptr(dev))
    if st == 2:
        i = int(bad.value)
        raise InvalidWeight(i + 1, float(w[i].item()))
    _lib.check(st, "make_weight_set")
    return WeightSet(weights=w, total=float(total.value), n=n)


def validate_table(t: AliasTable, w: WeightSet, tol: float = 1e-9,
                   row_tol: float = 1e-9) -> ValidationReport:
    """Row invariants and per-item mass conservation (model.py:111-144), on
    the device with compensated accumulation.  ``row_tol`` is the reference's
    fixed 1e-9 row bound (tw <= W/N * (1 + row_tol)); large-N checks scale it
    because W/N itself is rounded."""
    if t.n != w.n:
        raise SizeMismatch(f"table has {t.n} rows, weight set has {w.n}")
    import ctypes as C

    dev = t.rows.device
    L = _lib.lib()
    ws = _lib.workspace(L.ak_validate_workspace_bytes(t.n), dev, "validate")
    ok = C.c_int(0)
    worst = C.c_double(0.0)
    item = C.c_int64(0)
    with torch.cuda.device(dev):
        _lib.check(L.ak_validate_table(_lib.ptr(t.rows), t.dtype_code, t.n, _lib.ptr(w.weights),
                                       _lib.dtype_code(w.weights.dtype), w.average, float(row_tol),
                                       C.byref(ok), C.byref(worst), C.byref(item), _lib.ptr(ws),
                                       ws.numel(), _lib.stream_ptr(dev)),
                   "validate_table")
    werr = float(worst.value)
    return ValidationReport(ok=bool(ok.value) and werr <= tol and not math.isnan(werr),
                            worst_rel_error=werr, worst_item=int(item.value))


def rng_uniform(r: RngStream) -> float:
    """One uniform double in [0, 1) (host); advances the stream counter."""
    u = uniform_py(r.counter & MASK64, r.stream, r.seed)
    r.counter += 1
    return u
