"""Drawing weighted samples (mirror of aliaskit/sample.py) on the device.

``sample_batch``: one Philox counter per draw and the bucket rule over the
whole table (ak_sample_naive, sample.py:73-149).  ``sectioned_sample``:
binomial section counts from the communication-free recursion (host C++,
bit-exact with sample.py:152-240), then one CTA per section draws from the
section's rows staged in shared memory (ak_sample_sectioned,
sample.py:243-267).  With ``rng="reference"`` (default) both are
bit-identical to the reference for the same RngStream; ``rng="philox4x32"``
is the GPU-native stream (two draws per Philox4x32-10 call), checked by
chi-square goodness of fit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InvalidSectionSize
from .model import AliasTable, rng_uniform
from .rng import MASK64, RngStream

__all__ = [
    "InvalidSectionSize",
    "SectionAssignment",
    "sample_one",
    "sample_batch",
    "sample_from_uniforms",
    "assign_sections",
    "assign_subtree",
    "sectioned_sample",
    "sectioned_sample_into",
]


@dataclass
class SectionAssignment:
    """Per-section sample counts plus their key material (sample.py:44-56)."""

    section_size: int
    counts: np.ndarray
    total: int
    seed: int
    stream: int

    @property
    def n_sections(self) -> int:
        return int(self.counts.size)


def _rng_code(rng: str) -> int:
    try:
        return _lib.RNG_MODES[rng]
    except KeyError:
        raise ValueError(f"unknown rng mode {rng!r}: expected one of {sorted(_lib.RNG_MODES)}")


def _check_out(out: torch.Tensor, need: int, dev: torch.device, what: str, n_rows: int = 0) -> None:
    """A caller-supplied output buffer must be a contiguous int64 (or, for
    tables of at most 2^31-1 rows, int32) tensor on the table's device with
    room for every draw the kernel writes through its raw pointer; anything
    else raises instead of writing out of bounds."""
    if not isinstance(out, torch.Tensor):
        raise TypeError(f"{what}: out must be a torch.Tensor")
    if out.dtype not in (torch.int64, torch.int32):
        raise ValueError(f"{what}: out must be int64 (or int32), got {out.dtype}")
    if out.dtype == torch.int32 and n_rows > 0x7FFFFFFF:
        raise ValueError(f"{what}: int32 output needs n <= 2^31-1, the table has {n_rows} rows")
    if out.device != dev:
        raise ValueError(f"{what}: out is on {out.device}, the table on {dev}")
    if not out.is_contiguous():
        raise ValueError(f"{what}: out must be contiguous")
    if out.numel() < need:
        raise ValueError(f"{what}: out holds {out.numel()} draws, {need} are written")


def _out_code(out: torch.Tensor) -> int:
    return _lib.I32 if out.dtype == torch.int32 else _lib.I64


def _new_out(m: int, dev: torch.device, out_dtype) -> torch.Tensor:
    dt = torch.int64 if out_dtype is None else out_dtype
    if dt not in (torch.int64, torch.int32):
        raise ValueError(f"out_dtype must be torch.int64 or torch.int32, got {dt}")
    return torch.empty(m, dtype=dt, device=dev)


def sample_one(t: AliasTable, r: RngStream) -> int:
    """One weighted draw (host uniform, one row read); advances r by one."""
    u = rng_uniform(r)
    x = u * t.n
    k0 = int(x)
    if k0 >= t.n:
        k0 = t.n - 1
    tw = float(t.tw[k0].item())
    if (x - k0) * t.average < tw:
        return k0 + 1
    return int(t.alias[k0].item())


def sample_batch(t: AliasTable, m: int, r: RngStream, workers: int = 1, rng: str = "reference",
                 out: torch.Tensor | None = None, out_dtype: torch.dtype | None = None) -> torch.Tensor:
    """m independent draws (1-based item ids, device int64); advances r by m.

    ``workers`` is accepted for API parity; the output never depends on it
    (sample.py:131-147), as on the reference.  ``out_dtype=torch.int32``
    (tables of at most 2^31-1 rows) writes the same ids as int32.
    """
    if m < 0:
        raise ValueError("sample count must be non-negative")
    dev = t.rows.device
    if out is None:
        out = _new_out(m, dev, out_dtype)
    _check_out(out, m, dev, "sample_batch", t.n)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().ak_sample_naive_out(
            _lib.ptr(t.rows), t.dtype_code, t.n, t.average, 0, t.n, r.seed, r.stream,
            r.counter & MASK64, m, _lib.ptr(out), _out_code(out), _rng_code(rng),
            _lib.stream_ptr(dev)), "sample_batch")
    r.counter += m
    return out


def sample_from_uniforms(t: AliasTable, u, lo: int = 0, span: int | None = None) -> torch.Tensor:
    """The bucket rule on explicit uniforms (tests/test_sample.py:20-25)."""
    dev = t.rows.device
    uu = torch.as_tensor(u, dtype=torch.float64, device=dev).contiguous()
    span = t.n if span is None else span
    out = torch.empty(uu.numel(), dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().ak_sample_from_uniforms(
            _lib.ptr(t.rows), t.dtype_code, t.n, t.average, lo, span, _lib.ptr(uu), uu.numel(),
            _lib.ptr(out), _lib.stream_ptr(dev)), "sample_from_uniforms")
    return out


def _num_sections(n_rows: int, S: int) -> tuple[int, int]:
    S = min(S, n_rows)
    return S, -(-n_rows // S)


def assign_subtree(n_rows: int, S: int, seed: int, a: int, b: int, m: int,
                   stream: int = 0) -> np.ndarray:
    """Counts for sections [a, b) given that subtree's total m
    (sample.py:222-240); bit-exact host C++ (ak_assign_subtree)."""
    if S < 1:
        raise InvalidSectionSize(f"section size {S} must be at least 1")
    S, ns = _num_sections(n_rows, S)
    if not 0 <= a < b <= ns:
        raise ValueError(f"subtree [{a}, {b}) outside 0..{ns}")
    counts = np.zeros(b - a, dtype=np.int64)
    _lib.check(_lib.lib().ak_assign_subtree(n_rows, S, seed & MASK64, stream & MASK64, a, b, m,
                                            counts.ctypes.data), "assign_subtree")
    return counts


def assign_sections(n_rows: int, S: int, M: int, seed: int, stream: int = 0) -> SectionAssignment:
    """Deterministic per-section sample counts summing exactly to M
    (sample.py:203-219)."""
    if n_rows < 1:
        raise ValueError("n_rows must be positive")
    if S < 1:
        raise InvalidSectionSize(f"section size {S} must be at least 1")
    if M < 0:
        raise ValueError("sample count must be non-negative")
    S_eff, ns = _num_sections(n_rows, S)
    counts = assign_subtree(n_rows, S_eff, seed, 0, ns, M, stream)
    return SectionAssignment(section_size=S_eff, counts=counts, total=M, seed=seed, stream=stream)


def sectioned_sample_into(t: AliasTable, S_eff: int, counts_d: torch.Tensor,
                          offsets_d: torch.Tensor, first: int, count: int, r: RngStream,
                          out: torch.Tensor, out_base: int, rng: str = "reference",
                          n_out: int | None = None) -> None:
    """Draw sections [first, first+count) into out[offsets - out_base ...]
    without touching r (the building block of sectioned_sample and of the
    multi-GPU / multi-pass drivers).

    ``out`` must hold offsets[last] + counts[last] - out_base draws; pass that
    number as ``n_out`` when the host already knows it (the multi-pass drivers
    do), otherwise it is read back from the device (one synchronisation)."""
    dev = t.rows.device
    if count <= 0:
        return
    for name, x in (("counts", counts_d), ("offsets", offsets_d)):
        if x.dtype != torch.int64 or x.device != dev or not x.is_contiguous():
            raise ValueError(f"sectioned_sample: {name} must be contiguous int64 on {dev}")
        if x.numel() < first + count:
            raise ValueError(f"sectioned_sample: {name} has {x.numel()} entries, "
                             f"sections [{first}, {first + count}) are drawn")
    if n_out is None:
        last = first + count - 1
        n_out = int((offsets_d[last] + counts_d[last]).item()) - out_base
    _check_out(out, n_out, dev, "sectioned_sample", t.n)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().ak_sample_sectioned_out(
            _lib.ptr(t.rows), t.dtype_code, t.n, t.average, S_eff, _lib.ptr(counts_d),
            _lib.ptr(offsets_d), first, count, r.seed, r.stream, r.counter & MASK64,
            _lib.ptr(out), _out_code(out), out_base, _rng_code(rng), _lib.stream_ptr(dev)),
            "sectioned_sample")


def sectioned_sample(t: AliasTable, S: int, M: int, r: RngStream, rng: str = "reference",
                     out: torch.Tensor | None = None,
                     out_dtype: torch.dtype | None = None) -> torch.Tensor:
    """M draws confined section by section to contiguous row ranges
    (sample.py:243-267); section-major output; advances r by M.
    ``out_dtype=torch.int32`` (n <= 2^31-1) writes the same ids as int32."""
    if M < 0:
        raise ValueError("sample count must be non-negative")
    asg = assign_sections(t.n, S, M, r.seed, r.stream)
    dev = t.rows.device
    if out is None:
        out = _new_out(M, dev, out_dtype)
    _check_out(out, M, dev, "sectioned_sample", t.n)
    if M:
        counts = torch.from_numpy(asg.counts).to(dev)
        offsets = torch.from_numpy(np.concatenate([[0], np.cumsum(asg.counts)[:-1]])).to(dev)
        sectioned_sample_into(t, asg.section_size, counts, offsets, 0, asg.n_sections, r, out, 0,
                              rng, n_out=M)
    r.counter += M
    return out
