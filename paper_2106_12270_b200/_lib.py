"""ctypes binding of libaliaskit_b200.so (the C ABI in include/aliaskit_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every call raises.  Status codes map 1:1 onto the
reference's exception classes (see errors.py).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import torch

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AK_LIB_PATH") or os.path.join(_HERE, "libaliaskit_b200.so")

F32, F64 = 0, 1
I32, I64 = 2, 3  # sample index dtypes (ak_sample_*_out)
RNG_REFERENCE, RNG_PHILOX4X32 = 0, 1
RNG_MODES = {"reference": RNG_REFERENCE, "philox4x32": RNG_PHILOX4X32}

_lib = None
_lock = threading.Lock()

u64, i64, dbl, vp, ci, sz = C.c_uint64, C.c_int64, C.c_double, C.c_void_p, C.c_int, C.c_size_t

_SIGS = {
    "ak_version": (C.c_char_p, []),
    "ak_last_error": (C.c_char_p, []),
    "ak_row_bytes": (sz, [ci]),
    "ak_fill_uniform": (ci, [u64, u64, u64, u64, vp, vp]),
    "ak_philox2x64": (ci, [vp, vp, vp, u64, vp, vp, vp]),
    "ak_philox4x32": (ci, [vp, vp, u64, vp, vp]),
    "ak_derive_stream": (u64, [u64, u64, u64, u64]),
    "ak_weights_workspace_bytes": (sz, [u64]),
    "ak_weights_validate_total": (ci, [vp, ci, u64, vp, vp, vp, sz, vp]),
    "ak_partition_workspace_bytes": (sz, [u64]),
    "ak_partition": (ci, [vp, ci, u64, dbl, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
    "ak_split_plan": (ci, [vp, u64, vp, u64, vp, ci, u64, u64, dbl, vp, vp, vp, ci, vp]),
    "ak_partial_pary_search": (ci, [vp, u64, vp, u64, C.c_uint32, vp, vp]),
    "ak_pack_sections": (ci, [vp, vp, u64, vp, vp, u64, ci, vp, vp, vp, u64, u64, u64, dbl, vp,
                              vp, C.c_uint32, vp]),
    "ak_build_workspace_bytes": (sz, [u64, ci]),
    "ak_build_psa": (ci, [vp, ci, u64, dbl, vp, vp, sz, vp]),
    "ak_build_stats": (ci, [vp, u64, vp, vp, vp, vp]),
    "ak_build_psa_avg": (ci, [vp, ci, u64, dbl, vp, vp, sz, vp]),
    "ak_prepack_workspace_bytes": (sz, [u64, C.c_uint32]),
    "ak_greedy_prepack": (ci, [vp, ci, u64, dbl, C.c_uint32, C.c_uint32, vp, vp, vp, vp, vp, vp,
                               sz, vp]),
    "ak_residual_scatter": (ci, [vp, vp, u64, dbl, ci, vp, vp]),
    "ak_residual_scatter_count": (ci, [vp, vp, u64, dbl, ci, vp, vp, vp]),
    "ak_build_psa_residual": (ci, [vp, u64, dbl, vp, ci, vp, vp, vp, sz, vp]),
    "ak_greedy_prepack_ex": (ci, [vp, ci, u64, dbl, C.c_uint32, C.c_uint32, ci, vp, vp, vp, vp, vp, vp,
                                  sz, vp]),
    "ak_sample_naive": (ci, [vp, ci, u64, dbl, u64, u64, u64, u64, u64, u64, vp, ci, vp]),
    "ak_sample_naive_out": (ci, [vp, ci, u64, dbl, u64, u64, u64, u64, u64, u64, vp, ci, ci, vp]),
    "ak_sample_from_uniforms": (ci, [vp, ci, u64, dbl, u64, u64, vp, u64, vp, vp]),
    "ak_num_sections": (u64, [u64, u64]),
    "ak_assign_subtree": (ci, [u64, u64, u64, u64, u64, u64, u64, vp]),
    "ak_sample_sectioned": (ci, [vp, ci, u64, dbl, u64, vp, vp, u64, u64, u64, u64, u64, vp, i64,
                                 ci, vp]),
    "ak_sample_sectioned_out": (ci, [vp, ci, u64, dbl, u64, vp, vp, u64, u64, u64, u64, u64, vp,
                                     ci, i64, ci, vp]),
    "ak_validate_workspace_bytes": (sz, [u64]),
    "ak_validate_table": (ci, [vp, ci, u64, vp, ci, dbl, dbl, vp, vp, vp, vp, sz, vp]),
    "ak_validate_table_range": (ci, [vp, ci, u64, u64, u64, vp, ci, dbl, dbl, vp, vp, vp, vp, sz, vp]),
    "ak_frequency_counts": (ci, [vp, u64, u64, vp, vp]),
    "ak_chi2_partial": (ci, [vp, vp, ci, u64, dbl, dbl, vp, vp]),
    "ak_rows_to_soa": (ci, [vp, ci, u64, vp, vp, vp]),
    "ak_soa_to_rows": (ci, [vp, vp, u64, ci, vp, vp]),
    "ak_count_unwritten": (ci, [vp, ci, u64, vp, vp]),
    "ak_rows_to_alt1": (ci, [vp, ci, u64, u64, u64, vp, vp]),
}


def lib():
    """Load the CUDA library (built in-tree by build.py); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2106_12270_b200.build` "
                "(there is no CPU fallback)"
            )
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def symbols() -> list[str]:
    return sorted(_SIGS)


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("aliaskit_b200 needs a CUDA device (no CPU fallback)")
    lib()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def check(status: int, what: str = "", index: int | None = None, value=None):
    if status == 0:
        return
    msg = what
    if status == errors.AK_ERR_CUDA:
        msg = f"{what}: {lib().ak_last_error().decode(errors='replace')}"
    raise errors.from_status(status, msg, index=index, value=value)


def workspace(nbytes: int, device: torch.device, tag: str = "default") -> torch.Tensor:
    """Device scratch of at least nbytes for ONE call, from torch's caching
    allocator.  The allocator is stream-ordered, so a buffer is only reused by
    work queued after this call's kernels on the same stream; two host threads
    (even on one shared stream) never receive the same live buffer, which a
    process-wide cache keyed by stream could not guarantee.  ``tag`` is kept
    for call-site readability."""
    del tag
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def aligned32(t: torch.Tensor) -> torch.Tensor:
    """t itself when its data is 32-byte aligned (the builder's 256-bit loads
    and stores need it), else a contiguous aligned copy."""
    if t.data_ptr() % 32 == 0 and t.is_contiguous():
        return t
    return t.contiguous().clone()


def dtype_code(t: torch.dtype) -> int:
    if t == torch.float32:
        return F32
    if t == torch.float64:
        return F64
    raise ValueError(f"unsupported weight dtype {t}: expected float32 or float64")


def row_words(dtype_c: int) -> int:
    """Row size in 8-byte words: f32 rows are 8 B, f64 rows 16 B."""
    return 1 if dtype_c == F32 else 2
