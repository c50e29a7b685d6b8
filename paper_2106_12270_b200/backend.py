"""Kernel backend registry (mirror of aliaskit/backend.py).

The reference selects between numba-compiled and numpy kernels
(backend.py:16-73).  This package has exactly one backend — hand-written
sm_100a CUDA behind the C ABI of include/aliaskit_b200.h — and no CPU
fallback: asking for anything else raises, and a missing library or device
raises on first use.
"""

from __future__ import annotations

BACKENDS = ("cuda",)
HAVE_NUMBA = False
_active = "cuda"


def active_backend() -> str:
    return _active


def set_backend(name: str) -> None:
    if name not in BACKENDS:
        raise ValueError(f"unknown backend {name!r}: expected one of {BACKENDS}")


def using_numba() -> bool:
    return False
