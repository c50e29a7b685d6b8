"""Counter-based random numbers (mirror of aliaskit/rng.py).

Philox2x64-10, 10 rounds, multiplier 0xD2B74407B1CE6E93, Weyl 0x9E3779B97F4A7C15,
word 0 kept; u = (word0 >> 11) * 2^-53 (rng.py:21-69).  ``uniform_block``
fills device memory with a CUDA kernel (ak_fill_uniform) bit-identical to the
reference's ``uniform_block`` (rng.py:153-164); the scalar helpers stay on the
host (they serve single draws and recursion-node keys, rng.py:53-69, 167-169).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib

MASK64 = (1 << 64) - 1
_MULT = 0xD2B74407B1CE6E93
_WEYL = 0x9E3779B97F4A7C15
_ROUNDS = 10
_INV53 = 1.0 / 9007199254740992.0
SALT_STREAM = 0x6A09E667F3BCC909
SALT_NODE = 0xBB67AE8584CAA73B
SALT_SECTION = 0x3C6EF372FE94F82B


@dataclass
class RngStream:
    """Deterministic stream handle (rng.py:32-50): output depends only on
    (seed, stream, counter).  Single-owner; the counter is a Python int masked
    to 64 bits on use."""

    seed: int
    stream: int = 0
    counter: int = 0

    def __post_init__(self) -> None:
        self.seed = int(self.seed) & MASK64
        self.stream = int(self.stream) & MASK64
        self.counter = int(self.counter)

    def clone(self) -> "RngStream":
        return RngStream(self.seed, self.stream, self.counter)


def _philox_py(ctr: int, strm: int, key: int) -> int:
    """One 2x64 block (rng.py:53-65), host Python ints; first output word."""
    x0 = ctr & MASK64
    x1 = strm & MASK64
    k = key & MASK64
    for _ in range(_ROUNDS):
        prod = x0 * _MULT
        x0 = ((prod >> 64) & MASK64) ^ k ^ x1
        x1 = prod & MASK64
        k = (k + _WEYL) & MASK64
    return x0


def uniform_py(ctr: int, strm: int, key: int) -> float:
    return (_philox_py(ctr, strm, key) >> 11) * _INV53


def derive_stream(seed: int, stream: int, tag0: int, tag1: int) -> int:
    """Independent 64-bit stream id for a tagged purpose (rng.py:167-169)."""
    return int(_lib.lib().ak_derive_stream(seed & MASK64, stream & MASK64, tag0 & MASK64,
                                           tag1 & MASK64))


def uniform_block(r: RngStream, m: int, device=None) -> torch.Tensor:
    """m uniform doubles in [0, 1) from r's counter, on the device; advances r."""
    dev = _lib.require_cuda(device)
    m = int(m)
    if m < 0:
        raise ValueError("count must be non-negative")
    out = torch.empty(m, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().ak_fill_uniform(r.seed, r.stream, r.counter & MASK64, m,
                                              _lib.ptr(out), _lib.stream_ptr(dev)),
                   "uniform_block")
    r.counter += m
    return out
