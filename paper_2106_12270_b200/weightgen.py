"""Seeded weight generators (mirror of aliaskit/weightgen.py) on the device.

Both consume the shared Philox stream exactly as the reference does, so the
weights are bit-identical to ``gen_uniform`` / ``gen_power_law`` for
alpha in {0, 1} (numpy evaluates x ** -1.0 as a correctly rounded
reciprocal, its scalar-power fast path) — other exponents go through CUDA's
pow, which may differ from glibc's in the last bit.  N = 1e9 is generated in milliseconds instead of the
reference's ~57 s on the host.
"""

from __future__ import annotations

import torch

from .model import WeightSet, make_weight_set
from .rng import RngStream, uniform_block


def gen_uniform(n: int, r: RngStream, dtype=torch.float64, device=None) -> WeightSet:
    """n draws from (0, 1); exact zeros are redrawn at fresh counters
    (weightgen.py:15-24).  dtype=float32 casts the f64 draws (the f32
    configs of the benchmark)."""
    if n < 1:
        raise ValueError("n must be at least 1")
    w = uniform_block(r, n, device)
    zeros = torch.nonzero(w == 0.0).flatten()
    while zeros.numel():
        w[zeros] = uniform_block(r, zeros.numel(), w.device)
        zeros = zeros[torch.nonzero(w[zeros] == 0.0).flatten()]
    if dtype == torch.float32:
        w32 = w.to(torch.float32)
        del w
        return make_weight_set(w32)
    return make_weight_set(w)


def gen_power_law(n: int, alpha: float, r: RngStream, dtype=torch.float64,
                  device=None) -> WeightSet:
    """Weights i**(-alpha), i = 1..n, in seeded shuffled order: the order is
    a stable argsort of n uniforms (weightgen.py:27-35)."""
    if n < 1:
        raise ValueError("n must be at least 1")
    if alpha < 0:
        raise ValueError("alpha must be non-negative")
    u = uniform_block(r, n, device)
    dev = u.device
    order = torch.sort(u, stable=True).indices
    del u
    i = order.to(torch.float64).add_(1.0)
    del order
    a = float(alpha)
    if a == 1.0:
        w = torch.reciprocal(i)
    elif a == 0.0:
        w = torch.ones_like(i)
    else:
        w = torch.pow(i, -a)
    del i
    if dtype == torch.float32:
        w = w.to(torch.float32)
    return make_weight_set(w)
