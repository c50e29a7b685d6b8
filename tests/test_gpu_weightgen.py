"""Device weight generators against the reference's (weightgen.py:15-35),
restated with the oracle's uniform_block and numpy's stable argsort."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2106_12270_b200 as ak

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 1000, 1_000_003])
def test_gen_uniform_bit_exact(n):
    r = ak.RngStream(seed=7, stream=3, counter=11)
    ws = ak.gen_uniform(n, r)
    want = O.uniform_block(7, 3, 11, n)
    assert not np.any(want == 0.0)  # no redraw needed at these seeds
    assert np.array_equal(ws.weights.cpu().numpy(), want)
    assert r.counter == 11 + n
    w32 = ak.gen_uniform(n, ak.RngStream(seed=7, stream=3, counter=11), dtype=torch.float32)
    assert np.array_equal(w32.weights.cpu().numpy(), want.astype(np.float32))


@pytest.mark.parametrize("alpha", [1.0, 0.0, 0.5])
def test_gen_power_law(alpha):
    n = 200_003
    ws = ak.gen_power_law(n, alpha, ak.RngStream(seed=5))
    u = O.uniform_block(5, 0, 0, n)
    want = (np.arange(1, n + 1, dtype=np.float64) ** -np.float64(alpha))[np.argsort(u, kind="stable")]
    got = ws.weights.cpu().numpy()
    if alpha in (0.0, 1.0):
        assert np.array_equal(got, want)
    else:  # CUDA pow vs glibc pow: within one ulp
        assert np.max(np.abs(got - want) / want) <= 2.3e-16
