"""Property-based parity (hypothesis, as the reference's own tests do for
Vose, tests/test_seqbuild.py:67-77): arbitrary small weight vectors, the
fused device construction against the oracle's sequential Vose, and the
device samplers against the oracle's bit-exact samplers."""

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle as O
import paper_2106_12270_b200 as ak

pytestmark = pytest.mark.gpu

weights = st.lists(st.floats(min_value=1e-6, max_value=1e6, allow_nan=False, allow_infinity=False),
                   min_size=1, max_size=300)


@settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(weights)
def test_psa_equals_vose(ws_list):
    w = np.asarray(ws_list, dtype=np.float64)
    ws = ak.make_weight_set(w)
    _, tot = O.make_weight_set(w)
    assert ws.total == tot
    t = ak.psa_construct(ws)
    tw, al = t.to_numpy()
    ref = O.vose_construct(w, tot)
    diff = np.nonzero(al != ref.alias)[0]
    if diff.size:
        # only exact real ties may differ (decided by the reference's rounding)
        from conftest import near_tie_margins
        assert all(m < 1e-9 for m in near_tie_margins(w, tot, diff + 1)), diff
    assert ak.validate_table(t, ws).ok


@settings(max_examples=80, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(weights, st.integers(min_value=0, max_value=2**63 - 1), st.integers(min_value=1, max_value=64))
def test_samplers_bit_exact(ws_list, seed, S):
    w = np.asarray(ws_list, dtype=np.float64)
    _, tot = O.make_weight_set(w)
    ref = O.vose_construct(w, tot)
    t = ak.AliasTable.from_numpy(ref.tw, ref.alias, w.size, tot)
    rt = O.Table(ref.tw, ref.alias, w.size, tot)
    got = ak.sample_batch(t, 3000, ak.RngStream(seed, 2, 5)).cpu().numpy()
    assert np.array_equal(got, O.sample_batch(rt, 3000, seed, 2, 5))
    got = ak.sectioned_sample(t, S, 3000, ak.RngStream(seed, 4, 9)).cpu().numpy()
    assert np.array_equal(got, O.sectioned_sample(rt, S, 3000, seed, 4, 9))
