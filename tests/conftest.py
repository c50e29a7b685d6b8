"""Shared fixtures.

Markers: ``gpu`` tests need a CUDA device and call the product through the C
ABI; everything else runs on the CPU (oracle pinning, host logic, library
exports).  GPU tests do not skip without a device: the product has no CPU
fallback, so they fail loudly instead.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"
ACCEPTANCE_LINES = []


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); calls the C-ABI library")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "golden.npz"))


@pytest.fixture(scope="session")
def hand():
    with open(os.path.join(GOLDEN, "hand_vectors.json")) as f:
        return json.load(f)


@pytest.fixture
def rng():
    return np.random.default_rng(0xA11A5)


@pytest.fixture(scope="session")
def reference():
    """The live reference package (build container only; skipped elsewhere)."""
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference not present (GPU box): golden fixtures cover it")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if REF_SRC not in sys.path:
        sys.path.append(REF_SRC)
    import aliaskit

    return aliaskit


@pytest.fixture
def acceptance():
    def record(line: str) -> None:
        ACCEPTANCE_LINES.append(line)
        print(line)

    return record


def pytest_terminal_summary(terminalreporter):
    if ACCEPTANCE_LINES:
        terminalreporter.section("acceptance criteria")
        for line in ACCEPTANCE_LINES:
            terminalreporter.write_line(line)


def random_weights(rng, n, kind):
    """tests_util.py:6-12 plus integer and shuffled-Zipf shapes."""
    if kind == 0:
        return rng.random(n) + 1e-9
    if kind == 1:
        return rng.pareto(1.1, n) + 1e-6
    if kind == 2:
        return np.exp(rng.normal(0.0, 3.0, n))
    if kind == 3:
        return rng.integers(1, 6, n).astype(np.float64)
    w = np.arange(1, n + 1, dtype=np.float64) ** -1.0
    rng.shuffle(w)
    return w


def golden_cases(golden):
    return list(range(len(golden["sizes"])))


def near_tie_margins(w, total, rows):
    """For 1-based rows whose alias differs from the reference, the distance
    (in units of avg) from the row's key to the nearest key of the other
    class, with every prefix summed exactly (math.fsum).  A decision taken
    inside the reference's own rounding noise (a near-tie) has a margin of
    ~1e-13; a real disagreement has a margin of order 1."""
    import math

    w = np.asarray(w, dtype=np.float64)
    n = w.size
    avg = total / n
    light = w <= avg
    li = np.nonzero(light)[0]
    hi = np.nonzero(~light)[0]
    # exact prefix keys, correctly rounded
    dl = [math.fsum([avg] * k + [-x for x in w[li[:k]]]) for k in range(len(li) + 1)]
    dh = [math.fsum([x for x in w[hi[: j + 1]]] + [-avg] * (j + 1)) for j in range(len(hi))]
    dl_arr, dh_arr = np.array(dl[:-1]), np.array(dh)
    pos_l = {int(i): k for k, i in enumerate(li)}
    pos_h = {int(i): j for j, i in enumerate(hi)}
    out = []
    for r in rows:
        i = int(r) - 1
        if i in pos_l:
            x = dl_arr[pos_l[i]]
            m = float(np.min(np.abs(dh_arr - x))) if dh_arr.size else math.inf
        else:
            y = dh_arr[pos_h[i]]
            m = float(np.min(np.abs(dl_arr - y))) if dl_arr.size else math.inf
        out.append(m / avg)
    return out
