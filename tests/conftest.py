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
