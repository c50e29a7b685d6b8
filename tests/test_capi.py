"""The drop-in boundary: the C-ABI library loads, exports every symbol the
header declares, and its host-only entry points (section assignment, stream
derivation) agree with the oracle.  No device compute here (CPU suite)."""

import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2106_12270_b200 import _lib, errors

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "aliaskit_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ak_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(_lib.symbols()), set(declared) ^ set(_lib.symbols())


def test_version_and_row_sizes():
    L = _lib.lib()
    assert b"sm_100a" in L.ak_version()
    assert L.ak_row_bytes(_lib.F32) == 8 and L.ak_row_bytes(_lib.F64) == 16


def test_derive_stream_matches_oracle(rng):
    L = _lib.lib()
    for _ in range(100):
        a, b, c, d = (int(x) for x in rng.integers(0, 2**63, 4))
        assert L.ak_derive_stream(a, b, c, d) == O.derive_stream(a, b, c, d)


def test_assign_subtree_host_matches_golden(golden):
    from paper_2106_12270_b200.sample import assign_sections

    for i, (nr, S, M, seed, st) in enumerate(golden["asg_params"]):
        got = assign_sections(int(nr), int(S), int(M), int(seed), int(st)).counts
        assert np.array_equal(got, golden[f"asg_{i}"]), i


def test_assign_subtree_host_matches_oracle(rng):
    from paper_2106_12270_b200.sample import assign_sections, assign_subtree

    for _ in range(200):
        n = int(rng.integers(1, 5_000_000))
        S = int(rng.integers(1, n + 10))
        M = int(rng.integers(0, 10**10))
        seed = int(rng.integers(2**63))
        asg = assign_sections(n, S, M, seed, stream=5)
        assert int(asg.counts.sum()) == M
        assert np.array_equal(asg.counts, O.assign_sections(n, S, M, seed, 5))
        # any node of the recursion recomputes bit-exactly (sample.py:222-240)
        a, b = 0, asg.n_sections
        for _ in range(int(rng.integers(0, 12))):
            if b - a == 1:
                break
            mid = (a + b) // 2
            a, b = (a, mid) if rng.random() < 0.5 else (mid, b)
        sub = assign_subtree(n, S, seed, a, b, int(asg.counts[a:b].sum()), stream=5)
        assert np.array_equal(sub, asg.counts[a:b])


def test_assignment_edges():
    from paper_2106_12270_b200.sample import assign_sections

    assert assign_sections(100, 10, 0, seed=3).counts.tolist() == [0] * 10
    one = assign_sections(7, 99, 1234, seed=3)
    assert one.section_size == 7 and one.counts.tolist() == [1234]
    with pytest.raises(errors.InvalidSectionSize):
        assign_sections(10, 0, 5, seed=1)
    with pytest.raises(ValueError):
        assign_sections(0, 4, 5, seed=1)
    with pytest.raises(ValueError):
        assign_sections(10, 4, -1, seed=1)


def test_status_codes_map_to_reference_exceptions():
    cases = {
        errors.AK_ERR_EMPTY_INPUT: errors.EmptyInput,
        errors.AK_ERR_SIZE_MISMATCH: errors.SizeMismatch,
        errors.AK_ERR_INVALID_SECTION_COUNT: errors.InvalidSectionCount,
        errors.AK_ERR_UNSORTED_INPUT: errors.UnsortedInput,
        errors.AK_ERR_PLAN_INCONSISTENT: errors.PlanInconsistent,
        errors.AK_ERR_INVALID_SECTION_SIZE: errors.InvalidSectionSize,
        errors.AK_ERR_INDEX_OUT_OF_RANGE: errors.IndexOutOfRange,
    }
    for code, cls in cases.items():
        e = errors.from_status(code, "x")
        assert isinstance(e, cls) and isinstance(e, ValueError)
    e = errors.from_status(errors.AK_ERR_INVALID_WEIGHT, index=3, value=-1.0)
    assert isinstance(e, errors.InvalidWeight) and e.index == 3
    assert isinstance(errors.from_status(errors.AK_ERR_CUDA, "boom"), RuntimeError)
    # argument errors are detected on the host side of the ABI, before any launch
    L = _lib.lib()
    assert L.ak_assign_subtree(10, 0, 1, 0, 0, 1, 5, None) == errors.AK_ERR_INVALID_SECTION_SIZE
    assert L.ak_split_plan(None, 0, None, 0, None, 1, 5, 0, 1.0, None, None, None, 0, None) == \
        errors.AK_ERR_INVALID_SECTION_COUNT
    assert L.ak_build_psa(None, 1, 0, 1.0, None, None, 0, None) == errors.AK_ERR_EMPTY_INPUT


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2106_12270_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "liboracle" not in src, f
