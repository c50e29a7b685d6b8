"""ALT1 / WTS1 files (io.py:18-71): device tables round-trip bit-exactly, the
bytes are the reference's format, and corrupt files are rejected the way the
reference rejects them (tests/test_io.py, tests/test_cli.py:116-136)."""

import struct

import numpy as np
import pytest
import torch

import paper_2106_12270_b200 as ak
from paper_2106_12270_b200.io import FormatError

pytestmark = pytest.mark.gpu


def reference_bytes(tw, alias, n, total):
    rows = np.empty(n, dtype=[("tw", "<f8"), ("alias", "<u8")])
    rows["tw"] = tw
    rows["alias"] = alias
    return b"ALT1" + struct.pack("<Q", n) + struct.pack("<d", total) + rows.tobytes()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_table_round_trip_and_format(tmp_path, rng, dtype):
    w = rng.pareto(1.1, 5000) + 1e-6
    ws = ak.make_weight_set(torch.from_numpy(w.astype(np.float32) if dtype == torch.float32 else w).cuda())
    t = ak.psa_construct(ws)
    p = tmp_path / "t.alt"
    ak.save_table(t, p)
    tw, al = t.to_numpy()
    assert p.read_bytes() == reference_bytes(tw, al, t.n, t.total)
    u = ak.load_table(p)
    tw2, al2 = u.to_numpy()
    assert np.array_equal(tw2, tw) and np.array_equal(al2, al) and u.total == t.total


def test_weights_round_trip(tmp_path, rng):
    w = rng.random(1000) + 0.1
    p = tmp_path / "w.wts"
    ak.save_weights(w, p)
    ws = ak.load_weights(p)
    assert np.array_equal(ws.weights.cpu().numpy(), w) and ws.total == ak.make_weight_set(w).total


def test_corrupt_files_rejected(tmp_path):
    t = ak.psa_construct(ak.make_weight_set([3.0, 1.0, 2.0, 2.0]))
    p = tmp_path / "t.alt"
    ak.save_table(t, p)
    good = p.read_bytes()
    for bad in (b"XLT1" + good[4:], good[:-3], good + b"\0" * 16):
        p.write_bytes(bad)
        with pytest.raises(FormatError):
            ak.load_table(p)
    # an alias outside 1..n (bit flip in the last row's alias)
    b = bytearray(good)
    b[-8:] = struct.pack("<Q", 99)
    p.write_bytes(bytes(b))
    with pytest.raises(FormatError):
        ak.load_table(p)
    q = tmp_path / "w.wts"
    q.write_bytes(b"WTS1" + struct.pack("<Q", 3) + b"\0" * 8)
    with pytest.raises(FormatError):
        ak.load_weights(q)


def test_bench_rows_on_device():
    """aliaskit.bench-schema rows measured on the device (bench.py:135-203)."""
    from paper_2106_12270_b200.bench import BenchConfig, bench_run, rows_to_csv
    cfg = BenchConfig(n=20_000, methods=("vose", "psa", "psa-plus"), samplers=("baseline", "sectioned"),
                      samples=50_000, section_size=1024, repetitions=5, warmup=1)
    rows = bench_run(cfg)
    assert len(rows) == 5 * 6
    med = [r for r in rows if r["repetition"] == "median"]
    assert [r["method"] for r in med] == ["vose", "psa", "psa-plus", "baseline", "sectioned"]
    assert all(r["throughput_per_s"] > 0 and "backend=b200" in r["param"] for r in rows)
    assert [r["s"] for r in med] == [1, 64, 64, 0, 1024]
    assert rows_to_csv(rows).count("\n") == len(rows) + 1
