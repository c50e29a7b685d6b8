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


_STREAM_SCRIPT = r"""
import os, sys, torch
sys.path.insert(0, os.environ["AK_ROOT"])
import paper_2106_12270_b200 as ak

def hwm():
    for line in open("/proc/self/status"):
        if line.startswith("VmHWM"):
            return int(line.split()[1]) * 1024
dt = torch.float32 if sys.argv[1] == "f32" else torch.float64
n, path = int(sys.argv[2]), sys.argv[3]
ws = ak.gen_uniform(n, ak.RngStream(seed=5), dtype=dt)
t = ak.psa_construct(ws)
torch.cuda.synchronize()
base = hwm()
ak.save_table(t, path)
ak.save_weights(ws, path + ".w")
u = ak.load_table(path)
v = ak.load_weights(path + ".w")
peak = hwm() - base
same_rows = torch.equal(u.rows.view(torch.float64)[0::2].to(t.rows.device),
                        (t.rows.view(torch.float32)[0::2].double() if dt == torch.float32
                         else t.rows.view(torch.float64)[0::2]))
same_alias = torch.equal(u.rows[1::2], (t.rows.view(torch.int32)[1::2].long() if dt == torch.float32
                                       else t.rows[1::2]))
same_w = torch.equal(v.weights, ws.weights.double()) and v.total == ak.make_weight_set(ws.weights.double()).total
print(peak, os.path.getsize(path), int(same_rows), int(same_alias), int(same_w))
"""


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_streaming_round_trip_1e8_bounded_host_memory(tmp_path, dtype):
    """N = 1e8: the table (1.6 GB ALT1) and weights round-trip bit-exactly
    through the streamed writers/readers, and the process's host memory grows
    by about the two pinned chunk buffers (2 x 64 MB), not by the file size."""
    import os
    import subprocess
    import sys

    n = 10**8
    path = str(tmp_path / "t.alt")
    env = dict(os.environ, AK_ROOT=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    out = subprocess.run([sys.executable, "-c", _STREAM_SCRIPT, dtype, str(n), path], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    peak, size, same_rows, same_alias, same_w = (int(x) for x in out.stdout.split()[-5:])
    assert size == 20 + 16 * n
    assert same_rows and same_alias and same_w
    assert peak < 512 * 2**20, f"host memory grew by {peak / 2**20:.0f} MiB"
