"""bench.py keeps the driver contract: one JSON line with the required keys.
The reference arm runs on the CPU (oracle port); our arm needs a GPU."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                       text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--n", "1e5",
             "--ref-samples", "1e5"], 300)
    assert KEYS <= set(d) and d["impl"] == "reference"
    c = d["config"]
    assert c["n"] == 100_000 and c["same_config"]["build"] is True and c["nproc"] >= 1
    assert c["sectioned_samples_per_s"] > 0 and c["naive_samples_per_s"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["value"] > 0 and d["higher_is_better"] is True


@pytest.mark.gpu
def test_our_arm_contract():
    d = run(["--steps", "1", "--warmup", "1", "--n", "1e6", "--samples", "1e8", "--no-cpu",
             "--e2e-samples", "1e7", "--e2e-steps", "1"], 600)
    assert KEYS <= set(d)
    for k in ("roofline", "clocks", "gpu_launches", "build", "build_psa_plus", "e2e_int32",
              "c5_float64", "dtypes"):
        assert k in d
    assert d["e2e_int32"]["d2h_bytes_per_step"] * 2 == d["e2e"]["d2h_bytes_per_step"]
    assert 0 < d["c5_float64"]["build"]["roofline"]["frac"] < 1.5
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["scaling"] == "weak"


@pytest.mark.gpu
def test_reference_arm_weights_match_gpu_arm():
    """bench.py --impl reference regenerates the GPU arm's weights on the host
    (gen_uniform(N, RngStream(seed=1)) cast to float32, upcast to float64):
    bit-identical to the device generator's."""
    import numpy as np
    import torch

    sys.path.insert(0, ROOT)
    import bench
    import paper_2106_12270_b200 as ak

    n = 1_000_003
    host = bench.reference_weights(n)
    dev = ak.gen_uniform(n, ak.RngStream(seed=1), dtype=torch.float32).weights.double().cpu().numpy()
    assert np.array_equal(host, dev)


@pytest.mark.gpu
def test_two_rank_bench_line_under_torchrun():
    """The driver's N>1 launch (torch.distributed.run, one process per rank)
    end to end: barriers, max-over-ranks timing, the whole-job value, the
    e2e split across ranks and the broadcast step variant.  Two ranks share
    one GPU over gloo (NCCL needs a GPU per rank), so this checks the
    multi-rank code path, not scaling."""
    for extra in ([], ["--broadcast"]):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(29600 + len(extra)),
               os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo",
               "--items", "1e7", "--samples", "2e8", "--steps", "2", "--warmup", "3", "--no-cpu",
               "--e2e-samples", "4e7", "--e2e-steps", "1"] + extra
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-3000:]
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
        d = json.loads(lines[0])
        assert KEYS <= set(d) and d["n_gpus"] == 2 and d["scaling"] == "weak"
        assert d["config"]["samples_total"] == 2 * d["config"]["samples_per_gpu"]
        assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["table_broadcast"]["bytes"] > 0
        assert ("broadcast" in d["step_variant"]) == bool(extra)


def test_bench_options_parse_under_torchrun_spelling():
    """--items (the spelling torchrun's own parser leaves alone) and --n set
    the same value; --dist-backend accepts nccl and gloo (CPU-only check)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True,
                       text=True, timeout=120, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "--items" in r.stdout and "--n" in r.stdout and "--dist-backend" in r.stdout
    assert "gloo" in r.stdout
