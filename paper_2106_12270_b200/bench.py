"""Benchmark rows in the reference's CSV schema, measured on the device.

Mirrors ``aliaskit.bench`` (bench.py:25-203): the same configuration fields
and validation errors, the same row layout (``method,n,s,workers,param,
repetition,wall_time_ns,throughput_per_s``, per-repetition rows followed by a
``repetition=median`` row) and the same workloads (vose / psa / psa-plus
construction, baseline / sectioned sampling with ``RngStream(seed, 7)``), so a
CSV from this package sits next to the reference's own.  Rows carry
``backend=b200`` in ``param``; a wall time is the API call plus a device
synchronisation (the call's inputs and outputs stay in device memory).
"""

from __future__ import annotations

import statistics
import time
from dataclasses import dataclass

import torch

from .model import RngStream, WeightSet
from .pack import psa_construct, psa_plus_construct
from .sample import sample_batch, sectioned_sample
from .seqbuild import vose_construct
from .weightgen import gen_power_law, gen_uniform

CSV_HEADER = "method,n,s,workers,param,repetition,wall_time_ns,throughput_per_s"
METHODS = ("vose", "psa", "psa-plus")
SAMPLERS = ("baseline", "sectioned")
DISTS = ("uniform", "powerlaw")


class ConfigError(ValueError):
    """An invalid benchmark configuration (bench.py:32-33)."""


@dataclass
class BenchConfig:
    """Fields and defaults of the reference's BenchConfig (bench.py:36-54)."""

    n: int = 10**6
    dist: str = "uniform"
    alpha: float = 1.0
    methods: tuple = ()
    splits: int = 64
    workers: int = 1
    chunked: bool = False
    chunk_capacity: int = 1024
    samplers: tuple = ()
    samples: int = 10**6
    section_size: int = 2**14
    seed: int = 1
    repetitions: int = 5
    warmup: int = 1
    compare_backends: bool = False

    def validate(self) -> None:
        """The reference's checks, in its order (bench.py:56-76)."""
        problems = [
            (self.n < 1, "n must be at least 1"),
            (self.dist not in DISTS, f"unknown distribution {self.dist!r}"),
        ]
        for msg_bad, msg in problems:
            if msg_bad:
                raise ConfigError(msg)
        bad_m = [m for m in self.methods if m not in METHODS]
        if bad_m:
            raise ConfigError(f"unknown method {bad_m[0]!r}")
        bad_s = [s for s in self.samplers if s not in SAMPLERS]
        if bad_s:
            raise ConfigError(f"unknown sampler {bad_s[0]!r}")
        if not self.methods and not self.samplers:
            raise ConfigError("nothing to benchmark: no methods and no samplers")
        if self.repetitions < 5:
            raise ConfigError("medians need at least 5 repetitions")
        if self.warmup < 0:
            raise ConfigError("warmup must be non-negative")
        if self.splits < 1 or self.workers < 1:
            raise ConfigError("splits and workers must be positive")
        if self.samples < 1 or self.section_size < 1:
            raise ConfigError("samples and section_size must be positive")
        if self.chunk_capacity < 2:
            raise ConfigError("chunk_capacity must be at least 2")


def _params(pairs: dict) -> str:
    return ";".join(f"{k}={v}" for k, v in pairs.items())


def _rows(method, n, s, workers, params, times, work):
    base = {"method": method, "n": n, "s": s, "workers": workers, "param": _params(params)}
    out = [dict(base, repetition=i, wall_time_ns=t, throughput_per_s=work / (t * 1e-9))
           for i, t in enumerate(times)]
    med = statistics.median(times)
    out.append(dict(base, repetition="median", wall_time_ns=med, throughput_per_s=work / (med * 1e-9)))
    return out


def _timed(fn, reps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter_ns() - t0)
    return ts


def _weights(cfg: BenchConfig) -> WeightSet:
    r = RngStream(seed=cfg.seed)
    return gen_uniform(cfg.n, r) if cfg.dist == "uniform" else gen_power_law(cfg.n, cfg.alpha, r)


def bench_run(cfg: BenchConfig) -> list[dict]:
    """Time the configured constructions and samplers; CSV-ready rows
    (bench.py:135-194).  ``compare_backends`` has one backend to compare."""
    cfg.validate()
    w = _weights(cfg)
    params = {"dist": cfg.dist, "seed": cfg.seed}
    if cfg.dist == "powerlaw":
        params["alpha"] = cfg.alpha
    params["backend"] = "b200"
    rows: list[dict] = []
    build = {
        "vose": lambda: vose_construct(w),
        "psa": lambda: psa_construct(w, s=cfg.splits, workers=cfg.workers, chunked=cfg.chunked,
                                     chunk_capacity=cfg.chunk_capacity),
        "psa-plus": lambda: psa_plus_construct(w, s=cfg.splits, workers=cfg.workers),
    }
    for m in cfg.methods:
        p = dict(params)
        if m != "vose":
            p["chunked"] = int(cfg.chunked)
            if cfg.chunked:
                p["chunk_capacity"] = cfg.chunk_capacity
        times = _timed(build[m], cfg.repetitions, cfg.warmup)
        rows += _rows(m, cfg.n, cfg.splits if m != "vose" else 1, cfg.workers if m != "vose" else 1,
                      p, times, cfg.n)
    if cfg.samplers:
        t = vose_construct(w)
        for smp in cfg.samplers:
            p = dict(params, samples=cfg.samples)
            if smp == "sectioned":
                p["section_size"] = cfg.section_size
                fn = lambda: sectioned_sample(t, cfg.section_size, cfg.samples,  # noqa: E731
                                              RngStream(seed=cfg.seed, stream=7))
                s = cfg.section_size
            else:
                fn = lambda: sample_batch(t, cfg.samples, RngStream(seed=cfg.seed, stream=7),  # noqa: E731
                                          workers=cfg.workers)
                s = 0
            rows += _rows(smp, cfg.n, s, cfg.workers, p, _timed(fn, cfg.repetitions, cfg.warmup),
                          cfg.samples)
    return rows


def rows_to_csv(rows: list[dict]) -> str:
    """The reference's CSV text (bench.py:197-203)."""
    lines = [CSV_HEADER] + [
        f"{r['method']},{r['n']},{r['s']},{r['workers']},{r['param']},{r['repetition']},"
        f"{r['wall_time_ns']},{r['throughput_per_s']}" for r in rows]
    return "\n".join(lines) + "\n"
