"""CPU oracle for the alias-table path — TEST INFRASTRUCTURE ONLY.

ctypes/numpy wrapper over ``liboracle.so`` (built from ``aliaskit_oracle.c``
by ``oracle/Makefile``), a plain-C restatement of the reference package
``aliaskit`` (/root/reference/pkg/src/aliaskit).  Each wrapper names the
reference function it restates.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` leg may import this
module; the product package never does (and fails loudly without its own
CUDA library instead of falling back here).

Pinned by tests/test_oracle.py against the Random123 Philox KATs, the
reference's hand vectors and golden fixtures generated from the reference
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

MASK64 = (1 << 64) - 1
SALT_STREAM = 0x6A09E667F3BCC909
SALT_NODE = 0xBB67AE8584CAA73B
SALT_SECTION = 0x3C6EF372FE94F82B


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "aliaskit_oracle.c")
        ):
            build()
        L = C.CDLL(_LIB_PATH)
        u64, i64, dbl, vp = C.c_uint64, C.c_int64, C.c_double, C.c_void_p
        L.ako_philox2x64_w0.restype = u64
        L.ako_philox2x64_w0.argtypes = [u64, u64, u64]
        L.ako_philox2x64_both.argtypes = [u64, u64, u64, vp, vp]
        L.ako_uniform.restype = dbl
        L.ako_uniform.argtypes = [u64, u64, u64]
        L.ako_derive_stream.restype = u64
        L.ako_derive_stream.argtypes = [u64, u64, u64, u64]
        L.ako_fill_uniform.argtypes = [u64, u64, u64, u64, vp]
        L.ako_pairwise_sum.restype = dbl
        L.ako_pairwise_sum.argtypes = [vp, u64]
        L.ako_make_weight_set.restype = C.c_int
        L.ako_make_weight_set.argtypes = [vp, u64, vp, vp]
        L.ako_validate_table.argtypes = [vp, vp, vp, u64, dbl, vp, vp, vp]
        L.ako_vose.argtypes = [vp, u64, dbl, vp, vp]
        L.ako_vose_quad.argtypes = [vp, u64, dbl, vp, vp]
        L.ako_vose_fixed.argtypes = [vp, u64, dbl, vp, vp]
        L.ako_vose_fixed_margins.argtypes = [vp, u64, dbl, vp, u64, vp]
        L.ako_exclusive_prefix.argtypes = [vp, u64, vp]
        L.ako_partition.restype = u64
        L.ako_partition.argtypes = [vp, u64, dbl, vp, vp, vp, vp, vp, vp, vp]
        L.ako_split_plan.argtypes = [vp, u64, vp, u64, vp, u64, u64, dbl, vp, vp, vp]
        L.ako_contract_range.argtypes = [vp, u64, dbl, dbl, i64, vp, vp, vp]
        L.ako_partial_pary_search.argtypes = [vp, u64, vp, u64, i64, vp]
        L.ako_pack_range.argtypes = [vp, vp, vp, vp, u64, vp, vp, vp, i64, i64, dbl, vp, vp, vp]
        L.ako_chunked_pack_range.argtypes = [vp, vp, vp, vp, u64, vp, vp, vp, i64, i64, dbl, i64,
                                             vp, vp, vp]
        L.ako_psa_construct.restype = C.c_int
        L.ako_psa_construct.argtypes = [vp, u64, dbl, u64, C.c_int, C.c_int, i64, vp, vp]
        L.ako_greedy_prepack.restype = u64
        L.ako_greedy_prepack.argtypes = [vp, u64, dbl, i64, i64, vp, vp, vp, vp, vp, vp, vp]
        L.ako_fill_samples.argtypes = [vp, vp, dbl, i64, i64, u64, u64, u64, vp, u64]
        L.ako_rule_from_uniforms.argtypes = [vp, vp, dbl, i64, i64, vp, u64, vp]
        L.ako_sample_batch.argtypes = [vp, vp, u64, dbl, u64, u64, u64, u64, C.c_int, vp]
        L.ako_probit.restype = dbl
        L.ako_probit.argtypes = [dbl]
        L.ako_binom_draw.restype = i64
        L.ako_binom_draw.argtypes = [i64, dbl, dbl]
        L.ako_assign_subtree.argtypes = [u64, u64, u64, u64, i64, i64, i64, vp]
        L.ako_sectioned_sample.argtypes = [vp, vp, u64, dbl, u64, vp, u64, u64, u64, u64, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


# ---- rng.py ---------------------------------------------------------------

def philox_w0(ctr: int, strm: int, key: int) -> int:
    """_philox_py (rng.py:53-65)."""
    return int(lib().ako_philox2x64_w0(ctr & MASK64, strm & MASK64, key & MASK64))


def philox_both(ctr: int, strm: int, key: int) -> tuple[int, int]:
    out = np.zeros(2, dtype=np.uint64)
    lib().ako_philox2x64_both(ctr & MASK64, strm & MASK64, key & MASK64,
                              _p(out[:1]), out[1:].ctypes.data_as(C.c_void_p))
    return int(out[0]), int(out[1])


def uniform(ctr: int, strm: int, key: int) -> float:
    """uniform_py (rng.py:68-69)."""
    return float(lib().ako_uniform(ctr & MASK64, strm & MASK64, key & MASK64))


def derive_stream(seed: int, stream: int, tag0: int, tag1: int) -> int:
    """derive_stream (rng.py:167-169)."""
    return int(lib().ako_derive_stream(seed & MASK64, stream & MASK64, tag0 & MASK64, tag1 & MASK64))


def uniform_block(seed: int, stream: int, ctr0: int, m: int) -> np.ndarray:
    """uniform_block (rng.py:153-164) without the counter advance."""
    out = np.empty(m, dtype=np.float64)
    lib().ako_fill_uniform(seed & MASK64, stream & MASK64, ctr0 & MASK64, m, _p(out))
    return out


# ---- model.py -------------------------------------------------------------

@dataclass
class Table:
    tw: np.ndarray
    alias: np.ndarray
    n: int
    total: float

    @property
    def average(self) -> float:
        return self.total / self.n


def pairwise_sum(a) -> float:
    a = _f64(a)
    return float(lib().ako_pairwise_sum(_p(a), a.size))


def make_weight_set(w):
    """make_weight_set (model.py:95-108): (weights f64, total) or raises."""
    a = _f64(w)
    tot = np.zeros(1)
    bad = np.zeros(1, dtype=np.int64)
    rc = lib().ako_make_weight_set(_p(a), a.size, _p(tot), _p(bad))
    if rc == 1:
        raise ValueError("EmptyInput")
    if rc == 2:
        raise ValueError(f"InvalidWeight {int(bad[0]) + 1}")
    return a, float(tot[0])


def validate_table(tw, alias, w, total):
    """validate_table (model.py:111-144) → (ok_rows, worst_rel, worst_item)."""
    tw, alias, w = _f64(tw), _i64(alias), _f64(w)
    ok = np.zeros(1, dtype=np.int32)
    worst = np.zeros(1)
    wi = np.zeros(1, dtype=np.int64)
    lib().ako_validate_table(_p(tw), _p(alias), _p(w), w.size, total, _p(ok), _p(worst), _p(wi))
    return bool(ok[0]), float(worst[0]), int(wi[0])


# ---- seqbuild.py / partition.py / split.py / pack.py -----------------------

def vose_construct(w, total: float) -> Table:
    """vose_construct (seqbuild.py:64-70)."""
    w = _f64(w)
    n = w.size
    tw = np.zeros(n)
    alias = np.zeros(n, dtype=np.int64)
    lib().ako_vose(_p(w), n, total / n, _p(tw), _p(alias))
    return Table(tw, alias, n, total)


def vose_construct_quad(w, total: float) -> Table:
    """Vose with a binary128 residual (diagnostic: the reference's decisions
    without its f64 drift)."""
    w = _f64(w)
    n = w.size
    tw = np.zeros(n)
    alias = np.zeros(n, dtype=np.int64)
    lib().ako_vose_quad(_p(w), n, total / n, _p(tw), _p(alias))
    return Table(tw, alias, n, total)


def vose_construct_fixed(w, total: float) -> Table:
    """Vose in the device builder's exact fixed-point arithmetic (diagnostic:
    the table psa_construct must reproduce bit for bit; see ako_vose_fixed)."""
    w = _f64(w)
    n = w.size
    tw = np.zeros(n)
    alias = np.zeros(n, dtype=np.int64)
    lib().ako_vose_fixed(_p(w), n, total / n, _p(tw), _p(alias))
    return Table(tw, alias, n, total)


def decision_margins(w, total: float, rows) -> np.ndarray:
    """Exact decision margins (units of avg) of 1-based ``rows`` in Vose's
    order (ako_vose_fixed_margins): how far each row's alias/threshold
    decision is from flipping.  Certifies near-ties at any N in O(N)."""
    w = _f64(w)
    rows = np.ascontiguousarray(np.sort(np.asarray(rows, dtype=np.int64)))
    out = np.empty(rows.size)
    lib().ako_vose_fixed_margins(_p(w), w.size, total / w.size, _p(rows), rows.size, _p(out))
    return out


def partition_items(w, total: float):
    """partition_items (partition.py:106-131) → dict of arrays."""
    w = _f64(w)
    n = w.size
    l_idx = np.empty(n, dtype=np.int64)
    h_idx = np.empty(n, dtype=np.int64)
    l_w = np.empty(n)
    h_w = np.empty(n)
    lpre = np.empty(n + 1)
    hpre = np.empty(n + 1)
    nh = np.zeros(1, dtype=np.uint64)
    avg = total / n
    nl = int(lib().ako_partition(_p(w), n, avg, _p(l_idx), _p(l_w), _p(h_idx), _p(h_w),
                                 _p(lpre), _p(hpre), _p(nh)))
    nh = int(nh[0])
    return dict(l_index=l_idx[:nl].copy(), l_weight=l_w[:nl].copy(), h_index=h_idx[:nh].copy(),
                h_weight=h_w[:nh].copy(), lprefix=lpre[: nl + 1].copy(),
                hprefix=hpre[: nh + 1].copy(), avg=avg)


def exclusive_prefix(v) -> np.ndarray:
    v = _f64(v)
    out = np.empty(v.size + 1)
    lib().ako_exclusive_prefix(_p(v), v.size, _p(out))
    return out


def compute_split_plan(lprefix, hprefix, h_weight, n_total: int, s: int, avg: float):
    """_fill_plan_kernel (split.py:52-88) → (lcounts, hcounts, spills)."""
    lpre, hpre, hw = _f64(lprefix), _f64(hprefix), _f64(h_weight)
    lc = np.empty(s + 1, dtype=np.int64)
    hc = np.empty(s + 1, dtype=np.int64)
    sp = np.empty(s + 1)
    lib().ako_split_plan(_p(lpre), lpre.size - 1, _p(hpre), hpre.size - 1, _p(hw), n_total, s,
                         avg, _p(lc), _p(hc), _p(sp))
    return lc, hc, sp


def contract_range(hay, qmin, qmax, p):
    hay = _f64(hay)
    a = np.zeros(1, dtype=np.int64)
    b = np.zeros(1, dtype=np.int64)
    r = np.zeros(1, dtype=np.int64)
    lib().ako_contract_range(_p(hay), hay.size, qmin, qmax, p, _p(a), _p(b), _p(r))
    return int(a[0]), int(b[0]), int(r[0])


def partial_pary_search(hay, q, p=32) -> np.ndarray:
    """partial_pary_search (split.py:190-213) sans validation."""
    hay, q = _f64(hay), _f64(q)
    out = np.empty(q.size, dtype=np.int64)
    lib().ako_partial_pary_search(_p(hay), hay.size, _p(q), q.size, p, _p(out))
    return out


def pack_sections(part: dict, lc, hc, sp, i0: int, i1: int, tw, alias, chunk_capacity=0):
    """_pack_range / _chunked_pack_range (pack.py:30-159) into tw/alias."""
    lc, hc, sp = _i64(lc), _i64(hc), _f64(sp)
    out = np.empty(i1 - i0 + 1)
    args = [_p(part["l_index"]), _p(part["l_weight"]), _p(part["h_index"]), _p(part["h_weight"]),
            part["h_index"].size, _p(lc), _p(hc), _p(sp), i0, i1, part["avg"]]
    if chunk_capacity:
        lib().ako_chunked_pack_range(*args, chunk_capacity, _p(tw), _p(alias), _p(out))
    else:
        lib().ako_pack_range(*args, _p(tw), _p(alias), _p(out))
    return out


def psa_construct(w, total: float, s=64, workers=1, chunked=False, chunk_capacity=1024) -> Table:
    """psa_construct (pack.py:255-277), pthread workers."""
    w = _f64(w)
    n = w.size
    tw = np.zeros(n)
    alias = np.zeros(n, dtype=np.int64)
    rc = lib().ako_psa_construct(_p(w), n, total, s, workers, int(chunked), chunk_capacity,
                                 _p(tw), _p(alias))
    if rc:
        raise ValueError("PlanInconsistent")
    return Table(tw, alias, n, total)


def greedy_prepack(w, total: float, block_size=4096, threshold=8):
    """_greedy_kernel (partition.py:134-227)."""
    w = _f64(w)
    n = w.size
    tw = np.zeros(n)
    alias = np.zeros(n, dtype=np.int64)
    written = np.zeros(n, dtype=np.uint8)
    res_idx = np.empty(n, dtype=np.int64)
    res_w = np.empty(n)
    res_light = np.empty(n, dtype=np.uint8)
    nw = np.zeros(1, dtype=np.uint64)
    nres = int(lib().ako_greedy_prepack(_p(w), n, total / n, block_size, threshold, _p(tw),
                                        _p(alias), _p(written), _p(res_idx), _p(res_w),
                                        _p(res_light), _p(nw)))
    return dict(tw=tw, alias=alias, written=written.astype(bool), res_idx=res_idx[:nres].copy(),
                res_w=res_w[:nres].copy(), res_light=res_light[:nres].copy(),
                nwritten=int(nw[0]))


# ---- sample.py ------------------------------------------------------------

def rule(tw, alias, avg, u, lo=0, span=None) -> np.ndarray:
    """The bucket rule on explicit uniforms (sample.py:76-84)."""
    tw, alias, u = _f64(tw), _i64(alias), _f64(u)
    span = tw.size if span is None else span
    out = np.empty(u.size, dtype=np.int64)
    lib().ako_rule_from_uniforms(_p(tw), _p(alias), avg, lo, span, _p(u), u.size, _p(out))
    return out


def sample_batch(t: Table, m: int, seed: int, stream: int, counter: int = 0, workers=1):
    """sample_batch (sample.py:120-149)."""
    out = np.empty(m, dtype=np.int64)
    lib().ako_sample_batch(_p(_f64(t.tw)), _p(_i64(t.alias)), t.n, t.total, m, seed & MASK64,
                           stream & MASK64, counter & MASK64, workers, _p(out))
    return out


def probit(p: float) -> float:
    return float(lib().ako_probit(p))


def binom_draw(m: int, q: float, u: float) -> int:
    """_binom_draw (sample.py:152-174)."""
    return int(lib().ako_binom_draw(m, q, u))


def num_sections(n_rows: int, S: int) -> tuple[int, int]:
    S = min(S, n_rows)
    return S, -(-n_rows // S)


def assign_subtree(n_rows, S, seed, a, b, m, stream=0) -> np.ndarray:
    """assign_subtree (sample.py:222-240)."""
    S, _ = num_sections(n_rows, S)
    out = np.zeros(b - a, dtype=np.int64)
    lib().ako_assign_subtree(n_rows, S, seed & MASK64, stream & MASK64, a, b, m, _p(out))
    return out


def assign_sections(n_rows, S, M, seed, stream=0) -> np.ndarray:
    """assign_sections (sample.py:203-219) → counts."""
    S, ns = num_sections(n_rows, S)
    return assign_subtree(n_rows, S, seed, 0, ns, M, stream)


def sectioned_sample(t: Table, S: int, M: int, seed: int, stream: int, counter: int = 0):
    """sectioned_sample (sample.py:243-267)."""
    S_eff, ns = num_sections(t.n, S)
    counts = assign_sections(t.n, S_eff, M, seed, stream)
    out = np.empty(M, dtype=np.int64)
    lib().ako_sectioned_sample(_p(_f64(t.tw)), _p(_i64(t.alias)), t.n, t.total, S_eff,
                               _p(counts), ns, seed & MASK64, stream & MASK64, counter & MASK64,
                               _p(out))
    return out
