// ak_weights.cu — make_weight_set (model.py:95-108) on the device.
//
// Validation (finite and > 0; the first bad index wins) and the total.  The
// reference takes the total from np.sum, which for a contiguous float64
// vector is numpy's pairwise summation: blocks of <= 128 values summed with 8
// interleaved accumulators, larger ranges split at n/2 rounded down to a
// multiple of 8 (numpy 2.3.5 pairwise_sum; restated in the oracle and pinned
// against np.sum by tests).  The tree depends on n only, so the device
// evaluates exactly the same additions in the same order — the total is
// bit-identical to the reference's — with every subtree of the cut at depth D
// summed by one warp (k_pairwise_leaves) and the top D levels combined by one
// or two more launches.
#include "ak_common.cuh"
#include <math_constants.h>

namespace {

constexpr u64 PW_BLOCK = 128;
constexpr u64 SUBTREE_TARGET = 2048;  // elements per thread at the cut depth

struct Node {
    u64 off, size;
    bool exists;  // false: below an earlier leaf, on a non-leftmost path
    bool leaf;    // size <= 128 (reached at or above this depth)
};

__host__ __device__ __forceinline__ u64 split_point(u64 size)
{
    u64 n2 = size / 2;
    return n2 - n2 % 8;
}

// node at depth d, index idx (bits MSB first: 0 = left, 1 = right)
__host__ __device__ inline Node node_at(u64 n, int d, u64 idx)
{
    Node nd{0, n, true, n <= PW_BLOCK};
    for (int lvl = 0; lvl < d; ++lvl) {
        int bit = (int)((idx >> (d - 1 - lvl)) & 1);
        if (nd.size <= PW_BLOCK) {
            // leaf already: only the all-left path carries it down
            if (bit) {
                nd.exists = false;
                return nd;
            }
            continue;
        }
        u64 n2 = split_point(nd.size);
        if (bit == 0) nd.size = n2;
        else {
            nd.off += n2;
            nd.size -= n2;
        }
    }
    nd.leaf = nd.size <= PW_BLOCK;
    return nd;
}

template <typename T>
__device__ __forceinline__ double ld_val(const T *p, u64 i)
{
    return (double)__ldg(p + i);
}

// numpy pairwise_sum leaf (n <= 128)
template <typename T>
__device__ double leaf_sum(const T *a, u64 off, u64 n)
{
    if (n < 8) {
        double res = 0.0;
        for (u64 i = 0; i < n; ++i) res += ld_val(a, off + i);
        return res;
    }
    double r0 = ld_val(a, off + 0), r1 = ld_val(a, off + 1), r2 = ld_val(a, off + 2),
           r3 = ld_val(a, off + 3), r4 = ld_val(a, off + 4), r5 = ld_val(a, off + 5),
           r6 = ld_val(a, off + 6), r7 = ld_val(a, off + 7);
    u64 i;
    for (i = 8; i < n - (n % 8); i += 8) {
        r0 += ld_val(a, off + i + 0);
        r1 += ld_val(a, off + i + 1);
        r2 += ld_val(a, off + i + 2);
        r3 += ld_val(a, off + i + 3);
        r4 += ld_val(a, off + i + 4);
        r5 += ld_val(a, off + i + 5);
        r6 += ld_val(a, off + i + 6);
        r7 += ld_val(a, off + i + 7);
    }
    double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    for (; i < n; ++i) res += ld_val(a, off + i);
    return res;
}

// full pairwise recursion over [off, off+n) with an explicit stack
template <typename T>
__device__ double subtree_sum(const T *a, u64 off, u64 n)
{
    // post-order evaluation: stack of (off, size, state); values stack
    struct Fr {
        u64 off, size;
        int state;
    };
    Fr st[48];
    double vals[48];
    int sp = 0, vp = 0;
    st[sp++] = {off, n, 0};
    while (sp) {
        Fr &f = st[sp - 1];
        if (f.size <= PW_BLOCK) {
            vals[vp++] = leaf_sum(a, f.off, f.size);
            --sp;
            continue;
        }
        u64 n2 = split_point(f.size);
        if (f.state == 0) {
            f.state = 1;
            st[sp++] = {f.off, n2, 0};
        } else if (f.state == 1) {
            f.state = 2;
            st[sp++] = {f.off + n2, f.size - n2, 0};
        } else {
            double r = vals[--vp];
            double l = vals[--vp];
            vals[vp++] = l + r;
            --sp;
        }
    }
    return vals[0];
}

// One warp per node of the cut (<= ~2300 values).  Lane l takes the node's
// descendant slot l at depth 5 below it: every leaf of the node (<= 128
// values) sits in exactly one slot (its leftmost), because no descendant at
// depth 5 exceeds 128 values.  The leaves are summed four at a time, one
// 8-lane group per leaf with lane k holding numpy's accumulator r_k (a warp
// load touches four 32-byte runs), the groups fold their accumulators in
// numpy's order and add the tail values; then the five levels above the
// slots are folded by shuffles, each internal node adding its right child to
// its left.  Every addition is numpy's, in its order: the sum is
// bit-identical.  Validation (finite, > 0) rides on the same loads.
constexpr int PW_WARPS = 4;
constexpr int PW_SLOT_DEPTH = 5;

// descendant of `root` at relative depth d, index idx (MSB first: 0 = left)
__device__ __forceinline__ Node node_below(Node root, int d, u32 idx)
{
    Node nd = root;
    for (int lvl = 0; lvl < d; ++lvl) {
        const int bit = (int)((idx >> (d - 1 - lvl)) & 1);
        if (nd.size <= PW_BLOCK) {
            if (bit) {
                nd.exists = false;
                return nd;
            }
            continue;
        }
        const u64 h = split_point(nd.size);
        if (bit == 0) nd.size = h;
        else {
            nd.off += h;
            nd.size -= h;
        }
    }
    nd.leaf = nd.size <= PW_BLOCK;
    return nd;
}

template <typename T>
__global__ void __launch_bounds__(PW_WARPS * 32) k_pairwise_leaves(const T *__restrict__ w, u64 n, int D,
                                                                   double *__restrict__ part,
                                                                   unsigned long long *__restrict__ first_bad)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u64 idx = (u64)blockIdx.x * PW_WARPS + wid;
    if (idx >= (1ull << D)) return;
    const Node nd = node_at(n, D, idx);
    if (!nd.exists) return;
    if (nd.size > 32 * PW_BLOCK) {  // cut nodes are <= ~2300 values; n > 2^41 only
        if (lane == 0) {
            for (u64 i = nd.off; i < nd.off + nd.size; ++i) {
                const double v = ld_val(w, i);
                if (!(isfinite(v) && v > 0.0)) {
                    atomicMin(first_bad, (unsigned long long)i);
                    break;
                }
            }
            part[idx] = nd.size <= PW_BLOCK ? leaf_sum(w, nd.off, nd.size) : subtree_sum(w, nd.off, nd.size);
        }
        return;
    }
    const Node mine = node_below(nd, PW_SLOT_DEPTH, (u32)lane);  // a leaf or nothing
    const u32 myoff = (u32)(mine.off - nd.off), mylen = mine.exists ? (u32)mine.size : 0u;
    // the slots that hold a leaf, in order: a node's leaves sit above depth 5
    // on every path where the sizes reach 128 early (at N=1e9 a ~1900-value
    // node has 16 leaves of ~119 values in its 32 slots), so the groups walk
    // the leaf list, not the slots
    const unsigned leafm = __ballot_sync(0xffffffffu, mine.exists);
    const int nleaf = __popc(leafm);
    const int myrank = __popc(leafm & ((1u << lane) - 1u));
    // lane r < nleaf: the slot of leaf r, the largest p with r set bits below it
    int leafslot = 0;
#pragma unroll
    for (int b = 16; b >= 1; b >>= 1) {
        const int c = leafslot + b;
        if (__popc(leafm & (c >= 32 ? 0xffffffffu : (1u << c) - 1u)) <= lane) leafslot = c;
    }
    u64 bad = ~0ull;
    double leafsum = 0.0;
    // f32 weights 8-byte aligned: float2 loads, 4 lanes per leaf (lane k of
    // a group holds numpy's accumulators r_2k and r_2k+1), 8 leaves per pass.
    // Leaves start at multiples of 8 (numpy splits at multiples of 8), so the
    // pairs are aligned.  The additions are numpy's, in its order.
    if (sizeof(T) == 4 && (((uintptr_t)w) & 7) == 0) {
        const int g = lane >> 2, k = lane & 3;
        for (int s0 = 0; s0 < nleaf; s0 += 8) {
            const int j = s0 + g;  // leaf handled by this group
            const int sl = __shfl_sync(0xffffffffu, leafslot, j & 31);
            const u32 off = __shfl_sync(0xffffffffu, myoff, sl);
            u32 len = __shfl_sync(0xffffffffu, mylen, sl);
            if (j >= nleaf) len = 0;
            const u64 base = nd.off + off;
            const u32 m8 = len >= 8 ? len - len % 8 : 0;
            const float2 *wp = reinterpret_cast<const float2 *>(reinterpret_cast<const float *>(w) + base);
            float2 x[PW_BLOCK / 8];
#pragma unroll
            for (int q = 0; q < (int)(PW_BLOCK / 8); ++q)
                x[q] = 8u * q < m8 ? __ldg(wp + 4 * q + k) : make_float2(1.f, 1.f);
            const u32 nt = len - m8;  // tail values (< 8): lane k holds tail values 2k, 2k + 1
            const double t0 = (u32)(2 * k) < nt ? ld_val(w, base + m8 + 2 * k) : 1.0;
            const double t1 = (u32)(2 * k + 1) < nt ? ld_val(w, base + m8 + 2 * k + 1) : 1.0;
            double ra = 0.0, rb = 0.0;
            if (len >= 8) {
                ra = (double)x[0].x;
                rb = (double)x[0].y;
#pragma unroll
                for (int q = 1; q < (int)(PW_BLOCK / 8); ++q)
                    if (8u * q < m8) {
                        ra += (double)x[q].x;
                        rb += (double)x[q].y;
                    }
            }
            float mn = fminf(x[0].x, x[0].y);
#pragma unroll
            for (int q = 1; q < (int)(PW_BLOCK / 8); ++q) {
                mn = mn < x[q].x ? mn : x[q].x;
                mn = mn < x[q].y ? mn : x[q].y;
            }
            const bool ok = x[0].x == x[0].x && x[0].y == x[0].y && (double)mn > 0.0 && t0 > 0.0 &&
                            t1 > 0.0 && isfinite(ra + rb + t0 + t1);
            if (!__all_sync(0xffffffffu, ok)) {
#pragma unroll
                for (int q = 0; q < (int)(PW_BLOCK / 8); ++q) {
                    const u64 i = base + 8u * q + 2 * k;
                    const double xa = (double)x[q].x, xb = (double)x[q].y;
                    if (!(xa > 0.0 && xa < CUDART_INF)) bad = bad < i ? bad : i;
                    if (!(xb > 0.0 && xb < CUDART_INF)) bad = bad < i + 1 ? bad : i + 1;
                }
                const u64 it = base + m8 + 2 * k;
                if (!(t0 > 0.0 && t0 < CUDART_INF)) bad = bad < it ? bad : it;
                if (!(t1 > 0.0 && t1 < CUDART_INF)) bad = bad < it + 1 ? bad : it + 1;
            }
            // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7))
            const double s = ra + rb;
            const double s1 = s + __shfl_down_sync(0xffffffffu, s, 1);
            double res = s1 + __shfl_down_sync(0xffffffffu, s1, 2);
            if (len < 8) res = 0.0;
#pragma unroll
            for (int jj = 0; jj < 7; ++jj) {  // the tail, in order
                const double va = __shfl_sync(0xffffffffu, t0, (lane & ~3) + (jj >> 1));
                const double vb = __shfl_sync(0xffffffffu, t1, (lane & ~3) + (jj >> 1));
                if ((u32)jj < nt) res += (jj & 1) ? vb : va;
            }
            // leaf j's sum -> the lane of its slot
            const double got = __shfl_sync(0xffffffffu, res, ((myrank - s0) & 7) * 4);
            if (mine.exists && myrank >= s0 && myrank < s0 + 8) leafsum = got;
        }
    } else {
        const int g = lane >> 3, k = lane & 7;
        for (int s0 = 0; s0 < nleaf; s0 += 4) {
            const int j = s0 + g;  // leaf handled by this group
            const int sl = __shfl_sync(0xffffffffu, leafslot, j & 31);
            u32 off = __shfl_sync(0xffffffffu, myoff, sl);
            u32 len = __shfl_sync(0xffffffffu, mylen, sl);
            if (j >= nleaf) len = 0;
            const u64 base = nd.off + off;
            const u32 m8 = len >= 8 ? len - len % 8 : 0;
            // all (<= 16) loads of the accumulator first (kept in the input
            // type), then its additions in order
            T x[PW_BLOCK / 8];
    #pragma unroll
            for (int q = 0; q < (int)(PW_BLOCK / 8); ++q) {
                const u32 i = 8u * q + k;
                x[q] = i < m8 ? __ldg(w + base + i) : T(1);
            }
            const u32 nt = len - m8;  // tail values (< 8), lane k holds tail value k
            const double xt = (u32)k < nt ? ld_val(w, base + m8 + k) : 1.0;
            double r = 0.0;
            if (len >= 8) {
                r = (double)x[0];
    #pragma unroll
                for (int q = 1; q < (int)(PW_BLOCK / 8); ++q)
                    if (8u * q < m8) r += (double)x[q];
            }
            // finite and > 0: a NaN or inf makes the lane's sum non-finite and a
            // value <= 0 shows in the minimum; only then is the exact first bad
            // index searched for (a finite sum overflowing to inf just searches)
            T mn = x[0];
    #pragma unroll
            for (int q = 1; q < (int)(PW_BLOCK / 8); ++q) mn = mn < x[q] ? mn : x[q];
            const bool ok = (double)mn > 0.0 && xt > 0.0 && isfinite(r + xt);
            if (!__all_sync(0xffffffffu, ok)) {
    #pragma unroll
                for (int q = 0; q < (int)(PW_BLOCK / 8); ++q) {
                    const u64 i = base + 8u * q + k;
                    const double xv = (double)x[q];
                    if (!(xv > 0.0 && xv < CUDART_INF)) bad = bad < i ? bad : i;
                }
                if (!(xt > 0.0 && xt < CUDART_INF)) bad = bad < base + m8 + k ? bad : base + m8 + k;
            }
            // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)) within the group
            const double s1 = r + __shfl_down_sync(0xffffffffu, r, 1);
            const double s2 = s1 + __shfl_down_sync(0xffffffffu, s1, 2);
            double res = s2 + __shfl_down_sync(0xffffffffu, s2, 4);
            if (len < 8) res = 0.0;
    #pragma unroll
            for (int jj = 0; jj < 7; ++jj) {  // the tail, in order
                const double v = __shfl_sync(0xffffffffu, xt, (lane & ~7) + jj);
                if ((u32)jj < nt) res += v;
            }
            // leaf j's sum -> the lane of its slot
            const double got = __shfl_sync(0xffffffffu, res, ((myrank - s0) & 3) * 8);
            if (mine.exists && myrank >= s0 && myrank < s0 + 4) leafsum = got;
        }
    }
    // fold the 5 levels above the slots: node (lv, t) spans slots
    // [t 2^(5-lv), (t+1) 2^(5-lv)); its right child starts halfway
    double v = leafsum;
#pragma unroll
    for (int lv = PW_SLOT_DEPTH - 1; lv >= 0; --lv) {
        const int span = 1 << (PW_SLOT_DEPTH - lv);
        const double o = __shfl_down_sync(0xffffffffu, v, span / 2);
        if ((lane & (span - 1)) == 0) {
            const Node p = node_below(nd, lv, (u32)(lane >> (PW_SLOT_DEPTH - lv)));
            if (p.exists && !p.leaf) v = v + o;
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const u64 o = __shfl_xor_sync(0xffffffffu, bad, d);
        bad = bad < o ? bad : o;
    }
    if (lane == 0) {
        if (bad != ~0ull) atomicMin(first_bad, (unsigned long long)bad);
        part[idx] = v;
    }
}

// Combine levels [d_lo, d_hi) in place: part holds values at depth d_hi in
// slots [0, 2^d_hi); each block folds 2^(d_hi-d_lo) children into one value
// at depth d_lo stored in out[block index].
__global__ void k_pairwise_combine(u64 n, int d_hi, int d_lo, const double *__restrict__ part,
                                   double *__restrict__ out)
{
    extern __shared__ double sv[];
    const int span_lv = d_hi - d_lo;  // levels folded by this block
    const u64 width = 1ull << span_lv;
    const u64 base = (u64)blockIdx.x * width;
    for (u64 t = threadIdx.x; t < width; t += blockDim.x) {
        Node nd = node_at(n, d_hi, base + t);
        sv[t] = nd.exists ? part[base + t] : 0.0;
    }
    __syncthreads();
    for (int lv = d_hi - 1; lv >= d_lo; --lv) {
        u64 cnt = 1ull << (lv - d_lo);
        u64 stride = 1ull << (d_hi - lv);  // slot spacing of this level's nodes
        for (u64 t = threadIdx.x; t < cnt; t += blockDim.x) {
            u64 gidx = ((u64)blockIdx.x << (lv - d_lo)) + t;  // index at depth lv
            Node nd = node_at(n, lv, gidx);
            u64 s = t * stride;
            if (nd.exists && !nd.leaf) sv[s] = sv[s] + sv[s + stride / 2];
            // leaf: value already sits in the leftmost slot
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = sv[0];
}

int cut_depth(u64 n)
{
    int D = 0;
    while ((n >> D) > SUBTREE_TARGET && D < 30) ++D;
    return D;
}

}  // namespace

extern "C" {

size_t ak_weights_workspace_bytes(uint64_t n)
{
    int D = cut_depth(n);
    size_t parts = (size_t)1 << D;
    return 256 + parts * sizeof(double) * 2 + 4096;
}

int ak_weights_validate_total(const void *w, int dtype, uint64_t n, double *total,
                              int64_t *bad_index, void *ws, size_t ws_bytes, void *stream)
{
    *bad_index = -1;
    if (n == 0) return AK_ERR_EMPTY_INPUT;
    if (dtype != AK_F32 && dtype != AK_F64) return AK_ERR_VALUE;
    if (ws_bytes < ak_weights_workspace_bytes(n)) return AK_ERR_WORKSPACE;
    cudaStream_t st = ak_stream(stream);
    const int D = cut_depth(n);
    unsigned char *base = (unsigned char *)ws;
    unsigned long long *bad = (unsigned long long *)base;
    double *part = (double *)(base + 256);
    double *part2 = part + ((size_t)1 << D);
    {
        const int rc = ak_fill_small(bad, 0xff, sizeof(unsigned long long), st);
        if (rc != AK_OK) return rc;
    }
    const u64 nthreads = 1ull << D;
    const unsigned g = (unsigned)((nthreads + PW_WARPS - 1) / PW_WARPS);
    const int tb = PW_WARPS * 32;
    if (dtype == AK_F32)
        k_pairwise_leaves<float><<<g, tb, 0, st>>>((const float *)w, n, D, part, bad);
    else
        k_pairwise_leaves<double><<<g, tb, 0, st>>>((const double *)w, n, D, part, bad);
    AK_LAUNCH_CHECK("k_pairwise_leaves");
    // fold the top D levels, at most 10 levels (1024 slots) per block
    int d = D;
    double *src = part, *dst = part2;
    while (d > 0) {
        int lo = d > 10 ? d - 10 : 0;
        u64 blocks = 1ull << lo;
        size_t smem = ((size_t)1 << (d - lo)) * sizeof(double);
        k_pairwise_combine<<<(unsigned)blocks, 256, smem, st>>>(n, d, lo, src, dst);
        AK_LAUNCH_CHECK("k_pairwise_combine");
        double *t = src;
        src = dst;
        dst = t;
        d = lo;
    }
    double tot = 0.0;
    unsigned long long b = 0;
    {
        const int rc = ak_readback(st, &tot, src, sizeof(double), &b, bad, sizeof(b));
        if (rc != AK_OK) return rc;
    }
    if (b != ~0ull) {
        *bad_index = (int64_t)b;
        return AK_ERR_INVALID_WEIGHT;
    }
    *total = tot;
    return AK_OK;
}

}  // extern "C"
