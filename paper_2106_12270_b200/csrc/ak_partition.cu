// ak_partition.cu — the structured PSA path in the reference's own layout:
//
//   ak_partition           partition_items (partition.py:106-131)
//   ak_split_plan          compute_split_plan (split.py:94-104, 52-88)
//   ak_partial_pary_search partial_pary_search (split.py:190-213)
//   ak_pack_sections       pack_section / chunked_pack_section (pack.py:30-232)
//
// These exist so the reference's step-by-step API (partition -> plan -> pack)
// runs on the device with the reference's semantics; the split and pack
// kernels are bit-identical to the reference on the same inputs.  The fast
// construction path is the fused builder in ak_build.cu.
#include "ak_common.cuh"

namespace {

constexpr int PT_THREADS = 256;
constexpr int PT_V = 8;
constexpr int PT_TILE = PT_THREADS * PT_V;

// ---------------------------------------------------------------------------
// partition: tile counts + double-double sums, scan, scatter
// ---------------------------------------------------------------------------
struct PartAgg {
    u64 nl;
    dd sl, sh;
};

template <typename T>
__device__ __forceinline__ void load_tile(const T *w, u64 n, u64 base, double v[PT_V], bool ok[PT_V])
{
    const u64 i0 = base + (u64)threadIdx.x * PT_V;
    if (i0 + PT_V <= n && ((((uintptr_t)(w + i0)) & 15) == 0)) {
        // the thread's 8 consecutive values as 16-byte vector loads
        if (sizeof(T) == 4) {
            const float4 a = __ldg(reinterpret_cast<const float4 *>(w + i0));
            const float4 b = __ldg(reinterpret_cast<const float4 *>(w + i0) + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int q = 0; q < PT_V / 2; ++q) {
                const double2 a = __ldg(reinterpret_cast<const double2 *>(w + i0) + q);
                v[2 * q] = a.x;
                v[2 * q + 1] = a.y;
            }
        }
#pragma unroll
        for (int k = 0; k < PT_V; ++k) ok[k] = true;
        return;
    }
#pragma unroll
    for (int k = 0; k < PT_V; ++k) {
        u64 i = i0 + k;
        ok[k] = i < n;
        v[k] = ok[k] ? (double)w[i] : 0.0;
    }
}

__device__ __forceinline__ dd shfl_up_dd(dd x, int d)
{
    return dd_make(shfl_up_d(x.hi, d), shfl_up_d(x.lo, d));
}

// block exclusive scan of (count, dd, dd); returns block totals in *tot
__device__ void block_scan3(u64 c, dd a, dd b, u64 &c_ex, dd &a_ex, dd &b_ex, u64 *ctot, dd *atot,
                            dd *btot)
{
    __shared__ u64 sc[PT_THREADS / 32];
    __shared__ dd sa[PT_THREADS / 32], sb[PT_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u64 ci = c;
    dd ai = a, bi = b;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        u64 cu = __shfl_up_sync(0xffffffffu, ci, d);
        dd au = shfl_up_dd(ai, d), bu = shfl_up_dd(bi, d);
        if (lane >= d) {
            ci += cu;
            ai = dd_add(au, ai);
            bi = dd_add(bu, bi);
        }
    }
    if (lane == 31) {
        sc[wid] = ci;
        sa[wid] = ai;
        sb[wid] = bi;
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = PT_THREADS / 32;
        u64 wc = lane < nw ? sc[lane] : 0;
        dd wa = lane < nw ? sa[lane] : dd_make(0.0), wb = lane < nw ? sb[lane] : dd_make(0.0);
#pragma unroll
        for (int d = 1; d < nw; d <<= 1) {
            u64 cu = __shfl_up_sync(0xffffffffu, wc, d);
            dd au = shfl_up_dd(wa, d), bu = shfl_up_dd(wb, d);
            if (lane >= d) {
                wc += cu;
                wa = dd_add(au, wa);
                wb = dd_add(bu, wb);
            }
        }
        if (lane < nw) {
            sc[lane] = wc;
            sa[lane] = wa;
            sb[lane] = wb;
        }
    }
    __syncthreads();
    u64 wbase_c = wid ? sc[wid - 1] : 0;
    dd wbase_a = wid ? sa[wid - 1] : dd_make(0.0), wbase_b = wid ? sb[wid - 1] : dd_make(0.0);
    // exclusive within warp = inclusive - own
    u64 ce = __shfl_up_sync(0xffffffffu, ci, 1);
    dd ae = shfl_up_dd(ai, 1), be = shfl_up_dd(bi, 1);
    if (lane == 0) {
        ce = 0;
        ae = dd_make(0.0);
        be = dd_make(0.0);
    }
    c_ex = wbase_c + ce;
    a_ex = dd_add(wbase_a, ae);
    b_ex = dd_add(wbase_b, be);
    *ctot = sc[PT_THREADS / 32 - 1];
    *atot = sa[PT_THREADS / 32 - 1];
    *btot = sb[PT_THREADS / 32 - 1];
    __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(PT_THREADS) k_part_tiles(const T *__restrict__ w, u64 n,
                                                           double avg, PartAgg *__restrict__ agg)
{
    double v[PT_V];
    bool ok[PT_V];
    const u64 base = (u64)blockIdx.x * PT_TILE;
    load_tile(w, n, base, v, ok);
    u64 c = 0;
    dd a = dd_make(0.0), b = dd_make(0.0);
#pragma unroll
    for (int k = 0; k < PT_V; ++k) {
        if (!ok[k]) continue;
        if (v[k] <= avg) {
            ++c;
            a = dd_add_d(a, v[k]);
        } else {
            b = dd_add_d(b, v[k]);
        }
    }
    u64 ce, ct;
    dd ae, be, at, bt;
    block_scan3(c, a, b, ce, ae, be, &ct, &at, &bt);
    if (threadIdx.x == 0) agg[blockIdx.x] = PartAgg{ct, at, bt};
}

// Exclusive scan over the tile aggregates in three steps that perform the
// single-block scan's additions in its order (the prefixes are bit-identical
// to it): every chunk of PT_THREADS tiles is scanned by its own CTA
// (block_scan3, in place, chunk total aside), one thread chains the chunk
// totals into carries sequentially, and the scatter adds its chunk's carry to
// its tile's local prefix.  One CTA walking 48828 tiles took 0.52 ms at
// N=1e8 (5.2 ms at 1e9).
__global__ void __launch_bounds__(PT_THREADS) k_part_chunk_scan(PartAgg *__restrict__ agg, u64 ntiles,
                                                                PartAgg *__restrict__ ctot)
{
    const u64 i = (u64)blockIdx.x * PT_THREADS + threadIdx.x;
    const PartAgg x = i < ntiles ? agg[i] : PartAgg{0, dd_make(0.0), dd_make(0.0)};
    u64 ce, ct;
    dd ae, be, at, bt;
    block_scan3(x.nl, x.sl, x.sh, ce, ae, be, &ct, &at, &bt);
    if (i < ntiles) agg[i] = PartAgg{ce, ae, be};
    if (threadIdx.x == 0) ctot[blockIdx.x] = PartAgg{ct, at, bt};
}

__global__ void k_part_carry(const PartAgg *__restrict__ ctot, u64 nchunks, PartAgg *__restrict__ carry,
                             PartAgg *__restrict__ total)
{
    // one warp: 32 chunk totals loaded at once, then the chain in order; every
    // lane computes the same carries (the same additions as one thread), lane
    // j stores carry j of the batch
    const int lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    PartAgg cr{0, dd_make(0.0), dd_make(0.0)};
    for (u64 b0 = 0; b0 < nchunks; b0 += 32) {
        const PartAgg mine = b0 + lane < nchunks ? ctot[b0 + lane] : PartAgg{0, dd_make(0.0), dd_make(0.0)};
        const int m = nchunks - b0 < 32 ? (int)(nchunks - b0) : 32;
        for (int j = 0; j < m; ++j) {
            if (lane == j) carry[b0 + j] = cr;
            const u64 tn = __shfl_sync(0xffffffffu, mine.nl, j);
            const dd tl = dd_make(__shfl_sync(0xffffffffu, mine.sl.hi, j), __shfl_sync(0xffffffffu, mine.sl.lo, j));
            const dd th = dd_make(__shfl_sync(0xffffffffu, mine.sh.hi, j), __shfl_sync(0xffffffffu, mine.sh.lo, j));
            cr = PartAgg{cr.nl + tn, dd_add(cr.sl, tl), dd_add(cr.sh, th)};
        }
    }
    if (lane == 0) *total = cr;
}

// Tile scatter.  The per-item arithmetic is the single-pass one (sequential
// double-double prefixes per thread from the tile's exclusive base); the
// outputs are staged in shared memory in output order (lights [0, ct),
// heavies [ct, len)) and written out by consecutive threads, instead of each
// thread storing its own interleaved ranks (32 scattered 8-byte stores per
// warp instruction).
template <typename T>
__global__ void __launch_bounds__(PT_THREADS) k_part_scatter(
    const T *__restrict__ w, u64 n, double avg, const PartAgg *__restrict__ loc,
    const PartAgg *__restrict__ carry, i64 *l_idx, T *l_w, i64 *h_idx, T *h_w, double *lpre,
    double *hpre)
{
    __shared__ double s_pre[PT_TILE];
    __shared__ T s_tw[PT_TILE];
    __shared__ unsigned short s_loc[PT_TILE];
    double v[PT_V];
    bool ok[PT_V];
    const u64 base = (u64)blockIdx.x * PT_TILE;
    load_tile(w, n, base, v, ok);
    u64 c = 0;
    dd a = dd_make(0.0), b = dd_make(0.0);
#pragma unroll
    for (int k = 0; k < PT_V; ++k) {
        if (!ok[k]) continue;
        if (v[k] <= avg) {
            ++c;
            a = dd_add_d(a, v[k]);
        } else {
            b = dd_add_d(b, v[k]);
        }
    }
    u64 ce, ct;
    dd ae, be, at, bt;
    block_scan3(c, a, b, ce, ae, be, &ct, &at, &bt);
    const PartAgg lt = loc[blockIdx.x], cr = carry[blockIdx.x / PT_THREADS];
    const PartAgg t{cr.nl + lt.nl, dd_add(cr.sl, lt.sl), dd_add(cr.sh, lt.sh)};
    u32 kl = (u32)ce;                                     // tile-local light rank
    u32 kh = (u32)ct + threadIdx.x * PT_V - (u32)ce;      // heavies go after the lights
    dd L = dd_add(t.sl, ae), H = dd_add(t.sh, be);
#pragma unroll
    for (int k = 0; k < PT_V; ++k) {
        const u32 li = threadIdx.x * PT_V + k;
        if (!ok[k]) continue;
        s_tw[li] = (T)v[k];
        if (v[k] <= avg) {
            s_loc[kl] = (unsigned short)li;
            L = dd_add_d(L, v[k]);
            s_pre[kl] = L.hi + L.lo;
            ++kl;
        } else {
            s_loc[kh] = (unsigned short)li;
            H = dd_add_d(H, v[k]);
            s_pre[kh] = H.hi + H.lo;
            ++kh;
        }
    }
    __syncthreads();
    const u32 len = (u32)(base + PT_TILE <= n ? PT_TILE : n - base);
    const u64 l0 = t.nl, h0 = base - t.nl;  // lights / heavies before this tile
    for (u32 j = threadIdx.x; j < (u32)ct; j += PT_THREADS) {
        const u32 li = s_loc[j];
        l_idx[l0 + j] = (i64)(base + li) + 1;
        l_w[l0 + j] = s_tw[li];
        lpre[l0 + j + 1] = s_pre[j];
    }
    for (u32 j = (u32)ct + threadIdx.x; j < len; j += PT_THREADS) {
        const u32 li = s_loc[j], r = j - (u32)ct;
        h_idx[h0 + r] = (i64)(base + li) + 1;
        h_w[h0 + r] = s_tw[li];
        hpre[h0 + r + 1] = s_pre[j];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        lpre[0] = 0.0;
        hpre[0] = 0.0;
    }
}

// ---------------------------------------------------------------------------
// split plan (split.py:52-88)
// ---------------------------------------------------------------------------
struct PlanArgs {
    const double *lpre, *hpre;
    i64 nl, nh;
    u64 n_total, s;
    double avg;
    i64 *lc, *hc;
    double *sp;
};

__device__ __forceinline__ i64 boundary_n(u64 i, u64 n, u64 s)
{
    return (i64)(((unsigned __int128)i * n) / s);
}

template <typename T>
__device__ __forceinline__ void plan_finish(const PlanArgs &A, const T *h_w, u64 i, i64 ni,
                                            double cap, i64 h)
{
    i64 l = ni - h;
    double taken = cap - (A.lpre[l] + A.hpre[h]);
    double sp = 0.0;
    if (h < A.nh && taken > 0.0) {
        sp = (double)h_w[h] - taken;
        if (sp < 0.0) sp = 0.0;
    }
    A.lc[i] = l;
    A.hc[i] = h;
    A.sp[i] = sp;
}

template <typename T>
__global__ void k_plan_binary(PlanArgs A, const T *__restrict__ h_w)
{
    u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        A.lc[0] = 0;
        A.hc[0] = 0;
        A.sp[0] = 0.0;
        A.lc[A.s] = A.nl;
        A.hc[A.s] = A.nh;
        A.sp[A.s] = 0.0;
    }
    if (i < 1 || i >= A.s) return;
    i64 ni = boundary_n(i, A.n_total, A.s);
    double cap = (double)ni * A.avg;
    i64 lo = ni - A.nl;
    if (lo < 0) lo = 0;
    i64 hi = ni < A.nh ? ni : A.nh;
    i64 best = lo, a = lo, b = hi;
    while (a <= b) {
        i64 mid = (a + b) >> 1;
        if (A.lpre[ni - mid] + A.hpre[mid] <= cap) {
            best = mid;
            a = mid + 1;
        } else {
            b = mid - 1;
        }
    }
    plan_finish(A, h_w, i, ni, cap, best);
}

// Batched split (the paper's generalised parallel search): a CTA owns RUN
// consecutive boundaries.  Warp 0 locates the two end states with 32-ary
// probes (each round 32 lanes test 32 evenly spaced h), which bounds every
// interior boundary's h range; the H and L prefix windows covering that range
// are then staged in shared memory and each thread finishes its boundary
// with a binary search there.
constexpr int PLAN_RUN = 256;
constexpr int PLAN_SMEM_DOUBLES = 12 * 1024;  // 96 KB of staged prefix values

__device__ i64 pary_boundary(const PlanArgs &A, i64 ni, double cap)
{
    // greatest h in [lo, hi] with L[ni-h] + H[h] <= cap, 32-ary then finish
    const int lane = threadIdx.x & 31;
    i64 lo = ni - A.nl;
    if (lo < 0) lo = 0;
    i64 hi = ni < A.nh ? ni : A.nh;
    // invariant: pred(lo) true or lo is the range floor; pred(hi+1) false
    i64 a = lo, b = hi;  // answer in [a, b]
    while (b - a > 32) {
        i64 width = b - a;
        i64 h = a + (i64)(((__int128)(lane + 1) * width) / 33);
        bool pr = A.lpre[ni - h] + A.hpre[h] <= cap;
        unsigned m = __ballot_sync(0xffffffffu, pr);
        // pred is monotone (true then false): count of true probes
        int t = __popc(m);
        i64 na = t ? a + (i64)(((__int128)t * width) / 33) : a;
        i64 nb = t < 32 ? a + (i64)(((__int128)(t + 1) * width) / 33) - 1 : b;
        a = na;
        b = nb;
    }
    // finish: lanes test a..b (<= 33 values)
    i64 h = a + lane;
    bool pr = h <= b && (A.lpre[ni - h] + A.hpre[h] <= cap);
    unsigned m = __ballot_sync(0xffffffffu, pr);
    i64 best = lo;
    if (m) best = a + 31 - __clz(m);  // greatest true
    // b - a can be 32 (33 values): test the last one separately
    if (b - a == 32) {
        bool pb = A.lpre[ni - b] + A.hpre[b] <= cap;
        if (pb) best = b;
    }
    return best;
}

template <typename T>
__global__ void __launch_bounds__(PLAN_RUN) k_plan_batched(PlanArgs A, const T *__restrict__ h_w)
{
    __shared__ i64 ends[2];
    __shared__ __align__(8) u64 bar;
    extern __shared__ __align__(16) double stage[];
    const u64 i0 = 1 + (u64)blockIdx.x * PLAN_RUN;
    if (i0 >= A.s) return;
    u64 i1 = i0 + PLAN_RUN - 1;  // inclusive
    if (i1 > A.s - 1) i1 = A.s - 1;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        A.lc[0] = 0;
        A.hc[0] = 0;
        A.sp[0] = 0.0;
        A.lc[A.s] = A.nl;
        A.hc[A.s] = A.nh;
        A.sp[A.s] = 0.0;
    }
    if (threadIdx.x < 64) {
        const int which = threadIdx.x >> 5;  // warp 0: first, warp 1: last
        u64 i = which ? i1 : i0;
        i64 ni = boundary_n(i, A.n_total, A.s);
        i64 h = pary_boundary(A, ni, (double)ni * A.avg);
        if ((threadIdx.x & 31) == 0) ends[which] = h;
    }
    __syncthreads();
    const i64 hA = ends[0], hB = ends[1];
    const i64 nA = boundary_n(i0, A.n_total, A.s), nB = boundary_n(i1, A.n_total, A.s);
    // windows: H[hA .. hB], L[nA - hB .. nB - hA] clipped to [0, nl] (every
    // probe ni - h of the searches below lies in that range)
    const i64 hlen = hB - hA + 1;
    const i64 l0 = nA - hB > 0 ? nA - hB : 0;
    const i64 l1 = nB - hA < A.nl ? nB - hA : A.nl;
    const i64 llen = l1 - l0 + 1;
    // the windows are staged with 1-D bulk async copies (the TMA engine) at
    // 16-byte-congruent offsets: H window at stage[k - hA2], L window at
    // stage[lbase + k - l02] (hA2, l02 = the window starts rounded down to
    // even); the odd end elements a bulk copy cannot cover are plain loads
    const i64 hA2 = hA & ~(i64)1, l02 = l0 & ~(i64)1;
    const i64 lbase = (hB - hA2 + 2) & ~(i64)1;
    const bool staged = hlen > 0 && llen > 0 && lbase + (l1 - l02 + 2) <= PLAN_SMEM_DOUBLES;
    const bool tma = ((((uintptr_t)A.hpre) | ((uintptr_t)A.lpre)) & 15) == 0;
    if (staged && tma) {
        // bulk parts: the even-aligned interiors [c0, c1) of each window
        const i64 hc0 = (hA + 1) & ~(i64)1, hc1 = (hB + 1) & ~(i64)1;
        const i64 lc0 = (l0 + 1) & ~(i64)1, lc1 = (l1 + 1) & ~(i64)1;
        const u32 hbytes = hc1 > hc0 ? (u32)((hc1 - hc0) * 8) : 0u;
        const u32 lbytes = lc1 > lc0 ? (u32)((lc1 - lc0) * 8) : 0u;
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            // one arrival (with the byte count of both copies) completes the phase
            mbar_expect_tx(&bar, hbytes + lbytes);
            if (hbytes) bulk_g2s(stage + (hc0 - hA2), A.hpre + hc0, hbytes, &bar);
            if (lbytes) bulk_g2s(stage + lbase + (lc0 - l02), A.lpre + lc0, lbytes, &bar);
        }
        // the odd ends (a window without a bulk part has at most two values)
        if (threadIdx.x == 1 && (hA < hc0 || !hbytes)) stage[hA - hA2] = A.hpre[hA];
        if (threadIdx.x == 2 && (hB >= hc1 || !hbytes)) stage[hB - hA2] = A.hpre[hB];
        if (threadIdx.x == 3 && (l0 < lc0 || !lbytes)) stage[lbase + l0 - l02] = A.lpre[l0];
        if (threadIdx.x == 4 && (l1 >= lc1 || !lbytes)) stage[lbase + l1 - l02] = A.lpre[l1];
        __syncthreads();  // barrier initialised before anyone waits on it
        mbar_wait(&bar, 0);
    } else if (staged) {  // prefix views not 16-byte aligned: plain loads
        for (i64 k = hA + threadIdx.x; k <= hB; k += blockDim.x) stage[k - hA2] = A.hpre[k];
        for (i64 k = l0 + threadIdx.x; k <= l1; k += blockDim.x) stage[lbase + k - l02] = A.lpre[k];
    }
    __syncthreads();
    const u64 i = i0 + threadIdx.x;
    if (i > i1) return;
    i64 ni = boundary_n(i, A.n_total, A.s);
    double cap = (double)ni * A.avg;
    i64 lo = ni - A.nl;
    if (lo < 0) lo = 0;
    i64 hi = ni < A.nh ? ni : A.nh;
    if (lo < hA) lo = hA;
    if (hi > hB) hi = hB;
    i64 best = lo, a = lo, b = hi;
    while (a <= b) {
        i64 mid = (a + b) >> 1;
        double L = staged ? stage[lbase + (ni - mid - l02)] : A.lpre[ni - mid];
        double H = staged ? stage[mid - hA2] : A.hpre[mid];
        if (L + H <= cap) {
            best = mid;
            a = mid + 1;
        } else {
            b = mid - 1;
        }
    }
    plan_finish(A, h_w, i, ni, cap, best);
}

// ---------------------------------------------------------------------------
// partial_pary_search (split.py:140-213)
// ---------------------------------------------------------------------------
__global__ void k_check_sorted(const double *a, u64 n, int *flag)
{
    u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n; i += stride)
        if (a[i] < a[i - 1]) atomicOr(flag, 1);
}

// _contract_range (split.py:157-187) by one warp: lanes evaluate the p
// pivots of a round in parallel; the reductions reproduce the sequential
// "last pivot < qmin" / "first pivot > qmax" picks exactly.
__global__ void k_contract(const double *hay, u64 n, const double *q, u64 m, int p, i64 *ab)
{
    const int lane = threadIdx.x;
    const double qmin = q[0], qmax = q[m - 1];
    i64 a = 0, b = (i64)n;
    while (b - a > p) {
        i64 width = b - a;
        i64 gs = -1, ls = -1, t_gs = -1, t_ls = -1;
        for (int t0 = 0; t0 < p; t0 += 32) {
            int t = t0 + lane;
            int cls = 0;  // 1: < qmin, 2: > qmax
            i64 s = 0;
            if (t < p) {
                s = a + (i64)t * (width - 1) / (p - 1);
                double v = hay[s];
                cls = v < qmin ? 1 : (v > qmax ? 2 : 0);
            }
            unsigned mlt = __ballot_sync(0xffffffffu, cls == 1);
            unsigned mgt = __ballot_sync(0xffffffffu, cls == 2);
            if (mlt) {  // greatest t with v < qmin (pivots are sorted by t)
                int l = 31 - __clz(mlt);
                t_gs = t0 + l;
                gs = __shfl_sync(0xffffffffu, s, l);
            }
            if (mgt && ls < 0) {  // least t with v > qmax
                int l = __ffs(mgt) - 1;
                t_ls = t0 + l;
                ls = __shfl_sync(0xffffffffu, s, l);
            }
        }
        i64 na = gs >= 0 ? gs + 1 : a;
        i64 nb = ls >= 0 ? ls : b;
        i64 band = (t_ls >= 0 ? t_ls : p) - (t_gs >= 0 ? t_gs : -1);
        a = na;
        b = nb;
        if (band >= p - 2 || 2 * (b - a) > width) break;
    }
    if (lane == 0) {
        ab[0] = a;
        ab[1] = b;
    }
}

__global__ void k_lower_bound(const double *hay, const double *q, u64 m, const i64 *ab, i64 *out)
{
    u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    i64 lo = ab[0], hi = ab[1];
    double x = q[i];
    while (lo < hi) {
        i64 mid = (lo + hi) >> 1;
        if (hay[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    out[i] = lo;
}

// ---------------------------------------------------------------------------
// pack sections (pack.py:30-159)
// ---------------------------------------------------------------------------
template <typename T>
struct PackArgs {
    const i64 *l_idx;
    const T *l_w;
    const i64 *h_idx;
    const T *h_w;
    i64 nl, nh;
    const i64 *lc, *hc;
    const double *sp;
    u64 s, sec_first, sec_last;
    double avg;
    typename RowOf<T>::type *rows;
    double *out_spills;
};

template <typename T>
__device__ __forceinline__ void put_row(typename RowOf<T>::type *rows, i64 it, double tw, i64 alias,
                                        double avg)
{
    typename RowOf<T>::type r;
    r.tw = tw_store<T>(tw, avg);
    r.alias = (decltype(r.alias))alias;
    rows[it - 1] = r;
}

// _pack_range (pack.py:30-71): one thread per section, the reference sweep
template <typename T>
__global__ void k_pack_plain(PackArgs<T> A)
{
    u64 sec = A.sec_first + (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (sec > A.sec_last) return;
    const i64 nh = A.nh;
    i64 la = A.lc[sec - 1], lb = A.lc[sec], ha = A.hc[sec - 1], hb = A.hc[sec];
    double spill_in = A.sp[sec - 1];
    i64 k = la, j = ha;
    double w = j < nh ? (spill_in > 0.0 ? spill_in : (double)A.h_w[j]) : 0.0;
    while (k < lb || j < hb) {
        if (j < nh && w > A.avg && k < lb) {
            i64 it = A.l_idx[k];
            double lw = (double)A.l_w[k];
            put_row<T>(A.rows, it, lw, A.h_idx[j], A.avg);
            w += lw - A.avg;
            k++;
        } else if (j < hb) {
            i64 it = A.h_idx[j];
            if (j + 1 < nh) {
                put_row<T>(A.rows, it, w, A.h_idx[j + 1], A.avg);
                w += (double)A.h_w[j + 1] - A.avg;
            } else {
                put_row<T>(A.rows, it, w, it, A.avg);
                w = 0.0;
            }
            j++;
        } else {
            i64 it = A.l_idx[k];
            put_row<T>(A.rows, it, (double)A.l_w[k], it, A.avg);
            k++;
        }
    }
    if (A.out_spills) A.out_spills[sec - A.sec_first] = j < nh ? w : 0.0;
}

// _chunked_pack_range (pack.py:74-159): one warp per section.  The warp
// copies light and heavy chunks of `cap` entries coalesced into its shared
// memory slice, refilling a buffer once more than two thirds of it has been
// consumed (heavy staging extends to hb+1); lane 0 runs the sweep from shared
// memory.  Arithmetic is the plain sweep's, so the rows are bit-identical.
constexpr int CH_WARPS = 4;

template <typename T>
__global__ void __launch_bounds__(CH_WARPS * 32) k_pack_chunked(PackArgs<T> A, int cap)
{
    extern __shared__ unsigned char ch_smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u64 sec = A.sec_first + (u64)blockIdx.x * CH_WARPS + wid;
    // per-warp slice: sl_idx, sh_idx (i64) then sl_w, sh_w (double)
    i64 *sl_idx = (i64 *)(ch_smem + (size_t)wid * cap * 32);
    i64 *sh_idx = sl_idx + cap;
    double *sl_w = (double *)(sh_idx + cap);
    double *sh_w = sl_w + cap;
    if (sec > A.sec_last) return;
    const i64 nh = A.nh;
    const i64 la = A.lc[sec - 1], lb = A.lc[sec], ha = A.hc[sec - 1], hb = A.hc[sec];
    const double spill_in = A.sp[sec - 1];
    const i64 hext = hb + 1 < nh ? hb + 1 : nh;
    i64 k = la, j = ha;
    i64 lw_lo = la, lw_hi = la, hw_lo = ha, hw_hi = ha;
    double w = 0.0;
    auto stage_l = [&](i64 from) {
        lw_lo = from;
        lw_hi = from + cap < lb ? from + cap : lb;
        for (i64 t = lw_lo + lane; t < lw_hi; t += 32) {
            sl_idx[t - lw_lo] = A.l_idx[t];
            sl_w[t - lw_lo] = (double)A.l_w[t];
        }
        __syncwarp();
    };
    auto stage_h = [&](i64 from) {
        hw_lo = from;
        hw_hi = from + cap < hext ? from + cap : hext;
        for (i64 t = hw_lo + lane; t < hw_hi; t += 32) {
            sh_idx[t - hw_lo] = A.h_idx[t];
            sh_w[t - hw_lo] = (double)A.h_w[t];
        }
        __syncwarp();
    };
    if (j < nh) {
        if (spill_in > 0.0) w = spill_in;
        else {
            stage_h(j);
            w = sh_w[0];
        }
    }
    // every lane runs the (uniform) control flow so refills stay warp-wide;
    // only lane 0 writes rows.
    while (k < lb || j < hb) {
        if (k < lb && (k >= lw_hi || 3 * (k - lw_lo) > 2 * (i64)cap)) stage_l(k);
        if (j < hext && (j >= hw_hi || (hw_hi < hext && 3 * ((j + 1) - hw_lo) > 2 * (i64)cap)))
            stage_h(j);
        if (j < nh && w > A.avg && k < lb) {
            i64 it = sl_idx[k - lw_lo];
            double lw = sl_w[k - lw_lo];
            if (lane == 0) put_row<T>(A.rows, it, lw, sh_idx[j - hw_lo], A.avg);
            w += lw - A.avg;
            k++;
        } else if (j < hb) {
            i64 it = sh_idx[j - hw_lo];
            if (j + 1 < nh) {
                if (lane == 0) put_row<T>(A.rows, it, w, sh_idx[j + 1 - hw_lo], A.avg);
                w += sh_w[j + 1 - hw_lo] - A.avg;
            } else {
                if (lane == 0) put_row<T>(A.rows, it, w, it, A.avg);
                w = 0.0;
            }
            j++;
        } else {
            i64 it = sl_idx[k - lw_lo];
            if (lane == 0) put_row<T>(A.rows, it, sl_w[k - lw_lo], it, A.avg);
            k++;
        }
    }
    if (lane == 0 && A.out_spills) A.out_spills[sec - A.sec_first] = j < nh ? w : 0.0;
}

template <typename T>
int run_partition(const void *wv, u64 n, double avg, i64 *l_idx, void *l_w, i64 *h_idx, void *h_w,
                  double *lpre, double *hpre, u64 *nl_out, u64 *nh_out, void *ws,
                  cudaStream_t st)
{
    const T *w = (const T *)wv;
    const u64 tiles = (n + PT_TILE - 1) / PT_TILE;
    const u64 chunks = (tiles + PT_THREADS - 1) / PT_THREADS;
    PartAgg *agg = (PartAgg *)ws;
    PartAgg *tot = agg + tiles;
    PartAgg *ctot = tot + 1;
    PartAgg *carry = ctot + chunks;
    k_part_tiles<T><<<(unsigned)tiles, PT_THREADS, 0, st>>>(w, n, avg, agg);
    AK_LAUNCH_CHECK("k_part_tiles");
    k_part_chunk_scan<<<(unsigned)chunks, PT_THREADS, 0, st>>>(agg, tiles, ctot);
    AK_LAUNCH_CHECK("k_part_chunk_scan");
    k_part_carry<<<1, 32, 0, st>>>(ctot, chunks, carry, tot);
    AK_LAUNCH_CHECK("k_part_carry");
    k_part_scatter<T><<<(unsigned)tiles, PT_THREADS, 0, st>>>(w, n, avg, agg, carry, l_idx, (T *)l_w,
                                                              h_idx, (T *)h_w, lpre, hpre);
    AK_LAUNCH_CHECK("k_part_scatter");
    PartAgg t;
    {
        const int rc = ak_readback(st, &t, tot, sizeof(t));
        if (rc != AK_OK) return rc;
    }
    *nl_out = t.nl;
    *nh_out = n - t.nl;
    return AK_OK;
}

template <typename T>
int run_plan(const double *lpre, u64 nl, const double *hpre, u64 nh, const void *h_w, u64 n_total,
             u64 s, double avg, i64 *lc, i64 *hc, double *sp, int method, cudaStream_t st)
{
    PlanArgs A{lpre, hpre, (i64)nl, (i64)nh, n_total, s, avg, lc, hc, sp};
    if (method == 0 || s < 2) {
        u64 thr = s + 1;
        k_plan_binary<T><<<(unsigned)((thr + 255) / 256), 256, 0, st>>>(A, (const T *)h_w);
        AK_LAUNCH_CHECK("k_plan_binary");
    } else {
        u64 runs = (s - 1 + PLAN_RUN - 1) / PLAN_RUN;
        size_t smem = PLAN_SMEM_DOUBLES * sizeof(double);
        AK_SMEM_ATTR(k_plan_batched<T>, (int)smem);
        k_plan_batched<T><<<(unsigned)runs, PLAN_RUN, smem, st>>>(A, (const T *)h_w);
        AK_LAUNCH_CHECK("k_plan_batched");
    }
    return AK_OK;
}

template <typename T>
int run_pack(const i64 *l_idx, const void *l_w, u64 nl, const i64 *h_idx, const void *h_w, u64 nh,
             const i64 *lc, const i64 *hc, const double *sp, u64 s, u64 f, u64 l, double avg,
             void *rows, double *out_spills, u32 cap, cudaStream_t st)
{
    PackArgs<T> A{l_idx, (const T *)l_w, h_idx, (const T *)h_w, (i64)nl, (i64)nh, lc, hc, sp, s,
                  f, l, avg, (typename RowOf<T>::type *)rows, out_spills};
    u64 cnt = l - f + 1;
    if (cap == 0) {
        k_pack_plain<T><<<(unsigned)((cnt + 127) / 128), 128, 0, st>>>(A);
        AK_LAUNCH_CHECK("k_pack_plain");
    } else {
        // device staging capacity: the caller's chunk capacity, bounded by
        // shared memory; the staging schedule never changes the arithmetic.
        int c = cap > 512 ? 512 : (int)cap;
        size_t smem = (size_t)CH_WARPS * c * 32;
        AK_SMEM_ATTR(k_pack_chunked<T>, (int)smem);
        k_pack_chunked<T><<<(unsigned)((cnt + CH_WARPS - 1) / CH_WARPS), CH_WARPS * 32, smem, st>>>(
            A, c);
        AK_LAUNCH_CHECK("k_pack_chunked");
    }
    return AK_OK;
}

}  // namespace

extern "C" {

size_t ak_partition_workspace_bytes(uint64_t n)
{
    u64 tiles = (n + PT_TILE - 1) / PT_TILE;
    u64 chunks = (tiles + PT_THREADS - 1) / PT_THREADS;
    return (tiles + 2 + 2 * chunks) * sizeof(PartAgg) + 256;
}

int ak_partition(const void *w, int dtype, uint64_t n, double avg, int64_t *l_idx, void *l_w,
                 int64_t *h_idx, void *h_w, double *lprefix, double *hprefix, uint64_t *nl_out,
                 uint64_t *nh_out, void *ws, size_t ws_bytes, void *stream)
{
    if (n == 0) return AK_ERR_EMPTY_INPUT;
    if (ws_bytes < ak_partition_workspace_bytes(n)) return AK_ERR_WORKSPACE;
    if (dtype == AK_F32)
        return run_partition<float>(w, n, avg, l_idx, l_w, h_idx, h_w, lprefix, hprefix, nl_out,
                                    nh_out, ws, ak_stream(stream));
    if (dtype == AK_F64)
        return run_partition<double>(w, n, avg, l_idx, l_w, h_idx, h_w, lprefix, hprefix, nl_out,
                                     nh_out, ws, ak_stream(stream));
    return AK_ERR_VALUE;
}

int ak_split_plan(const double *lprefix, uint64_t nl, const double *hprefix, uint64_t nh,
                  const void *h_w, int dtype, uint64_t n_total, uint64_t s, double avg,
                  int64_t *lcounts, int64_t *hcounts, double *spills, int method, void *stream)
{
    if (s < 1 || s > (n_total > 1 ? n_total : 1)) return AK_ERR_INVALID_SECTION_COUNT;
    if (nl + nh != n_total) return AK_ERR_VALUE;
    if (dtype == AK_F32)
        return run_plan<float>(lprefix, nl, hprefix, nh, h_w, n_total, s, avg, lcounts, hcounts,
                               spills, method, ak_stream(stream));
    if (dtype == AK_F64)
        return run_plan<double>(lprefix, nl, hprefix, nh, h_w, n_total, s, avg, lcounts, hcounts,
                                spills, method, ak_stream(stream));
    return AK_ERR_VALUE;
}

int ak_partial_pary_search(const double *hay, uint64_t n, const double *q, uint64_t m,
                           uint32_t p, int64_t *out, void *stream)
{
    cudaStream_t st = ak_stream(stream);
    if (p < 3) return AK_ERR_VALUE;
    int *flag = (int *)ak_stream_scratch(st);
    if (!flag) return AK_ERR_CUDA;
    i64 *ab = (i64 *)((char *)flag + 16);
    {
        const int rc0 = ak_fill_small(flag, 0, 2 * sizeof(int), st);
        if (rc0 != AK_OK) return rc0;
    }
    const unsigned g = (unsigned)ak_num_sms() * 8;
    if (n > 1) k_check_sorted<<<g, 256, 0, st>>>(hay, n, flag);
    if (m > 1) k_check_sorted<<<g, 256, 0, st>>>(q, m, flag + 1);
    int f[2] = {0, 0};
    {
        const int rc0 = ak_readback(st, f, flag, 2 * sizeof(int));
        if (rc0 != AK_OK) return rc0;
    }
    AK_LAUNCH_CHECK("k_check_sorted");
    int rc = AK_OK;
    if (f[0] || f[1]) rc = AK_ERR_UNSORTED_INPUT;
    else if (m > 0) {
        k_contract<<<1, 32, 0, st>>>(hay, n, q, m, (int)p, ab);
        k_lower_bound<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(hay, q, m, ab, out);
        rc = ak_check_launch("k_lower_bound");
    }
    return rc;
}

int ak_pack_sections(const int64_t *l_idx, const void *l_w, uint64_t nl, const int64_t *h_idx,
                     const void *h_w, uint64_t nh, int dtype, const int64_t *lcounts,
                     const int64_t *hcounts, const double *spills, uint64_t s,
                     uint64_t sec_first, uint64_t sec_last, double avg, void *rows,
                     double *out_spills, uint32_t chunk_capacity, void *stream)
{
    if (sec_first < 1 || sec_last > s || sec_first > sec_last) return AK_ERR_PLAN_INCONSISTENT;
    if (chunk_capacity == 1) return AK_ERR_VALUE;
    if (dtype == AK_F32)
        return run_pack<float>(l_idx, l_w, nl, h_idx, h_w, nh, lcounts, hcounts, spills, s,
                               sec_first, sec_last, avg, rows, out_spills, chunk_capacity,
                               ak_stream(stream));
    if (dtype == AK_F64)
        return run_pack<double>(l_idx, l_w, nl, h_idx, h_w, nh, lcounts, hcounts, spills, s,
                                sec_first, sec_last, avg, rows, out_spills, chunk_capacity,
                                ak_stream(stream));
    return AK_ERR_VALUE;
}

}  // extern "C"
