// ak_build.cu — fused PSA construction (psa_construct, pack.py:255-277).
//
// Formulation.  Let d_i = avg - w_i (light deficit) and e_i = w_i - avg (heavy
// excess).  The sequential construction (seqbuild.py:33-58) is a merge of two
// sorted key sequences: light k has key DL(k) = sum of the deficits of the
// lights before it, heavy j has key DH(j) = sum of the excess of the heavies
// up to and including it; heavy j closes before light k iff DH(j) <= DL(k).
// Hence
//   light k:  alias = first heavy (in item order) with DH > DL(k), else self;
//   heavy j:  tw = DH(j) - DL(first light with DL >= DH(j)) + avg,
//             alias = next heavy, or itself when it is the last;
// and the split predicate L[n-h] + H[h] <= n*avg of split.py:69-77 is exactly
// DH(h) <= DL(n-h).  Every row follows from prefix sums, in parallel.
//
// Keys.  Items are grouped in tiles of 2048 (8 chunks of 256, one warp each).
// A key is (tile base, double-double) + (local offset, double): the local part
// comes from a warp-level Kogge-Stone scan whose lane bases are clamped by a
// running max/min into the chunk's [base, bound] so keys never decrease and
// never pass the chunk bound; the chunk bases/bounds are a monotone scan of
// the chunk totals done once by pass 1 and stored.  Any warp can therefore
// rebuild the canonical keys of any chunk, bit-identically, without a block
// barrier.  Cross-tile comparisons are exact: a local key plus the double-
// double difference of two tile bases is formed as a normalised double-double
// and compared with a local key.
//
// Pipeline (four kernels):
//  1. k_build_scan   one pass over the weights, streamed chunk by chunk
//                    through a per-warp ring of shared-memory slots filled by
//                    1-D bulk async copies (TMA): classify, per-chunk totals
//                    (reduce-scatter), light counts, first heavies, the
//                    light bitmask, the tile's monotone chunk bounds; a
//                    single-pass decoupled look-back over super-tiles (32
//                    tiles per CTA; 4-32 for small inputs, so at least ~2
//                    CTAs per SM) produces the exclusive tile bases DLb[t],
//                    DHb[t] (double-double sums) and light counts kL[t].
//  2. k_build_coarse merge of the two tile-boundary sequences: for each tile
//                    the first heavy tile covering its light keys (T1) and
//                    the first heavy after it (nextH).
//  3. k_build_split  PSA split: for every section (light tile) boundary, the
//                    heavy rank J = #heavies with key <= DLb[u] (tile from the
//                    coarse merge, chunk from the stored bounds, count from
//                    one chunk's canonical keys).
//  4. k_build_pack   CTA per section: the tile's lights and the heavies of
//                    ranks [J(u), J(u+1)) (any tiles; L2-resident, being the
//                    lights' neighbours in key space) are merged once by a
//                    merge path over order-preserving 64-bit integer keys in
//                    shared memory; each row is written exactly once (light
//                    rows by consecutive threads, coalesced).  43 KB of shared
//                    memory and 48 registers: 5 CTAs per SM (the pack is
//                    occupancy bound: 3/4/5 per SM = 14.3/12.6/11.6 ms at 1e9).
//  DRAM traffic ~ read w twice + write the rows once = the algorithmic bytes
//  (ncu: profiles/r1k_ncu_bench_pass.json).
#include "ak_common.cuh"

namespace {

constexpr int TB = 256;            // threads per CTA
constexpr int VV = 8;              // items per lane
constexpr int CH = 32 * VV;        // items per chunk (one warp)
constexpr int NW = TB / 32;        // chunks per tile
constexpr int TILE = TB * VV;      // items per tile
constexpr int SUPER = 32;          // max tiles per pass-1 CTA (look-back granularity)
constexpr u64 NONE64 = ~0ull;
constexpr unsigned char NOFH = 0xFF;

// ---------------------------------------------------------------------------
// workspace layout
// ---------------------------------------------------------------------------
struct BuildWs {
    u64 nt, nst;  // tiles, super-tiles
    u32 super;    // tiles per super-tile (SUPER, fewer for small n: enough scan CTAs)
    unsigned int *counter;
    u32 *status;            // [nst] 0 none, 1 aggregate, 2 inclusive
    dd *agg_D, *agg_H;      // [nst] super-tile aggregates (write once)
    u64 *agg_k;             // [nst]
    dd *inc_D, *inc_H;      // [nst] inclusive prefixes (write once)
    u64 *inc_k;             // [nst]
    dd *DLb, *DHb;          // [nt+1] exclusive tile bases
    u64 *kL;                // [nt+1] lights before tile
    u64 *firstH;            // [nt]
    double *mD, *mE;        // [nt*8] chunk bounds (monotone inclusive scans)
    unsigned char *mfh;     // [nt*8] first heavy offset in chunk, NOFH if none
    unsigned short *mcl;    // [nt*8] lights in chunk
    u32 *T1;                // [nt+1]
    u64 *nextH;             // [nt]
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// tiles per scan CTA: 32, or as few as 4 (one per warp) so that small
// inputs still spread over ~2 CTAs per SM
inline u32 super_for(u64 nt)
{
    const u64 s = nt / 296;
    return (u32)(s >= SUPER ? SUPER : (s < 4 ? 4 : s & ~3ull));
}

template <typename F> inline void layout(u64 n, F &&take)
{
    u64 nt = (n + TILE - 1) / TILE;
    u64 nst = (nt + super_for(nt) - 1) / super_for(nt);
    size_t sizes[19] = {256,          nst * 4,      nst * 16,       nst * 16,       nst * 8,
                        nst * 16,     nst * 16,     nst * 8,        (nt + 1) * 16,  (nt + 1) * 16,
                        (nt + 1) * 8, nt * 8,       nt * NW * 8,    nt * NW * 8,    nt * NW,
                        (nt + 1) * 4, 0,            nt * 8,         nt * NW * 2};  // [16]: unused
    for (int i = 0; i < 19; ++i) take(i, sizes[i]);
}

inline BuildWs carve(void *ws, u64 n)
{
    BuildWs W;
    W.nt = (n + TILE - 1) / TILE;
    W.super = super_for(W.nt);
    W.nst = (W.nt + W.super - 1) / W.super;
    char *base = (char *)ws;
    size_t off = 0;
    char *p[19];
    layout(n, [&](int i, size_t b) {
        p[i] = base + off;
        off += align256(b);
    });
    W.counter = (unsigned int *)p[0];
    W.status = (u32 *)p[1];
    W.agg_D = (dd *)p[2];
    W.agg_H = (dd *)p[3];
    W.agg_k = (u64 *)p[4];
    W.inc_D = (dd *)p[5];
    W.inc_H = (dd *)p[6];
    W.inc_k = (u64 *)p[7];
    W.DLb = (dd *)p[8];
    W.DHb = (dd *)p[9];
    W.kL = (u64 *)p[10];
    W.firstH = (u64 *)p[11];
    W.mD = (double *)p[12];
    W.mE = (double *)p[13];
    W.mfh = (unsigned char *)p[14];
    W.T1 = (u32 *)p[15];
    W.nextH = (u64 *)p[17];
    W.mcl = (unsigned short *)p[18];
    return W;
}

size_t split_bytes(u64 n)
{
    const u64 nt = (n + TILE - 1) / TILE;
    return align256(3 * (nt + 2) * 8);
}

size_t ws_bytes_for(u64 n)
{
    size_t off = 0;
    layout(n, [&](int, size_t b) { off += align256(b); });
    return off + 256 + split_bytes(n);
}

// ---------------------------------------------------------------------------
// loads and the canonical warp scan
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void load8(const T *__restrict__ w, u64 n, u64 i0, double v[VV])
{
    if (i0 + VV <= n) {
        if (sizeof(T) == 4) {
            const float4 *p = reinterpret_cast<const float4 *>(w + i0);
            float4 a = __ldg(p), b = __ldg(p + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
            const double2 *p = reinterpret_cast<const double2 *>(w + i0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double2 a = __ldg(p + q);
                v[2 * q] = a.x;
                v[2 * q + 1] = a.y;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < VV; ++k) v[k] = (i0 + k < n) ? (double)w[i0 + k] : -1.0;  // absent
    }
}

// inclusive Kogge-Stone scan followed by a running max: non-decreasing
__device__ __forceinline__ double warp_scan_mono(double x, int lane)
{
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        double y = shfl_up_d(x, d);
        if (lane >= d) x = x + y;
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        double y = shfl_up_d(x, d);
        if (lane >= d) x = x > y ? x : y;
    }
    return x;
}

// Lane-level part of the canonical chunk scan for one class: per-item local
// prefixes (exclusive for lights, inclusive for heavies), the lane's
// exclusive base within the chunk and the chunk total.
template <bool LIGHT>
__device__ __forceinline__ void lane_class(const double v[VV], double avg, double loc[VV], u32 &mask,
                                           double &excl, double &total, int lane, bool full = false)
{
    double s = 0.0;
    u32 m = 0;
#pragma unroll
    for (int k = 0; k < VV; ++k) {
        const bool valid = full || v[k] >= 0.0;
        const bool in = LIGHT ? (valid && v[k] <= avg) : (valid && v[k] > avg);
        if (LIGHT) loc[k] = s;
        if (in) s = s + (LIGHT ? (avg - v[k]) : (v[k] - avg));
        if (!LIGHT) loc[k] = s;
        m |= (u32)in << k;
    }
    double inc = warp_scan_mono(s, lane);
    excl = shfl_up_d(inc, 1);
    if (lane == 0) excl = 0.0;
    total = inc;  // unused by callers that take bounds from pass 1
    mask = m;
}

// Canonical keys of one class given the chunk's [base, bound].
__device__ __forceinline__ void class_keys(double loc[VV], double excl, double base, double bound,
                                           int lane)
{
    double B = base + excl;
    B = B < bound ? B : bound;
    double U = __shfl_down_sync(0xffffffffu, B, 1);
    if (lane == 31) U = bound;
#pragma unroll
    for (int k = 0; k < VV; ++k) {
        const double x = B + loc[k];
        loc[k] = x < U ? x : U;
    }
}

// offset of the first set item in the chunk (lane-major), NOFH if none
__device__ __forceinline__ unsigned char first_item(u32 mask, int lane)
{
    unsigned b = __ballot_sync(0xffffffffu, mask != 0);
    if (!b) return NOFH;
    int fl = __ffs(b) - 1;
    u32 fm = __shfl_sync(0xffffffffu, mask, fl);
    return (unsigned char)(fl * VV + __ffs(fm) - 1);
}

// ---------------------------------------------------------------------------
// 1. scan + super-tile decoupled look-back
// ---------------------------------------------------------------------------
__device__ __forceinline__ dd shfl_xor_dd(dd x, int m)
{
    return dd_make(__shfl_xor_sync(0xffffffffu, x.hi, m), __shfl_xor_sync(0xffffffffu, x.lo, m));
}

// lane's 8 items of a chunk staged in shared memory (T values, not widened)
template <typename T>
__device__ __forceinline__ void lds8_raw(const T *p, T v[VV])
{
    if (sizeof(T) == 4) {
        const float4 a = reinterpret_cast<const float4 *>(p)[0], b = reinterpret_cast<const float4 *>(p)[1];
        const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int q = 0; q < VV; ++q) v[q] = (T)f[q];
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 a = reinterpret_cast<const double2 *>(p)[q];
            v[2 * q] = (T)a.x;
            v[2 * q + 1] = (T)a.y;
        }
    }
}

// the largest T not above avg: (double)v <= avg  <=>  v <= avg_t(avg)
template <typename T> __device__ __forceinline__ T avg_floor(double avg);
template <> __device__ __forceinline__ float avg_floor<float>(double avg)
{
    float f = __double2float_rd(avg);
    return f;
}
template <> __device__ __forceinline__ double avg_floor<double>(double avg) { return avg; }

// pairwise sum of 8 doubles (depth 3: independent adds for ILP)
__device__ __forceinline__ double sum8(const double x[8])
{
    return ((x[0] + x[1]) + (x[2] + x[3])) + ((x[4] + x[5]) + (x[6] + x[7]));
}

constexpr int SC_WARPS = 4;  // warps per scan CTA; each owns SUPER / SC_WARPS tiles
// TMA ring slots per scan warp (a power of two): 4 x 1 KB chunks for f32,
// 2 x 2 KB for f64 -- the same bytes in flight, and the smaller f64 ring
// fits more CTAs per SM (f64 build 14.17 -> 14.03 ms; f32 at 2 slots 11.48
// against 11.41 ms)
template <typename T> struct ScanRing {
    static constexpr int RS = sizeof(T) == 4 ? 4 : 2;
};
template <typename T> struct ScanBuf {
    // per warp a ring of NW chunk slots (chunk c of successive tiles in slot c),
    // then the per-lane class sums of the warp's current tile ([2][NW][32]
    // doubles: staged here instead of 32 registers, which held the scan at
    // 19.7% occupancy)
    static constexpr size_t RING = (size_t)SC_WARPS * ScanRing<T>::RS * CH * sizeof(T);
    static constexpr size_t BYTES = RING + (size_t)SC_WARPS * 2 * NW * 32 * sizeof(double);
};

// One pass over the weights.  Each warp streams its tiles chunk by chunk
// through a ring of shared-memory slots filled by 1-D bulk async copies (the
// TMA engine; ~7 chunks in flight per warp), classifies the items (in the
// weight type: v <= avg exactly), and forms per-chunk light/heavy totals as
// nl*avg - sum(light w) and sum(heavy w) - nh*avg (these only fix the chunk
// bounds that every key is clamped into, so their rounding is free), light
// counts, first-heavy offsets and the tile's monotone chunk bounds.  Warp 0
// then scans the super-tile's tile totals (double-double), publishes the
// aggregate, runs the decoupled look-back and writes the exclusive tile bases.
template <typename T>
__global__ void __launch_bounds__(SC_WARPS * 32) k_build_scan(const T *__restrict__ w, u64 n,
                                                              double avg, BuildWs W)
{
    constexpr int RS = ScanRing<T>::RS;
    extern __shared__ __align__(128) unsigned char scan_smem[];
    __shared__ __align__(8) u64 bars[SC_WARPS][RS];
    __shared__ double s_tD[SUPER], s_tE[SUPER];
    __shared__ u32 s_tL[SUPER];
    __shared__ u64 s_fH[SUPER];
    __shared__ unsigned int s_st;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_st = atomicAdd(W.counter, 1u);
    if (lane == 0) {
#pragma unroll
        for (int c = 0; c < RS; ++c) mbar_init(&bars[wid][c], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const u64 st = s_st;
    const u64 t0 = st * W.super;
    const u64 tn = (t0 + W.super <= W.nt) ? W.super : W.nt - t0;
    T *ring = reinterpret_cast<T *>(scan_smem) + (size_t)wid * RS * CH;
    const T avgT = avg_floor<T>(avg);
    auto full_chunk = [&](u64 g) { return (g + 1) * CH <= n; };
    auto issue = [&](u64 j, int c) {  // chunk c of the super-tile's tile j into slot c % RS
        const u64 g = (t0 + j) * NW + c;
        const int sl = c & (RS - 1);
        if (lane == 0 && j < tn && full_chunk(g)) {
            mbar_expect_tx(&bars[wid][sl], CH * sizeof(T));
            bulk_g2s(ring + sl * CH, w + g * CH, CH * sizeof(T), &bars[wid][sl]);
        }
    };
#pragma unroll
    for (int c = 0; c < RS; ++c) issue((u64)wid, c);
    u32 phase = 0;  // per-slot parity bits (a slot completes twice per tile)

    for (u64 j = wid; j < tn; j += SC_WARPS) {
        const u64 t = t0 + j;
        double *ssum = reinterpret_cast<double *>(scan_smem + ScanBuf<T>::RING) + (size_t)wid * 2 * NW * 32;
        u32 cl = 0;
        unsigned char cf = NOFH;
#pragma unroll
        for (int c = 0; c < NW; ++c) {
            const u64 g = t * NW + c;
            double xl[VV], xh[VV];
            u32 lm = 0, vm = 0;
            if (full_chunk(g)) {
                const int sl = c & (RS - 1);
                mbar_wait(&bars[wid][sl], (phase >> sl) & 1);
                phase ^= 1u << sl;
                T v[VV];
                lds8_raw(ring + sl * CH + lane * VV, v);
#pragma unroll
                for (int q = 0; q < VV; ++q) {
                    const bool li = v[q] <= avgT;
                    const double x = (double)v[q] - avg;  // avg - w == -(w - avg) exactly
                    xl[q] = li ? -x : 0.0;
                    xh[q] = li ? 0.0 : x;
                    lm |= (u32)li << q;
                }
                vm = 0xFFu;
                // the slot's reads are done (values consumed) and ordered
                // before the async-proxy refill: chunk c + RS of this tile or
                // chunk c + RS - NW of the warp's next tile
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (c + RS < NW) issue(j, c + RS);
                else issue(j + SC_WARPS, c + RS - NW);
            } else {
                double v[VV];
                load8(w, n, g * CH + (u64)lane * VV, v);
#pragma unroll
                for (int q = 0; q < VV; ++q) {
                    const bool valid = v[q] >= 0.0;
                    const bool li = valid && v[q] <= avg;
                    xl[q] = li ? avg - v[q] : 0.0;
                    xh[q] = valid && !li ? v[q] - avg : 0.0;
                    lm |= (u32)li << q;
                    vm |= (u32)valid << q;
                }
            }
            const u32 hm = vm & ~lm;
            const int nlq = __popc(lm), nhq = __popc(hm);
            (void)nhq;
            ssum[c * 32 + lane] = sum8(xl);
            ssum[(NW + c) * 32 + lane] = sum8(xh);
            const u32 nl = __reduce_add_sync(0xffffffffu, (u32)nlq);
            const unsigned char fh = first_item(hm, lane);
            if (lane == c) {
                cl = nl;
                cf = fh;
            }
        }
        // chunk totals -> lanes 0..7, then their monotone scan -> chunk bounds
        // chunk totals: lane l sums lanes 8q..8q+7 of chunk l>>2 (q = l&3)
        // for both classes, two butterfly steps finish: lanes 4c..4c+3 hold
        // chunk c's totals (a reduce-scatter layout)
        __syncwarp();
        double rD, rE;
        {
            const int cc = lane >> 2, qq = lane & 3;
            const double *pD = ssum + cc * 32 + qq * 8, *pE = ssum + (NW + cc) * 32 + qq * 8;
            rD = sum8(pD);
            rE = sum8(pE);
            rD = rD + __shfl_xor_sync(0xffffffffu, rD, 1);
            rE = rE + __shfl_xor_sync(0xffffffffu, rE, 1);
            rD = rD + __shfl_xor_sync(0xffffffffu, rD, 2);
            rE = rE + __shfl_xor_sync(0xffffffffu, rE, 2);
        }
        __syncwarp();  // ssum reads done before the next tile's writes
        double x = __shfl_sync(0xffffffffu, rD, (lane & 7) * 4), y = __shfl_sync(0xffffffffu, rE, (lane & 7) * 4);
        x = x > 0.0 ? x : 0.0;  // a class's chunk total is a sum of non-negative terms
        y = y > 0.0 ? y : 0.0;
        if (lane >= NW) x = y = 0.0;
#pragma unroll
        for (int d = 1; d < NW; d <<= 1) {
            double a = shfl_up_d(x, d), bb = shfl_up_d(y, d);
            if (lane >= d) { x = x + a; y = y + bb; }
        }
#pragma unroll
        for (int d = 1; d < NW; d <<= 1) {
            double a = shfl_up_d(x, d), bb = shfl_up_d(y, d);
            if (lane >= d) { x = x > a ? x : a; y = y > bb ? y : bb; }
        }
        if (lane < NW) {
            W.mD[t * NW + lane] = x;
            W.mE[t * NW + lane] = y;
            W.mfh[t * NW + lane] = cf;
            W.mcl[t * NW + lane] = (unsigned short)cl;
        }
        const u32 tl = __reduce_add_sync(0xffffffffu, lane < NW ? cl : 0u);
        const unsigned fhm = __ballot_sync(0xffffffffu, lane < NW && cf != NOFH);
        const int fc = fhm ? __ffs(fhm) - 1 : 0;
        const unsigned char ff = (unsigned char)__shfl_sync(0xffffffffu, (int)cf, fc);
        const double tD = shfl_idx_d(x, NW - 1), tE = shfl_idx_d(y, NW - 1);
        if (lane == 0) {
            s_tD[j] = tD;
            s_tE[j] = tE;
            s_tL[j] = tl;
            s_fH[j] = fhm ? t * TILE + (u64)fc * CH + ff : NONE64;
        }
    }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    // warp 0: inclusive scan of the tile totals (exact double-double sums)
    dd xD = dd_make((u64)lane < tn ? s_tD[lane] : 0.0), xH = dd_make((u64)lane < tn ? s_tE[lane] : 0.0);
    u64 xK = (u64)lane < tn ? s_tL[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const dd yD = dd_make(shfl_up_d(xD.hi, d), shfl_up_d(xD.lo, d));
        const dd yH = dd_make(shfl_up_d(xH.hi, d), shfl_up_d(xH.lo, d));
        const u64 yK = __shfl_up_sync(0xffffffffu, xK, d);
        if (lane >= d) {
            xD = dd_add(yD, xD);
            xH = dd_add(yH, xH);
            xK += yK;
        }
    }
    const dd aD = dd_make(shfl_idx_d(xD.hi, 31), shfl_idx_d(xD.lo, 31));
    const dd aH = dd_make(shfl_idx_d(xH.hi, 31), shfl_idx_d(xH.lo, 31));
    const u64 aK = __shfl_sync(0xffffffffu, xK, 31);
    if (lane == 0) {
        if (st == 0) {
            W.inc_D[0] = aD;
            W.inc_H[0] = aH;
            W.inc_k[0] = aK;
        } else {
            W.agg_D[st] = aD;
            W.agg_H[st] = aH;
            W.agg_k[st] = aK;
        }
        __threadfence();
        st_release_u32(&W.status[st], st == 0 ? 2u : 1u);
    }
    // decoupled look-back over the predecessors, 32 at a time
    dd eD = dd_make(0.0), eH = dd_make(0.0);
    u64 eK = 0;
    i64 pred = (i64)st - 1;
    while (pred >= 0) {
        const i64 p = pred - lane;
        u32 s = 2;
        if (p >= 0) {
            do { s = ld_acquire_u32(&W.status[p]); } while (s == 0);
        }
        const unsigned inc_mask = __ballot_sync(0xffffffffu, p >= 0 && s == 2);
        const int stop = inc_mask ? __ffs(inc_mask) - 1 : 32;
        dd cD = dd_make(0.0), cH = dd_make(0.0);
        u64 cK = 0;
        if (p >= 0 && lane < stop) {
            cD = W.agg_D[p];
            cH = W.agg_H[p];
            cK = W.agg_k[p];
        } else if (p >= 0 && lane == stop) {
            cD = W.inc_D[p];
            cH = W.inc_H[p];
            cK = W.inc_k[p];
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            cD = dd_add(cD, shfl_xor_dd(cD, m));
            cH = dd_add(cH, shfl_xor_dd(cH, m));
            cK += __shfl_xor_sync(0xffffffffu, cK, m);
        }
        eD = dd_add(eD, cD);
        eH = dd_add(eH, cH);
        eK += cK;
        if (stop < 32 || pred - 32 < 0) break;
        pred -= 32;
    }
    if (lane == 0 && st > 0) {
        W.inc_D[st] = dd_add(eD, aD);
        W.inc_H[st] = dd_add(eH, aH);
        W.inc_k[st] = eK + aK;
        __threadfence();
        st_release_u32(&W.status[st], 2u);
    }
    // exclusive bases of the super-tile's tiles
    const dd pD = dd_make(shfl_up_d(xD.hi, 1), shfl_up_d(xD.lo, 1));
    const dd pH = dd_make(shfl_up_d(xH.hi, 1), shfl_up_d(xH.lo, 1));
    const u64 pK = __shfl_up_sync(0xffffffffu, xK, 1);
    if ((u64)lane < tn) {
        const u64 t = t0 + lane;
        W.DLb[t] = lane ? dd_add(eD, pD) : eD;
        W.DHb[t] = lane ? dd_add(eH, pH) : eH;
        W.kL[t] = eK + (lane ? pK : 0);
        W.firstH[t] = s_fH[lane];
        if (t + 1 == W.nt) {
            W.DLb[W.nt] = dd_add(eD, xD);
            W.DHb[W.nt] = dd_add(eH, xH);
            W.kL[W.nt] = eK + xK;
        }
    }
}

// ---------------------------------------------------------------------------
// 2. coarse merge of the tile boundaries
// ---------------------------------------------------------------------------
// T1[u] = max{t : DHb[t] <= DLb[u]} for every section boundary u, as the
// paper's generalised parallel search: T1 is non-decreasing in u, so a CTA
// of 256 consecutive boundaries finds its first and last answer by two
// global binary searches, stages the tile-base window DHb[T1(first) ..
// T1(last)] in shared memory with one 1-D bulk async copy (TMA + mbarrier),
// and each thread searches its boundary there.  Windows wider than CW
// (rare: skewed inputs) search global memory instead.
constexpr int CW = 2048;  // staged tile bases (double-double): 32 KB
__global__ void __launch_bounds__(256) k_build_coarse(BuildWs W, u64 n)
{
    __shared__ __align__(16) dd win[CW];
    __shared__ __align__(8) u64 bar;
    __shared__ u64 ends[2];
    const u64 nt = W.nt;
    const u64 u0 = (u64)blockIdx.x * 256;
    const u64 u1 = u0 + 255 < nt ? u0 + 255 : nt;
    auto t1_global = [&](u64 u) {
        const dd x = W.DLb[u];
        u64 lo = 0, hi = nt;
        while (lo < hi) {
            const u64 mid = (lo + hi + 1) >> 1;
            if (dd_le(W.DHb[mid], x)) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    };
    if (threadIdx.x == 0) ends[0] = t1_global(u0);
    if (threadIdx.x == 32) ends[1] = t1_global(u1);
    __syncthreads();
    const u64 ta = ends[0], tb = ends[1];
    const u64 wl = tb - ta + 1;
    const bool staged = wl <= (u64)CW;
    if (staged) {
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_expect_tx(&bar, (u32)(wl * sizeof(dd)));
            bulk_g2s(win, W.DHb + ta, (u32)(wl * sizeof(dd)), &bar);
        }
        __syncthreads();
        mbar_wait(&bar, 0);
    }
    const u64 u = u0 + threadIdx.x;
    if (u > u1) return;
    {
        const dd x = W.DLb[u];
        u64 lo = ta, hi = tb;
        while (lo < hi) {
            const u64 mid = (lo + hi + 1) >> 1;
            if (dd_le(staged ? win[mid - ta] : W.DHb[mid], x)) lo = mid;
            else hi = mid - 1;
        }
        W.T1[u] = (u32)lo;
    }
    if (u < nt) {  // nextH[u]: first heavy item in tiles > u
        auto jH = [&](u64 t) -> u64 {
            u64 items = t * TILE < n ? t * TILE : n;
            return items - W.kL[t];
        };
        const u64 after = jH(u + 1);
        if (jH(nt) <= after) {
            W.nextH[u] = NONE64;
        } else {
            u64 lo = u + 1, hi = nt - 1;
            while (lo < hi) {
                u64 mid = (lo + hi) >> 1;
                if (jH(mid + 1) > after) hi = mid;
                else lo = mid + 1;
            }
            W.nextH[u] = W.firstH[lo];
        }
    }
}

__device__ __forceinline__ u32 warp_excl_count(u32 cnt, u32 &total, int lane)
{
    u32 inc = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        u32 a = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += a;
    }
    total = __shfl_sync(0xffffffffu, inc, 31);
    return inc - cnt;
}

// ---------------------------------------------------------------------------
// 3. PSA split: heavy rank at every section boundary
// ---------------------------------------------------------------------------
// Sections are the light tiles: section u holds the lights of tile u and the
// heavies whose keys fall in its light key range (DLb[u], DLb[u+1]].  Its
// boundary is J(DLb[u]) = #heavies with key <= DLb[u] — the reference's
// split (split.py:69-77: the greatest h with H[h] <= cap - L[n-h]).  One warp
// per boundary: the tile T1[u] from the coarse merge, the chunk from the
// pass-1 chunk bounds (8 lanes at once), the count inside the chunk from its
// canonical keys.  Outputs: the boundary's heavy rank, the chunk holding that
// rank, and the item of that heavy (the first heavy past the boundary).
constexpr int HCAP = 1300;       // heavies per merge round (shared memory for 5 CTAs per SM)

struct SplitOut {
    u64 *hrank;   // [nt+2]
    u64 *hchunk;  // [nt+2]
    u64 *hitem;   // [nt+2]
};

// d + x as a normalised double-double (exact for the key ranges in play)
__device__ __forceinline__ dd add_dd_d(dd d, double x)
{
    double s, e;
    two_sum(d.hi, x, s, e);
    e += d.lo;
    double h, l;
    fast_two_sum(s, e, h, l);
    return dd_make(h, l);
}

__device__ __forceinline__ u64 heavies_before_tile(const BuildWs &W, u64 n, u64 t)
{
    const u64 items = t * TILE < n ? t * TILE : n;
    return items - W.kL[t];
}
__device__ __forceinline__ u32 chunk_valid(u64 n, u64 g)
{
    const u64 cs = g * CH;
    return cs >= n ? 0u : (u32)(n - cs < (u64)CH ? n - cs : (u64)CH);
}

// first heavy item (0-based) after chunk c of tile t (NONE64 if none)
__device__ __forceinline__ u64 next_heavy_after(const BuildWs &W, u64 t, int c, int lane)
{
    const unsigned char fh = lane < NW ? W.mfh[t * NW + lane] : NOFH;
    unsigned m = __ballot_sync(0xffffffffu, lane < NW && lane > c && fh != NOFH);
    if (m) {
        int cc = __ffs(m) - 1;
        unsigned char f = (unsigned char)__shfl_sync(0xffffffffu, (int)fh, cc);
        return t * TILE + (u64)cc * CH + f;
    }
    return W.nextH[t];
}

template <typename T>
// 6 CTAs/SM (40 registers, a few bytes spilled): the warp-per-boundary
// search is latency-bound, and 48 warps/SM beat 32 at 64 registers
// (11.50 -> 11.41 ms for the N=1e9 f32 build)
__global__ void __launch_bounds__(TB, 6) k_build_split(const T *__restrict__ w, u64 n, double avg,
                                                    BuildWs W, SplitOut O)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u64 nt = W.nt;
    const u64 b = (u64)blockIdx.x * NW + wid;  // boundary
    if (b > nt) return;
    const dd x = W.DLb[b];
    const u64 t = W.T1[b];
    const u64 nh = heavies_before_tile(W, n, nt);
    if (t >= nt) {
        if (lane == 0) {
            O.hrank[b] = nh;
            O.hchunk[b] = nt * NW;
            O.hitem[b] = NONE64;
        }
        return;
    }
    const dd xr = dd_sub(x, W.DHb[t]);  // boundary in tile t's heavy frame
    // first chunk whose heavy bound passes xr (chunks before are entirely <= x)
    const double bnd = lane < NW ? W.mE[t * NW + lane] : 0.0;
    const unsigned pm = __ballot_sync(0xffffffffu, lane < NW && !(dd_le(dd_make(bnd), xr)));
    const int c = pm ? __ffs(pm) - 1 : NW - 1;
    // heavies of tile t in chunks before c
    u32 hc = 0;
    if (lane < c) hc = chunk_valid(n, t * NW + lane) - W.mcl[t * NW + lane];
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) hc += __shfl_xor_sync(0xffffffffu, hc, d);
    // canonical heavy keys of chunk (t, c): count those <= xr
    const double base = c ? W.mE[t * NW + c - 1] : 0.0, bound = W.mE[t * NW + c];
    double v[VV], k[VV], ex, tot;
    u32 m;
    load8(w, n, t * TILE + (u64)c * CH + (u64)lane * VV, v);
    lane_class<false>(v, avg, k, m, ex, tot, lane);
    class_keys(k, ex, base, bound, lane);
    u32 le = 0;
#pragma unroll
    for (int q = 0; q < VV; ++q) le += ((m >> q) & 1) && dd_le(dd_make(k[q]), xr);
    u32 cnt = __popc(m), allc = cnt, alle = le;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        allc += __shfl_xor_sync(0xffffffffu, allc, d);
        alle += __shfl_xor_sync(0xffffffffu, alle, d);
    }
    // item of the first heavy past x: the alle-th heavy of the chunk, or later
    u64 item = NONE64;
    if (alle < allc) {
        // locate the (alle)-th heavy in lane order
        u32 inc = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            u32 a = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += a;
        }
        const u32 exc = inc - cnt;
        u64 mine = NONE64;
        if (alle >= exc && alle < inc) {
            u32 r = alle - exc, mm = m;
            for (u32 s = 0; s < r; ++s) mm &= mm - 1;
            mine = t * TILE + (u64)c * CH + (u64)lane * VV + (__ffs(mm) - 1);
        }
        unsigned own = __ballot_sync(0xffffffffu, mine != NONE64);
        item = __shfl_sync(0xffffffffu, mine, __ffs(own) - 1);
    } else {
        item = next_heavy_after(W, t, c, lane);
    }
    if (lane == 0) {
        O.hrank[b] = heavies_before_tile(W, n, t) + hc + alle;
        O.hchunk[b] = t * NW + c;
        O.hitem[b] = item;
    }
}

// ---------------------------------------------------------------------------
// 4. section pack: merge the section's lights with its heavies
// ---------------------------------------------------------------------------
// CTA u = section u.  Lights: the 8 chunks of tile u, canonical keys in the
// tile's own frame (exact doubles).  Heavies: ranks [J(u), J(u+1)), rebuilt
// chunk by chunk (any tile) and converted to the own frame (exact
// double-doubles).  One merge path (heavy first on ties: DH <= DL) gives each
// light its successor heavy and each heavy its successor light; rows are
// written directly: lights by the threads that own them, heavies in rank
// order.  Large heavy ranges are processed in rounds of HCAP.
// Keys in shared memory are order-preserving 64-bit integers: for a key
// x >= 0, enc(x) = bits(x) << 1 (non-negative doubles order like their bit
// patterns); a heavy's double-double key (hi, lo) becomes
// (bits(hi) << 1) | (lo > 0), so "heavy <= light" (heavy first on ties) is
// one unsigned compare and exact against the double light keys.
struct SecSmem {
    u32 LS[TILE];                  // light successor heavy item (+1), 0 = unresolved
    u64 LK[TILE + 2];              // own light keys (own frame, encoded), rank order; ~0 sentinel
    u64 HK[HCAP + 1];              // heavy keys (own frame, encoded); ~0 sentinel
    u32 HI[HCAP + 1];              // heavy items; ~0 sentinel (LS = HI + 1 = 0: unresolved)
                                   // (HK holds the tile-frame key bits between the rebuild and
                                   // the conversion; a slot's chunk is its item's chunk)
    unsigned short SR[HCAP];       // heavy -> rank of its successor light (nL: none here)
    dd Dwin[32];                   // frame offset (chunk's tile base - own base) per window chunk
    u32 lfirst;
    u64 next_item;                 // item of the heavy ranked jend (first of the next round)
};

__device__ __forceinline__ u64 key_enc(double x) { return (u64)__double_as_longlong(x) << 1; }
__device__ __forceinline__ u64 key_enc_dd(dd x)
{
    return ((u64)__double_as_longlong(x.hi) << 1) | (x.lo > 0.0 ? 1ull : 0ull);
}
__device__ __forceinline__ double key_dec(u64 e) { return __longlong_as_double((long long)(e >> 1)); }
constexpr u64 KEY_INF = ~0ull;

// heavy rank of the first heavy of each of the 32 chunks g0 .. g0+31 (lane
// i holds chunk g0 + i; ~0 past the last chunk) and its heavy count; every
// warp computes the same table, so no block barrier is needed.
__device__ __forceinline__ void chunk_ranks(const BuildWs &W, u64 n, u64 g0, int lane, u64 &hb,
                                            u32 &hc)
{
    const u64 nch = W.nt * NW;
    const u64 g = g0 + lane;
    hc = g < nch ? chunk_valid(n, g) - W.mcl[g] : 0u;
    u32 inc = hc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u32 a = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += a;
    }
    const u64 t0 = g0 / NW;
    const int c0 = (int)(g0 % NW);
    u32 pre = 0;
    if (lane < c0) pre = chunk_valid(n, t0 * NW + lane) - W.mcl[t0 * NW + lane];
    pre = __reduce_add_sync(0xffffffffu, pre);
    const u64 base = (g0 < nch ? heavies_before_tile(W, n, t0) : heavies_before_tile(W, n, W.nt)) + pre;
    hb = g < nch ? base + (inc - hc) : ~0ull;
}

// Where the pack's rows go.  RowSink: row i of the table being built.
// RemapSink (PSA+'s residual build, T = double): the residual table's row r is
// the final table's row res_idx[r] - 1 and alias a its item res_idx[a - 1], so
// the residual rows land in the final table directly (thresholds rounded to
// the final table's type as ak_residual_scatter does), counting the rows.
template <typename T> struct RowSink {
    typedef typename RowOf<T>::type RowT;
    typedef decltype(RowT::tw) TwT;
    RowT *rows;
    __device__ __forceinline__ void put(u64 pos, TwT tw, u64 al) const
    {
        RowT r;
        r.tw = tw;
        r.alias = (decltype(RowT::alias))al;
        rows[pos] = r;
    }
    static constexpr bool counts = false;
};
template <typename RowOut> struct RemapSink {
    typedef double TwT;
    RowOut *rows;
    const i64 *res_idx;
    double avg;
    unsigned long long *written;
    __device__ __forceinline__ void put(u64 pos, double tw, u64 al) const
    {
        RowOut o;
        o.tw = tw_store<decltype(RowOut::tw)>(tw, avg);
        o.alias = al ? (decltype(RowOut::alias))res_idx[al - 1] : (decltype(RowOut::alias))0;
        rows[res_idx[pos] - 1] = o;
    }
    static constexpr bool counts = true;
};

template <typename T, typename Sink>
__global__ void __launch_bounds__(TB, 5) k_build_pack(const T *__restrict__ w, u64 n, double avg,
                                                      BuildWs W, SplitOut O, Sink sink, u32 pf_ahead)
{
    typedef typename Sink::TwT TwT;
    u32 nput = 0;  // rows written by this thread (RemapSink counts them)
    extern __shared__ __align__(16) unsigned char sec_smem[];
    SecSmem &P = *reinterpret_cast<SecSmem *>(sec_smem);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u64 nt = W.nt;
    const u64 u = blockIdx.x;  // section; u == nt: the heavies past every light
    const u64 J0 = O.hrank[u], J1 = u < nt ? O.hrank[u + 1] : heavies_before_tile(W, n, nt);
    const u64 after = u < nt ? O.hitem[u + 1] : NONE64;  // first heavy past the section
    const dd own = u < nt ? W.DLb[u] : W.DLb[nt];
    const double secbound = u < nt ? W.mD[u * NW + NW - 1] : 0.0;  // next light key, own frame

    if (threadIdx.x == 0 && pf_ahead) {
        // warm L2 for the section one resident grid ahead: its tile and the
        // start of its heavy window (so its loads hit L2, not DRAM)
        const u64 v = blockIdx.x + (u64)pf_ahead;
        if (v < W.nt && (v + 1) * TILE <= n)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(w + v * TILE),
                         "r"((u32)(TILE * sizeof(T))) : "memory");
        if (v < W.nt) {
            const u64 g = O.hchunk[v];
            if ((g + 8) * CH <= n)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(w + g * CH),
                             "r"((u32)(8 * CH * sizeof(T))) : "memory");
        }
    }
    // ---- lights of tile u (rank order = key order), keys into shared memory
    reinterpret_cast<uint4 *>(P.LS)[threadIdx.x] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4 *>(P.LS)[threadIdx.x + TB] = make_uint4(0, 0, 0, 0);
    u32 nL = 0, lrank0 = 0, lm = 0;
    double lv[VV];
    if (u < nt) {
        const uint4 cnt4 = *reinterpret_cast<const uint4 *>(W.mcl + u * NW);  // 8 x u16
        const u32 cw[4] = {cnt4.x, cnt4.y, cnt4.z, cnt4.w};
        u32 woff = 0;
#pragma unroll
        for (int k = 0; k < NW; ++k) {
            const u32 ck = (cw[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
            woff += k < wid ? ck : 0u;
            nL += ck;
        }
        load8(w, n, u * TILE + (u64)wid * CH + (u64)lane * VV, lv);
        const double b0 = wid ? W.mD[u * NW + wid - 1] : 0.0, b1 = W.mD[u * NW + wid];
        double lk[VV], ex, tot;
        lane_class<true>(lv, avg, lk, lm, ex, tot, lane, (u + 1) * TILE <= n);
        class_keys(lk, ex, b0, b1, lane);
        u32 tl;
        lrank0 = woff + warp_excl_count(__popc(lm), tl, lane);
#pragma unroll
        for (int q = 0; q < VV; ++q)
            if ((lm >> q) & 1) P.LK[lrank0 + __popc(lm & ((1u << q) - 1))] = key_enc(lk[q]);
    }
    if (threadIdx.x == 0) {
        P.LK[nL] = KEY_INF;
        P.next_item = NONE64;
    }
    __syncthreads();

    // ---- heavies in rounds of at most HCAP ranks (one round unless the
    // section's heavy range is large or spans more than 32 chunks)
    u64 jcur = J0;
    u64 gcur = O.hchunk[u];
    u32 lfirst = 0;  // first light not yet resolved
    while (jcur < J1) {
        u64 hb;
        u32 hc;
        chunk_ranks(W, n, gcur, lane, hb, hc);
        const u64 last = __shfl_sync(0xffffffffu, hb == ~0ull ? ~0ull : hb + hc, 31);
        u64 jend = J1 < jcur + HCAP ? J1 : jcur + HCAP;
        if (last < jend) jend = last;
        const u32 nH = (u32)(jend - jcur);
        const bool last_round = jend >= J1;
        const bool needed = hb != ~0ull && hb <= jend && hb + hc > jcur;
        const unsigned need = __ballot_sync(0xffffffffu, needed);
        if (wid == 0) {
            // frame offset of each needed window chunk
            if (needed) P.Dwin[lane] = dd_sub(W.DHb[(gcur + lane) / NW], own);
            if (lane == 0) {  // merge sentinels
                P.HK[nH] = KEY_INF;
                P.HI[nH] = 0xFFFFFFFFu;
            }
        }
        // rebuild the needed chunks' heavy keys (chunk frame) into their
        // rank slots; rank jend is the next round's first heavy
        for (int ci = wid; ci < 32; ci += NW) {
            if (!((need >> ci) & 1)) continue;
            const u64 cb = __shfl_sync(0xffffffffu, hb, ci);
            const u64 g = gcur + ci;
            const int c = (int)(g % NW);
            const double base = c ? W.mE[g - 1] : 0.0, bound = W.mE[g];
            double v[VV], k[VV], ex, tot;
            u32 m;
            load8(w, n, g * CH + (u64)lane * VV, v);
            lane_class<false>(v, avg, k, m, ex, tot, lane, (g + 1) * CH <= n);
            class_keys(k, ex, base, bound, lane);
            u32 tc;
            const int r0 = (int)((i64)cb - (i64)jcur) + (int)warp_excl_count(__popc(m), tc, lane);
            const u32 item0 = (u32)(g * CH + (u64)lane * VV);
#pragma unroll
            for (int q = 0; q < VV; ++q) {
                const int sl = r0 + __popc(m & ((1u << q) - 1));
                if (((m >> q) & 1) && sl >= 0 && sl < (int)nH) {
                    P.HK[sl] = (u64)__double_as_longlong(k[q]);  // tile frame until converted
                    P.HI[sl] = item0 + q;
                }
            }
            const int want = (int)nH - r0;  // this lane holds rank jend?
            if (want >= 0 && want < __popc(m)) {
                u32 mm = m;
                for (int z = 0; z < want; ++z) mm &= mm - 1;
                P.next_item = item0 + (u32)(__ffs(mm) - 1);
            }
        }
        __syncthreads();
        // heavy keys into the own frame (double-double), one thread per heavy
        for (u32 j = threadIdx.x; j < nH; j += TB)
            P.HK[j] = key_enc_dd(add_dd_d(P.Dwin[(u32)(P.HI[j] / CH - gcur)],
                                          __longlong_as_double((long long)P.HK[j])));
        if (!last_round && wid == 0 && P.next_item == NONE64) {
            // rank jend lies past the enumerated chunks
            const u64 gl = gcur + 31;
            const u64 nx = next_heavy_after(W, gl / NW, (int)(gl % NW), lane);
            if (lane == 0) P.next_item = nx;
        }
        __syncthreads();
        // merge path: lights [lfirst, nL) with heavies [0, nH); heavy first on
        // ties.  +inf sentinels end both lists; a taken heavy records the key
        // of its successor light, a taken light its successor heavy's item.
        {
            const u64 *LKp = P.LK + lfirst;
            u32 *LSp = P.LS + lfirst;
            const u32 na = nL - lfirst;
            const u32 total = na + nH;
            const u32 per = (total + TB - 1) / TB;
            const u32 d0 = threadIdx.x * per;
            if (d0 < total) {
                // lights among the first d0 merged: the greatest i with
                // light i-1 before heavy d0-i, by bisection (every lane
                // runs the same steps; galloping from the proportional
                // guess diverged and was 2% slower on Zipf-1)
                const u32 lo0 = d0 > nH ? d0 - nH : 0, hi0 = d0 < na ? d0 : na;
                auto light_first = [&](u32 i) {  // light i-1 precedes heavy d0-i
                    return P.HK[d0 - i] > LKp[i - 1];
                };
                u32 lo = lo0, hi = hi0;  // answer in [lo, hi]
                while (lo < hi) {
                    const u32 mid = (lo + hi + 1) >> 1;
                    if (light_first(mid)) lo = mid;
                    else hi = mid - 1;
                }
                u32 i = lo, j = d0 - lo;
                const u32 steps = d0 + per < total ? per : total - d0;
                u64 lk = LKp[i];
                u64 hk = P.HK[j];
                for (u32 d = 0; d < steps; ++d) {
                    if (hk <= lk) {
                        P.SR[j] = (unsigned short)(lfirst + i);
                        ++j;
                        hk = P.HK[j];
                    } else {
                        LSp[i] = P.HI[j] + 1;
                        ++i;
                        lk = LKp[i];
                    }
                }
            }
        }
        __syncthreads();
        // heavy rows of this round
        const u64 nxt = last_round ? after : P.next_item;
        for (u32 j = threadIdx.x; j < nH; j += TB) {
            const u32 item = P.HI[j];
            const u32 sr = P.SR[j];
            const double DL = sr < nL ? key_dec(P.LK[sr]) : secbound;
            const double tw = (key_dec(P.HK[j]) - DL) + avg;
            u64 al;
            if (j + 1 < nH) al = (u64)P.HI[j + 1] + 1;
            else al = nxt == NONE64 ? (u64)item + 1 : nxt + 1;
            sink.put(item, tw_store<TwT>(tw, avg), al);
            ++nput;
        }
        if (last_round) break;
        // the resolved lights form a prefix: the next round starts after it
        if (threadIdx.x == 0) {
            u32 a = lfirst, b = nL;
            while (a < b) {
                const u32 mid = (a + b) >> 1;
                if (P.LS[mid] != 0) a = mid + 1;
                else b = mid;
            }
            P.lfirst = a;
        }
        // next round starts at the chunk holding rank jend
        const unsigned upto = __ballot_sync(0xffffffffu, hb != ~0ull && hb <= jend);
        gcur += upto ? 31 - __clz(upto) : 0;
        __syncthreads();
        lfirst = P.lfirst;
        if (threadIdx.x == 0) P.next_item = NONE64;
        jcur = jend;
        __syncthreads();
    }
    // lights: unresolved ones alias the first heavy past the section (or
    // themselves).  The light keys are no longer needed: their space maps
    // each tile position to its light rank, so that consecutive threads write
    // consecutive rows (8 sectors per warp store instead of 32).
    if (u < nt) {
        unsigned short *LR = reinterpret_cast<unsigned short *>(P.LK);
        __syncthreads();  // every light key read (merge) before the space is reused
        const u32 p0 = wid * CH + lane * VV;
#pragma unroll
        for (int q = 0; q < VV; ++q)
            LR[p0 + q] = ((lm >> q) & 1) ? (unsigned short)(lrank0 + __popc(lm & ((1u << q) - 1)))
                                         : (unsigned short)0xFFFFu;
        __syncthreads();
        const u64 t0 = u * TILE;
        const u64 dflt = after == NONE64 ? 0 : after + 1;  // 0: self
#pragma unroll
        for (int k = 0; k < TILE / TB; ++k) {
            const u32 p = k * TB + threadIdx.x;
            const u32 r = LR[p];
            if (r != 0xFFFFu) {
                const u32 s = P.LS[r];
                const u64 al = s ? (u64)s : (dflt ? dflt : t0 + p + 1);
                sink.put(t0 + p, (TwT)w[t0 + p], al);
                ++nput;
            }
        }
    }
    if constexpr (Sink::counts) {
        __shared__ u32 s_put;
        if (threadIdx.x == 0) s_put = 0;
        __syncthreads();
        const u32 wsum = __reduce_add_sync(0xffffffffu, nput);
        if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(&s_put, wsum);
        __syncthreads();
        if (threadIdx.x == 0 && s_put) atomicAdd(sink.written, (unsigned long long)s_put);
    }
}

template <typename T, typename Sink>
int run_build(const void *wv, u64 n, double avg, Sink sink, void *ws, cudaStream_t st)
{
    const T *w = (const T *)wv;
    BuildWs W = carve(ws, n);
    SplitOut O;
    {
        char *tail = (char *)ws + ws_bytes_for(n) - split_bytes(n);
        O.hrank = (u64 *)tail;
        O.hchunk = O.hrank + (W.nt + 2);
        O.hitem = O.hchunk + (W.nt + 2);
    }
    {
        int rc = ak_fill_small(W.counter, 0, 256, st);
        if (rc == AK_OK) rc = ak_fill_small(W.status, 0, W.nst * 4, st);
        if (rc != AK_OK) return rc;
    }
    AK_SMEM_ATTR(k_build_scan<T>, (int)ScanBuf<T>::BYTES);
    k_build_scan<T><<<(unsigned)W.nst, SC_WARPS * 32, ScanBuf<T>::BYTES, st>>>(w, n, avg, W);
    AK_LAUNCH_CHECK("k_build_scan");
    k_build_coarse<<<(unsigned)((W.nt + 1 + 255) / 256), 256, 0, st>>>(W, n);
    AK_LAUNCH_CHECK("k_build_coarse");
    k_build_split<T><<<(unsigned)((W.nt + 1 + NW - 1) / NW), TB, 0, st>>>(w, n, avg, W, O);
    AK_LAUNCH_CHECK("k_build_split");
    const size_t smem = sizeof(SecSmem);
    AK_SMEM_ATTR((k_build_pack<T, Sink>), (int)smem);
    const u32 pf = ak_resident_ctas((const void *)k_build_pack<T, Sink>, TB, smem);  // queried once
    k_build_pack<T, Sink><<<(unsigned)(W.nt + 1), TB, smem, st>>>(w, n, avg, W, O, sink, pf);
    AK_LAUNCH_CHECK("k_build_pack");
    return AK_OK;
}

}  // namespace

extern "C" {

size_t ak_build_workspace_bytes(uint64_t n, int dtype)
{
    (void)dtype;
    return ws_bytes_for(n);
}

int ak_build_psa(const void *w, int dtype, uint64_t n, double total, void *rows, void *ws,
                 size_t ws_bytes, void *stream)
{
    return ak_build_psa_avg(w, dtype, n, total / (double)n, rows, ws, ws_bytes, stream);
}

int ak_build_psa_avg(const void *w, int dtype, uint64_t n, double avg, void *rows, void *ws,
                     size_t ws_bytes, void *stream)
{
    if (n == 0) return AK_ERR_EMPTY_INPUT;
    if (ws_bytes < ws_bytes_for(n)) return AK_ERR_WORKSPACE;
    if (((uintptr_t)w & 15) != 0 || ((uintptr_t)rows & 15) != 0) return AK_ERR_VALUE;
    cudaStream_t st = ak_stream(stream);
    if (dtype == AK_F32) {
        if (n >= 0xFFFFFFFFull) return AK_ERR_VALUE;  // u32 aliases
        return run_build<float>(w, n, avg, RowSink<float>{(RowF32 *)rows}, ws, st);
    }
    if (dtype == AK_F64) {
        if (n >= 0xFFFFFFFFull) return AK_ERR_VALUE;  // u32 item ids in the pack windows
        return run_build<double>(w, n, avg, RowSink<double>{(RowF64 *)rows}, ws, st);
    }
    return AK_ERR_VALUE;
}

int ak_build_psa_residual(const double *res_w, uint64_t k, double avg, const int64_t *res_idx,
                          int out_dtype, void *rows, uint64_t *written, void *ws, size_t ws_bytes,
                          void *stream)
{
    *written = 0;
    if (k == 0) return AK_OK;
    if (ws_bytes < ws_bytes_for(k)) return AK_ERR_WORKSPACE;
    if (((uintptr_t)res_w & 15) != 0 || k >= 0xFFFFFFFFull) return AK_ERR_VALUE;
    if (out_dtype != AK_F32 && out_dtype != AK_F64) return AK_ERR_VALUE;
    cudaStream_t st = ak_stream(stream);
    unsigned long long *c = (unsigned long long *)ak_stream_scratch(st);
    if (!c) return AK_ERR_CUDA;
    int rc = ak_fill_small(c, 0, 8, st);
    if (rc != AK_OK) return rc;
    if (out_dtype == AK_F32)
        rc = run_build<double>(res_w, k, avg, RemapSink<RowF32>{(RowF32 *)rows, res_idx, avg, c}, ws, st);
    else
        rc = run_build<double>(res_w, k, avg, RemapSink<RowF64>{(RowF64 *)rows, res_idx, avg, c}, ws, st);
    if (rc != AK_OK) return rc;
    unsigned long long h = 0;
    rc = ak_readback(st, &h, c, sizeof(h));
    *written = h;
    return rc;
}

int ak_build_stats(const void *ws, uint64_t n, uint64_t *nl, uint64_t *nh, uint64_t *tiles,
                   void *stream)
{
    BuildWs W = carve(const_cast<void *>(ws), n);
    u64 k = 0;
    cudaStream_t st = ak_stream(stream);
    {
        const int rc = ak_readback(st, &k, W.kL + W.nt, sizeof(u64));
        if (rc != AK_OK) return rc;
    }
    *nl = k;
    *nh = n - k;
    *tiles = W.nt;
    return AK_OK;
}

}  // extern "C"
