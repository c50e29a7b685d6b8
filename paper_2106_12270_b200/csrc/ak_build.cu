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
// Pipeline (three kernels):
//  1. k_build_scan   one pass over the weights (128-bit loads): classify, chunk
//                    scans, per-tile totals and chunk bounds; a single-pass
//                    decoupled look-back over super-tiles (32 tiles per CTA,
//                    so the inclusive frontier outruns DRAM) produces the
//                    exclusive tile bases DLb[t], DHb[t] (exact double-double
//                    sums) and light counts kL[t].
//  2. k_build_coarse merge of the two tile-boundary sequences: for each tile
//                    the first heavy tile covering its light keys (T1) and
//                    the first light tile covering its heavy keys (S1), and
//                    the first heavy after it (nextH).
//  3. k_build_pack   CTA per tile: rebuild the tile's keys (lights and heavies
//                    key-sorted in shared memory); per class, rebuild the run
//                    of foreign chunks its keys need (L2-resident: the
//                    neighbouring CTAs own them) in the tile's own frame and
//                    merge-path them against the own keys; rows staged in
//                    shared memory and stored once, coalesced.
//  DRAM traffic ~ read w twice + write the rows once = the algorithmic bytes.
#include "ak_common.cuh"

namespace {

constexpr int TB = 256;            // threads per CTA
constexpr int VV = 8;              // items per lane
constexpr int CH = 32 * VV;        // items per chunk (one warp)
constexpr int NW = TB / 32;        // chunks per tile
constexpr int TILE = TB * VV;      // items per tile
constexpr int SUPER = 32;          // tiles per pass-1 CTA (look-back granularity)
constexpr u64 NONE64 = ~0ull;
constexpr unsigned char NOFH = 0xFF;

// ---------------------------------------------------------------------------
// workspace layout
// ---------------------------------------------------------------------------
struct BuildWs {
    u64 nt, nst;  // tiles, super-tiles
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
    u32 *T1, *S1;           // [nt+1]
    u64 *nextH;             // [nt]
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

template <typename F> inline void layout(u64 n, F &&take)
{
    u64 nt = (n + TILE - 1) / TILE;
    u64 nst = (nt + SUPER - 1) / SUPER;
    size_t sizes[19] = {256,          nst * 4,      nst * 16,       nst * 16,       nst * 8,
                        nst * 16,     nst * 16,     nst * 8,        (nt + 1) * 16,  (nt + 1) * 16,
                        (nt + 1) * 8, nt * 8,       nt * NW * 8,    nt * NW * 8,    nt * NW,
                        (nt + 1) * 4, (nt + 1) * 4, nt * 8,         nt * NW * 2};
    for (int i = 0; i < 19; ++i) take(i, sizes[i]);
}

inline BuildWs carve(void *ws, u64 n)
{
    BuildWs W;
    W.nt = (n + TILE - 1) / TILE;
    W.nst = (W.nt + SUPER - 1) / SUPER;
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
    W.S1 = (u32 *)p[16];
    W.nextH = (u64 *)p[17];
    W.mcl = (unsigned short *)p[18];
    return W;
}

size_t ws_bytes_for(u64 n)
{
    size_t off = 0;
    layout(n, [&](int, size_t b) { off += align256(b); });
    return off + 256;
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
        if (lane >= d) x = fmax(x, y);
    }
    return x;
}

// Lane-level part of the canonical chunk scan for one class: per-item local
// prefixes (exclusive for lights, inclusive for heavies), the lane's
// exclusive base within the chunk and the chunk total.
template <bool LIGHT>
__device__ __forceinline__ void lane_class(const double v[VV], double avg, double loc[VV], u32 &mask,
                                           double &excl, double &total, int lane)
{
    double s = 0.0;
    u32 m = 0;
#pragma unroll
    for (int k = 0; k < VV; ++k) {
        const bool valid = v[k] >= 0.0;
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

// Lane sums of one class and the canonical chunk total: a butterfly (xor)
// tree sum, identical in every lane and every kernel.
template <bool LIGHT>
__device__ __forceinline__ double chunk_total(const double v[VV], double avg, u32 &mask)
{
    double s = 0.0;
    u32 m = 0;
#pragma unroll
    for (int k = 0; k < VV; ++k) {
        const bool valid = v[k] >= 0.0;
        const bool in = LIGHT ? (valid && v[k] <= avg) : (valid && v[k] > avg);
        if (in) s = s + (LIGHT ? (avg - v[k]) : (v[k] - avg));
        m |= (u32)in << k;
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) s = s + __shfl_xor_sync(0xffffffffu, s, d);
    mask = m;
    return s;
}

// Canonical keys of one class given the chunk's [base, bound].
__device__ __forceinline__ void class_keys(double loc[VV], double excl, double base, double bound,
                                           int lane)
{
    double B = fmin(base + excl, bound);
    double U = __shfl_down_sync(0xffffffffu, B, 1);
    if (lane == 31) U = bound;
#pragma unroll
    for (int k = 0; k < VV; ++k) loc[k] = fmin(B + loc[k], U);
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

template <typename T>
__global__ void __launch_bounds__(TB) k_build_scan(const T *__restrict__ w, u64 n, double avg,
                                                   BuildWs W)
{
    __shared__ double s_tD[SUPER], s_tE[SUPER];
    __shared__ u32 s_tL[SUPER];
    __shared__ u64 s_fH[SUPER];
    __shared__ unsigned int s_st;
    __shared__ dd s_exD, s_exH, s_agD, s_agH;
    __shared__ u64 s_exK, s_agK;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_st = atomicAdd(W.counter, 1u);
    __syncthreads();
    const u64 st = s_st;
    const u64 t0 = st * SUPER;
    const u64 tn = (t0 + SUPER <= W.nt) ? SUPER : W.nt - t0;

    // each warp owns whole tiles (no per-tile block barrier): 8 chunk totals
    // by butterfly sums, then their monotone scan within the warp
    for (u64 j = wid; j < tn; j += NW) {
        const u64 t = t0 + j;
        double cd = 0.0, ce = 0.0;  // lane c < 8 ends up holding chunk c's totals
        u32 cl = 0;
        unsigned char cf = NOFH;
        double va[VV], vb[VV];
        load8(w, n, t * TILE + (u64)lane * VV, va);
#pragma unroll
        for (int c = 0; c < NW; ++c) {
            double *v = (c & 1) ? vb : va;
            if (c + 1 < NW) load8(w, n, t * TILE + (u64)(c + 1) * CH + (u64)lane * VV, (c & 1) ? va : vb);
            u32 lm, hm;
            const double tD = chunk_total<true>(v, avg, lm);
            const double tE = chunk_total<false>(v, avg, hm);
            u32 nl = __popc(lm);
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) nl += __shfl_xor_sync(0xffffffffu, nl, d);
            const unsigned char fh = first_item(hm, lane);
            if (lane == c) {
                cd = tD;
                ce = tE;
                cl = nl;
                cf = fh;
            }
        }
        // monotone scan of the 8 chunk totals -> chunk bounds
        double x = lane < NW ? cd : 0.0, y = lane < NW ? ce : 0.0;
#pragma unroll
        for (int d = 1; d < NW; d <<= 1) {
            double a = shfl_up_d(x, d), b = shfl_up_d(y, d);
            if (lane >= d) { x = x + a; y = y + b; }
        }
#pragma unroll
        for (int d = 1; d < NW; d <<= 1) {
            double a = shfl_up_d(x, d), b = shfl_up_d(y, d);
            if (lane >= d) { x = fmax(x, a); y = fmax(y, b); }
        }
        if (lane < NW) {
            W.mD[t * NW + lane] = x;
            W.mE[t * NW + lane] = y;
            W.mfh[t * NW + lane] = cf;
            W.mcl[t * NW + lane] = (unsigned short)cl;
        }
        u32 tl = lane < NW ? cl : 0;
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) tl += __shfl_xor_sync(0xffffffffu, tl, d);
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
    // super-tile aggregate: exact double-double sum of the tile totals
    if (threadIdx.x == 0) {
        dd aD = dd_make(0.0), aH = dd_make(0.0);
        u64 aK = 0;
        for (u64 j = 0; j < tn; ++j) {
            aD = dd_add_d(aD, s_tD[j]);
            aH = dd_add_d(aH, s_tE[j]);
            aK += s_tL[j];
        }
        s_agD = aD;
        s_agH = aH;
        s_agK = aK;
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
    __syncthreads();
    // look-back by warp 0
    if (threadIdx.x < 32) {
        dd aD = dd_make(0.0), aH = dd_make(0.0);
        u64 aK = 0;
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
            aD = dd_add(aD, cD);
            aH = dd_add(aH, cH);
            aK += cK;
            if (stop < 32 || pred - 32 < 0) break;
            pred -= 32;
        }
        if (lane == 0) {
            if (st > 0) {
                W.inc_D[st] = dd_add(aD, s_agD);
                W.inc_H[st] = dd_add(aH, s_agH);
                W.inc_k[st] = aK + s_agK;
                __threadfence();
                st_release_u32(&W.status[st], 2u);
            }
            s_exD = aD;
            s_exH = aH;
            s_exK = aK;
        }
    }
    __syncthreads();
    // exclusive bases of the super-tile's tiles
    if (threadIdx.x == 0) {
        dd D = s_exD, H = s_exH;
        u64 K = s_exK;
        for (u64 j = 0; j < tn; ++j) {
            const u64 t = t0 + j;
            W.DLb[t] = D;
            W.DHb[t] = H;
            W.kL[t] = K;
            W.firstH[t] = s_fH[j];
            D = dd_add_d(D, s_tD[j]);
            H = dd_add_d(H, s_tE[j]);
            K += s_tL[j];
        }
        if (t0 + tn == W.nt) {
            W.DLb[W.nt] = D;
            W.DHb[W.nt] = H;
            W.kL[W.nt] = K;
        }
    }
}

// ---------------------------------------------------------------------------
// 2. coarse merge of the tile boundaries
// ---------------------------------------------------------------------------
__global__ void k_build_coarse(BuildWs W, u64 n)
{
    const u64 nt = W.nt;
    u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (u > nt) return;
    {  // T1[u] = max{t in [0, nt] : DHb[t] <= DLb[u]}
        const dd x = W.DLb[u];
        u64 lo = 0, hi = nt;
        while (lo < hi) {
            u64 mid = (lo + hi + 1) >> 1;
            if (dd_le(W.DHb[mid], x)) lo = mid;
            else hi = mid - 1;
        }
        W.T1[u] = (u32)lo;
    }
    {  // S1[u] = max{s in [0, nt] : DLb[s] < DHb[u]}, 0 if none
        const dd y = W.DHb[u];
        if (!dd_lt(W.DLb[0], y)) {
            W.S1[u] = 0;
        } else {
            u64 lo = 0, hi = nt;
            while (lo < hi) {
                u64 mid = (lo + hi + 1) >> 1;
                if (dd_lt(W.DLb[mid], y)) lo = mid;
                else hi = mid - 1;
            }
            W.S1[u] = (u32)lo;
        }
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

// ---------------------------------------------------------------------------
// 3. tile pack: merge-path against the needed foreign chunks
// ---------------------------------------------------------------------------
// One CTA owns one tile (8 warps).  (a) The warps rebuild the tile's
// canonical keys; lights and heavies are laid out key-sorted in shared
// memory.  (b) Per class, the own keys [x_min, x_max] need a contiguous run
// of foreign chunks of the other class (the chunk holding the first key past
// x_min through the one holding the first key past x_max).  Dense path: the
// warps rebuild those chunks' keys once, converted into the tile's own frame
// (exact double-doubles), at offsets known from the pass-1 chunk counts; one
// CTA-wide merge path then gives every own element its successor.  Sparse
// path (the run is too long, e.g. next to a giant heavy): every own element
// gets its target chunk, equal targets form groups, and a warp resolves each
// group against its one chunk.  (c) The rows are stored once, coalesced.
constexpr int MAXSLOT = 4;       // candidate foreign tiles with cached bounds
constexpr int GCAP = 256;        // groups per round (sparse path)
constexpr int FCAP = 1280;       // foreign keys per merge (dense path)
constexpr int MAXRUN = 32;       // foreign chunks per merge (dense path)
constexpr u32 TG_NONE = 0xFFFFFFFFu;

template <typename T> struct PackSmem {
    double OK[TILE];                    // own keys (tile-local): lights [0,nL), heavies [nL,nL+nH)
    typename RowOf<T>::type RW[TILE];   // staged rows
    unsigned short OP[TILE];            // own item offsets
    union {
        struct {                        // dense path
            dd FK[FCAP];                // foreign keys in the own frame
            u32 FI[FCAP];               // foreign heavy items (0-based, low 32 bits)
            u32 off[MAXRUN + 1];        // per-chunk offsets into FK
        } d;
        struct {                        // sparse path
            double F[NW][CH];
            u32 TG[TILE];
            unsigned char FP[NW][CH];
            u32 GT[GCAP];
            unsigned short GS[GCAP + 1];
        } s;
    } u;
    dd SB[MAXSLOT * NW];                // own-frame chunk bounds of the candidate tiles
    dd sent;                            // dense sentinel key (lights: bound after the run)
    u64 sent_item;                      // dense sentinel item (heavies: next heavy after the run)
    u32 cnt[NW], cnt2[NW];
    u32 gA, gB, dense, nf;
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
// f <= X and f < X for normalised X (double vs double-double)
__device__ __forceinline__ bool le_d_dd(double f, dd X) { return f < X.hi || (f == X.hi && X.lo >= 0.0); }
__device__ __forceinline__ bool lt_d_dd(double f, dd X) { return f < X.hi || (f == X.hi && X.lo > 0.0); }
// X <= f and X < f
__device__ __forceinline__ bool le_dd_d(dd X, double f) { return X.hi < f || (X.hi == f && X.lo <= 0.0); }
__device__ __forceinline__ bool lt_dd_d(dd X, double f) { return X.hi < f || (X.hi == f && X.lo < 0.0); }

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

// Canonical (tile-local) keys of one class of chunk (t, c) and their mask.
template <typename T, bool LIGHT>
__device__ __forceinline__ u32 chunk_keys(const T *__restrict__ w, u64 n, double avg,
                                          const BuildWs &W, u64 t, int c, double k[VV], int lane)
{
    const double *mB = LIGHT ? W.mD : W.mE;
    const double base = c ? mB[t * NW + c - 1] : 0.0, bound = mB[t * NW + c];
    double v[VV], ex, tot;
    u32 m;
    load8(w, n, t * TILE + (u64)c * CH + (u64)lane * VV, v);
    lane_class<LIGHT>(v, avg, k, m, ex, tot, lane);
    class_keys(k, ex, base, bound, lane);
    return m;
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

// Target chunk of own key x (tile-local, own frame): the foreign chunk of
// the other class holding the first key past x (ISL: first heavy key > x;
// else first light key >= x), TG_NONE if beyond every chunk.
template <bool ISL>
__device__ u32 target_of(const BuildWs &W, const dd *SB, bool fast, u32 nslot, u64 fT0, u64 fT1,
                         dd DLu, dd DHu, double x)
{
    const u64 nt = W.nt;
    if (fast) {
        u32 a = 0, b = nslot * NW;
        while (a < b) {
            const u32 mid = (a + b) >> 1;
            const bool before = ISL ? !lt_d_dd(x, SB[mid]) : !le_d_dd(x, SB[mid]);
            if (before) a = mid + 1;
            else b = mid;
        }
        if (a < nslot * NW) {
            const u64 t = fT0 + a / NW;
            return t < nt ? (u32)(t * NW + a % NW) : TG_NONE;
        }
        return TG_NONE;
    }
    u64 a = fT0, b = fT1 + 1;
    while (a < b) {
        const u64 mid = (a + b) >> 1;
        bool before;
        if (mid >= nt) before = false;
        else {
            const dd L = ISL ? dd_sub(W.DHb[mid + 1], DLu) : dd_sub(W.DLb[mid + 1], DHu);
            before = ISL ? !lt_d_dd(x, L) : !le_d_dd(x, L);
        }
        if (before) a = mid + 1;
        else b = mid;
    }
    if (a > fT1 || a >= nt) return TG_NONE;
    const dd D = ISL ? dd_sub(W.DHb[a], DLu) : dd_sub(W.DLb[a], DHu);  // foreign base - own base
    const double *mB = (ISL ? W.mE : W.mD) + a * NW;
    int c = 0;
    for (; c < NW - 1; ++c) {
        const dd B = add_dd_d(D, mB[c]);
        if (ISL ? lt_d_dd(x, B) : le_d_dd(x, B)) break;
    }
    return (u32)(a * NW + c);
}

template <typename T, bool ISL>
__device__ void resolve_class(const T *__restrict__ w, u64 n, double avg, const BuildWs &W,
                              PackSmem<T> &P, u64 u, u64 tb, u32 ob, u32 cnt)
{
    typedef typename RowOf<T>::type RowT;
    typedef decltype(RowT::alias) AliasT;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u64 nt = W.nt;
    const dd DLu = W.DLb[u], DHu = W.DHb[u];
    const dd own_base = ISL ? DLu : DHu;
    const u64 fT0 = ISL ? W.T1[u] : W.S1[u];
    const u64 fT1 = ISL ? W.T1[u + 1] : W.S1[u + 1];
    // foreign base - own base: a foreign local key f is f + Dn in the own frame
    auto Dn = [&](u64 t) -> dd { return dd_sub(ISL ? W.DHb[t] : W.DLb[t], own_base); };
    const bool fast = fT1 - fT0 + 1 <= (u64)MAXSLOT;
    const u32 nslot = fast ? (u32)(fT1 - fT0 + 1) : 0;
    if (fast) {
        for (u32 i = threadIdx.x; i < nslot * NW; i += TB) {
            const u64 t = fT0 + i / NW;
            P.SB[i] = t >= nt ? dd_make(INFINITY, 0.0)
                              : add_dd_d(Dn(t), (ISL ? W.mE : W.mD)[t * NW + i % NW]);
        }
    }
    __syncthreads();
    // ---- the run of foreign chunks needed by [x_min, x_max] (warp 0)
    if (wid == 0) {
        u32 ta = 0, tb2 = 0;
        if (lane < 2)
            ta = target_of<ISL>(W, P.SB, fast, nslot, fT0, fT1, DLu, DHu,
                                P.OK[ob + (lane ? cnt - 1 : 0)]);
        const u32 a = __shfl_sync(0xffffffffu, ta, 0);
        u32 b = __shfl_sync(0xffffffffu, ta, 1);
        (void)tb2;
        u32 dense = 0, nf = 0;
        const bool tail_none = b == TG_NONE;
        if (a != TG_NONE) {
            if (tail_none) b = (u32)(nt * NW - 1);
            const u32 len = b >= a ? b - a + 1 : 0;
            if (len >= 1 && len <= (u32)MAXRUN) {
                // per-chunk foreign counts of the run, one lane per chunk
                u32 c = 0;
                if ((u32)lane < len) {
                    const u32 g = a + lane;
                    const u64 cs = (u64)g * CH;
                    const u32 valid = (u32)(n - cs < (u64)CH ? n - cs : (u64)CH);
                    const u32 nlc = W.mcl[g];
                    c = ISL ? valid - nlc : nlc;
                }
                u32 tot;
                const u32 ex = warp_excl_count(c, tot, lane);
                if ((u32)lane <= len) P.u.d.off[lane] = (u32)lane < len ? ex : tot;
                if (tot <= (u32)FCAP) {
                    dense = 1;
                    nf = tot;
                }
            }
        }
        if (dense) {
            if (ISL) {
                const u64 sa = tail_none ? NONE64 : next_heavy_after(W, b / NW, (int)(b % NW), lane);
                if (lane == 0) P.sent_item = sa;
            } else if (lane == 0) {
                P.sent = tail_none ? dd_sub(W.DLb[nt], DHu) : add_dd_d(Dn(b / NW), W.mD[b]);
            }
        }
        if (lane == 0) {
            P.gA = a;
            P.gB = tail_none ? TG_NONE : b;
            P.dense = dense;
            P.nf = nf;
        }
    }
    __syncthreads();
    const u32 gA = P.gA, gB = P.gB;
    if (gA == TG_NONE) {
        // no foreign key past any own key
        for (u32 r = threadIdx.x; r < cnt; r += TB) {
            const u32 pos = P.OP[ob + r];
            if (ISL) {
                P.RW[pos].alias = (AliasT)(tb + pos + 1);
            } else {
                const dd tw = dd_add_d(add_dd_d(dd_neg(dd_sub(W.DLb[nt], DHu)), P.OK[ob + r]), avg);
                P.RW[pos].tw = tw_store<T>(tw.hi + tw.lo, avg);
            }
        }
        __syncthreads();
        return;
    }
    if (P.dense) {
        const u32 nf = P.nf;
        const u32 gEnd = gB == TG_NONE ? (u32)(nt * NW - 1) : gB;
        // rebuild the run's keys, into the own frame
        for (u32 g = gA + wid; g <= gEnd; g += NW) {
            const u64 t = g / NW;
            const int c = (int)(g % NW);
            double k[VV];
            const u32 m = chunk_keys<T, !ISL>(w, n, avg, W, t, c, k, lane);
            u32 tot;
            u32 r = P.u.d.off[g - gA] + warp_excl_count(__popc(m), tot, lane);
            const dd D = Dn(t);
#pragma unroll
            for (int q = 0; q < VV; ++q)
                if ((m >> q) & 1) {
                    P.u.d.FK[r] = add_dd_d(D, k[q]);
                    if (ISL) P.u.d.FI[r] = (u32)((u64)g * CH + lane * VV + q);
                    ++r;
                }
        }
        __syncthreads();
        // merge path: own [0,cnt) with foreign [0,nf); foreign first when
        //   ISL: F <= x (heavy closes before the light);  else F < y
        const u32 total = cnt + nf;
        const u32 per = (total + TB - 1) / TB;
        const u32 d0 = threadIdx.x * per;
        if (d0 < total) {
            u32 lo = d0 > nf ? d0 - nf : 0, hi = d0 < cnt ? d0 : cnt;
            while (lo < hi) {
                const u32 mid = (lo + hi) >> 1;
                const u32 j = d0 - mid - 1;  // own[mid] precedes foreign[j]?
                const dd Fj = P.u.d.FK[j];
                const bool own_first = ISL ? !le_dd_d(Fj, P.OK[ob + mid]) : !lt_dd_d(Fj, P.OK[ob + mid]);
                if (own_first) lo = mid + 1;
                else hi = mid;
            }
            u32 i = lo, j = d0 - lo;
            const u32 d1 = d0 + per < total ? d0 + per : total;
            for (u32 d = d0; d < d1; ++d) {
                bool take_own;
                if (i >= cnt) take_own = false;
                else if (j >= nf) take_own = true;
                else {
                    const dd Fj = P.u.d.FK[j];
                    take_own = ISL ? !le_dd_d(Fj, P.OK[ob + i]) : !lt_dd_d(Fj, P.OK[ob + i]);
                }
                if (!take_own) {
                    ++j;
                    continue;
                }
                const u32 pos = P.OP[ob + i];
                if (ISL) {
                    u64 al;
                    if (j < nf) al = (u64)P.u.d.FI[j] + 1;
                    else al = P.sent_item == NONE64 ? tb + pos + 1 : P.sent_item + 1;
                    P.RW[pos].alias = (AliasT)al;
                } else {
                    const dd DL = j < nf ? P.u.d.FK[j] : P.sent;
                    const dd tw = dd_add_d(add_dd_d(dd_neg(DL), P.OK[ob + i]), avg);
                    P.RW[pos].tw = tw_store<T>(tw.hi + tw.lo, avg);
                }
                ++i;
            }
        }
        __syncthreads();
        return;
    }
    // ---- sparse path: per-element targets, grouped
    for (u32 i = threadIdx.x; i < cnt; i += TB)
        P.u.s.TG[i] = target_of<ISL>(W, P.SB, fast, nslot, fT0, fT1, DLu, DHu, P.OK[ob + i]);
    __syncthreads();
    u32 e0 = 0;
    while (e0 < cnt) {
        const u32 per = (cnt - e0 + TB - 1) / TB;
        const u32 i0 = e0 + threadIdx.x * per, i1 = min(i0 + per, cnt);
        u32 nst = 0;
        for (u32 i = i0; i < i1; ++i) nst += (i == e0 || P.u.s.TG[i] != P.u.s.TG[i - 1]);
        u32 wt;
        const u32 ex = warp_excl_count(nst, wt, lane);
        if (lane == 0) P.cnt2[wid] = wt;
        __syncthreads();
        u32 wbase = 0, tot = 0;
        for (int k = 0; k < NW; ++k) {
            wbase += k < wid ? P.cnt2[k] : 0;
            tot += P.cnt2[k];
        }
        u32 g = wbase + ex;
        for (u32 i = i0; i < i1; ++i)
            if (i == e0 || P.u.s.TG[i] != P.u.s.TG[i - 1]) {
                if (g < GCAP) {
                    P.u.s.GS[g] = (unsigned short)i;
                    P.u.s.GT[g] = P.u.s.TG[i];
                }
                ++g;
            }
        __syncthreads();
        const u32 ngr = tot <= GCAP ? tot : GCAP - 1;
        const u32 e1 = tot <= GCAP ? cnt : P.u.s.GS[GCAP - 1];
        __syncthreads();
        if (threadIdx.x == 0) P.u.s.GS[ngr] = (unsigned short)e1;
        __syncthreads();
        for (u32 gi = wid; gi < ngr; gi += NW) {
            const u32 ga = P.u.s.GS[gi], gb = P.u.s.GS[gi + 1];
            const u32 tgt = P.u.s.GT[gi];
            if (tgt == TG_NONE) {
                for (u32 r = ga + lane; r < gb; r += 32) {
                    const u32 pos = P.OP[ob + r];
                    if (ISL) {
                        P.RW[pos].alias = (AliasT)(tb + pos + 1);
                    } else {
                        const dd tw = dd_add_d(add_dd_d(dd_neg(dd_sub(W.DLb[nt], DHu)), P.OK[ob + r]), avg);
                        P.RW[pos].tw = tw_store<T>(tw.hi + tw.lo, avg);
                    }
                }
                continue;
            }
            const u64 t = tgt / NW;
            const int c = (int)(tgt % NW);
            double *F = P.u.s.F[wid];
            unsigned char *FP = P.u.s.FP[wid];
            double k[VV];
            const u32 m = chunk_keys<T, !ISL>(w, n, avg, W, t, c, k, lane);
            u32 nF;
            u32 r = warp_excl_count(__popc(m), nF, lane);
            __syncwarp();
#pragma unroll
            for (int q = 0; q < VV; ++q)
                if ((m >> q) & 1) {
                    F[r] = k[q];
                    FP[r] = (unsigned char)(lane * VV + q);
                    ++r;
                }
            __syncwarp();
            const dd Do = dd_neg(Dn(t));  // own frame -> foreign frame: x - Dn
            if (ISL) {
                const u64 after = next_heavy_after(W, t, c, lane);
                const u64 fb = t * TILE + (u64)c * CH;
                for (u32 r2 = ga + lane; r2 < gb; r2 += 32) {
                    const dd X = add_dd_d(Do, P.OK[ob + r2]);
                    u32 a = 0, b = nF;  // first heavy key > X
                    while (a < b) {
                        const u32 mid = (a + b) >> 1;
                        if (le_d_dd(F[mid], X)) a = mid + 1;
                        else b = mid;
                    }
                    const u32 pos = P.OP[ob + r2];
                    u64 al;
                    if (a < nF) al = fb + FP[a] + 1;
                    else al = (after == NONE64) ? tb + pos + 1 : after + 1;
                    P.RW[pos].alias = (AliasT)al;
                }
            } else {
                const double bound = W.mD[t * NW + c];
                for (u32 r2 = ga + lane; r2 < gb; r2 += 32) {
                    const dd Y = add_dd_d(Do, P.OK[ob + r2]);
                    u32 a = 0, b = nF;  // first light key >= Y
                    while (a < b) {
                        const u32 mid = (a + b) >> 1;
                        if (lt_d_dd(F[mid], Y)) a = mid + 1;
                        else b = mid;
                    }
                    const double DL = a < nF ? F[a] : bound;
                    const dd tw = dd_add_d(add_dd_d(Y, -DL), avg);
                    P.RW[P.OP[ob + r2]].tw = tw_store<T>(tw.hi + tw.lo, avg);
                }
            }
            __syncwarp();
        }
        __syncthreads();
        e0 = e1;
    }
}

template <typename T>
__global__ void __launch_bounds__(TB, 3) k_build_pack(const T *__restrict__ w, u64 n, double avg,
                                                      BuildWs W,
                                                      typename RowOf<T>::type *__restrict__ rows_out)
{
    typedef typename RowOf<T>::type RowT;
    typedef decltype(RowT::alias) AliasT;
    extern __shared__ __align__(16) unsigned char pack_smem[];
    PackSmem<T> &P = *reinterpret_cast<PackSmem<T> *>(pack_smem);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u64 u = blockIdx.x;
    const u64 tb = u * TILE;
    const u64 cbase = tb + (u64)wid * CH;

    // (a) own tile: classify, counts, then canonical keys into sorted lists
    double v[VV];
    load8(w, n, cbase + (u64)lane * VV, v);
    u32 lm = 0, hm = 0;
#pragma unroll
    for (int k = 0; k < VV; ++k) {
        lm |= (u32)(v[k] >= 0.0 && v[k] <= avg) << k;
        hm |= (u32)(v[k] > avg) << k;
    }
    u32 wl, wh;
    const u32 el = warp_excl_count(__popc(lm), wl, lane);
    const u32 eh = warp_excl_count(__popc(hm), wh, lane);
    if (lane == 0) {
        P.cnt[wid] = wl;
        P.cnt2[wid] = wh;
    }
    __syncthreads();
    u32 offL = 0, offH = 0, nL = 0, nH = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        offL += k < wid ? P.cnt[k] : 0;
        offH += k < wid ? P.cnt2[k] : 0;
        nL += P.cnt[k];
        nH += P.cnt2[k];
    }
    {
        const double bD0 = wid ? W.mD[u * NW + wid - 1] : 0.0, bD1 = W.mD[u * NW + wid];
        const double bE0 = wid ? W.mE[u * NW + wid - 1] : 0.0, bE1 = W.mE[u * NW + wid];
        double kD[VV], kE[VV], exD, exE, tD, tE;
        u32 m1, m2;
        lane_class<true>(v, avg, kD, m1, exD, tD, lane);
        class_keys(kD, exD, bD0, bD1, lane);
        lane_class<false>(v, avg, kE, m2, exE, tE, lane);
        class_keys(kE, exE, bE0, bE1, lane);
        u32 rl = offL + el, rh = nL + offH + eh;
#pragma unroll
        for (int k = 0; k < VV; ++k) {
            const u32 pos = wid * CH + lane * VV + k;
            if ((lm >> k) & 1) {
                P.OK[rl] = kD[k];
                P.OP[rl] = (unsigned short)pos;
                P.RW[pos].tw = (decltype(RowT::tw))v[k];
                ++rl;
            } else if ((hm >> k) & 1) {
                P.OK[rh] = kE[k];
                P.OP[rh] = (unsigned short)pos;
                ++rh;
            }
        }
    }
    __syncthreads();
    // heavy aliases: the next heavy of the tile, else the first heavy after it
    {
        const u64 after = W.nextH[u];
        for (u32 r = threadIdx.x; r < nH; r += TB) {
            const u32 pos = P.OP[nL + r];
            u64 a;
            if (r + 1 < nH) a = tb + P.OP[nL + r + 1] + 1;
            else a = (after == NONE64) ? tb + pos + 1 : after + 1;
            P.RW[pos].alias = (AliasT)a;
        }
    }
    // (b) resolve lights, then heavies
    if (nL) resolve_class<T, true>(w, n, avg, W, P, u, tb, 0, nL);
    if (nH) resolve_class<T, false>(w, n, avg, W, P, u, tb, nL, nH);
    __syncthreads();
    // (c) store the tile's rows: each lane its 8 consecutive rows
    const u64 i0 = cbase + (u64)lane * VV;
    const u32 p0 = wid * CH + lane * VV;
    if (i0 + VV <= n) {
        const uint4 *src = reinterpret_cast<const uint4 *>(&P.RW[p0]);
        uint4 *dst = reinterpret_cast<uint4 *>(rows_out + i0);
#pragma unroll
        for (int q = 0; q < (int)(VV * sizeof(RowT) / 16); ++q) dst[q] = src[q];
    } else {
        for (int k = 0; k < VV; ++k)
            if (i0 + k < n) rows_out[i0 + k] = P.RW[p0 + k];
    }
}

template <typename T>
int run_build(const void *wv, u64 n, double total, void *rows, void *ws, cudaStream_t st)
{
    const T *w = (const T *)wv;
    BuildWs W = carve(ws, n);
    const double avg = total / (double)n;
    AK_CUDA_TRY(cudaMemsetAsync(W.counter, 0, 256, st));
    AK_CUDA_TRY(cudaMemsetAsync(W.status, 0, W.nst * 4, st));
    k_build_scan<T><<<(unsigned)W.nst, TB, 0, st>>>(w, n, avg, W);
    AK_LAUNCH_CHECK("k_build_scan");
    k_build_coarse<<<(unsigned)((W.nt + 1 + 255) / 256), 256, 0, st>>>(W, n);
    AK_LAUNCH_CHECK("k_build_coarse");
    const size_t smem = sizeof(PackSmem<T>);
    AK_CUDA_TRY(cudaFuncSetAttribute(k_build_pack<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    k_build_pack<T><<<(unsigned)W.nt, TB, smem, st>>>(w, n, avg, W, (typename RowOf<T>::type *)rows);
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
    if (n == 0) return AK_ERR_EMPTY_INPUT;
    if (ws_bytes < ws_bytes_for(n)) return AK_ERR_WORKSPACE;
    if (((uintptr_t)w & 15) != 0 || ((uintptr_t)rows & 15) != 0) return AK_ERR_VALUE;
    cudaStream_t st = ak_stream(stream);
    if (dtype == AK_F32) {
        if (n >= 0xFFFFFFFFull) return AK_ERR_VALUE;  // u32 aliases
        return run_build<float>(w, n, total, rows, ws, st);
    }
    if (dtype == AK_F64) {
        if (n >= 0xFFFFFFFFull) return AK_ERR_VALUE;  // u32 item ids in the pack windows
        return run_build<double>(w, n, total, rows, ws, st);
    }
    return AK_ERR_VALUE;
}

int ak_build_stats(const void *ws, uint64_t n, uint64_t *nl, uint64_t *nh, uint64_t *tiles,
                   void *stream)
{
    BuildWs W = carve(const_cast<void *>(ws), n);
    u64 k = 0;
    cudaStream_t st = ak_stream(stream);
    AK_CUDA_TRY(cudaMemcpyAsync(&k, W.kL + W.nt, sizeof(u64), cudaMemcpyDeviceToHost, st));
    AK_CUDA_TRY(cudaStreamSynchronize(st));
    *nl = k;
    *nh = n - k;
    *tiles = W.nt;
    return AK_OK;
}

}  // extern "C"
