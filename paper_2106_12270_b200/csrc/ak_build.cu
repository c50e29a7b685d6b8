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
//  3. k_build_split  PSA split: for every section (light tile) boundary, the
//                    heavy rank J = #heavies with key <= DLb[u] (tile from the
//                    coarse merge, chunk from the stored bounds, count from
//                    one chunk's canonical keys).
//  4. k_build_pack   CTA per section: the tile's lights and the heavies of
//                    ranks [J(u), J(u+1)) (any tiles; L2-resident, being the
//                    lights' neighbours in key space) are merged once by a
//                    merge path; each row is written exactly once.
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
constexpr int HCAP = 1408;       // heavies per merge round
constexpr int CB = 32;           // chunks enumerated per round
constexpr u32 NONE32 = 0xFFFFFFFFu;

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
// X <= f for normalised X
__device__ __forceinline__ bool le_dd_d(dd X, double f) { return X.hi < f || (X.hi == f && X.lo <= 0.0); }

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
__global__ void __launch_bounds__(TB) k_build_split(const T *__restrict__ w, u64 n, double avg,
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
template <typename T> struct SecSmem {
    double LK[TILE];               // own light keys (own frame), rank order
    dd HK[HCAP];                   // heavy keys (own frame)
    u32 HI[HCAP];                  // heavy items
    u32 LS[TILE];                  // light successor item (+1), 0 = unresolved
    unsigned short SL[HCAP];       // heavy -> successor light index
    u64 cbase[CB + 1];             // heavy rank of each enumerated chunk's first heavy
    u32 lcnt[NW];
    u32 lfirst;
    u64 next_item;                 // item of the heavy ranked jend (first of the next round)
};

template <typename T>
__global__ void __launch_bounds__(TB, 4) k_build_pack(const T *__restrict__ w, u64 n, double avg,
                                                      BuildWs W, SplitOut O,
                                                      typename RowOf<T>::type *__restrict__ rows)
{
    typedef typename RowOf<T>::type RowT;
    typedef decltype(RowT::tw) TwT;
    typedef decltype(RowT::alias) AliasT;
    extern __shared__ __align__(16) unsigned char sec_smem[];
    SecSmem<T> &P = *reinterpret_cast<SecSmem<T> *>(sec_smem);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u64 nt = W.nt;
    const u64 u = blockIdx.x;  // section; u == nt: the heavies past every light
    const u64 J0 = O.hrank[u], J1 = u < nt ? O.hrank[u + 1] : heavies_before_tile(W, n, nt);
    const u64 after = u < nt ? O.hitem[u + 1] : NONE64;  // first heavy past the section
    const dd own = u < nt ? W.DLb[u] : W.DLb[nt];
    const double secbound = u < nt ? W.mD[u * NW + NW - 1] : 0.0;  // next light key, own frame

    // ---- lights of tile u (rank order = key order)
    u32 nL = 0, lrank0 = 0, lm = 0;
    double lk[VV], lv[VV];
    if (u < nt) {
        if (lane == 0) P.lcnt[wid] = W.mcl[u * NW + wid];
        load8(w, n, u * TILE + (u64)wid * CH + (u64)lane * VV, lv);
        const double b0 = wid ? W.mD[u * NW + wid - 1] : 0.0, b1 = W.mD[u * NW + wid];
        double ex, tot;
        lane_class<true>(lv, avg, lk, lm, ex, tot, lane);
        class_keys(lk, ex, b0, b1, lane);
        u32 tl;
        const u32 el = warp_excl_count(__popc(lm), tl, lane);
        __syncthreads();
        u32 woff = 0;
        for (int k = 0; k < NW; ++k) {
            woff += k < wid ? P.lcnt[k] : 0;
            nL += P.lcnt[k];
        }
        lrank0 = woff + el;
        u32 r = lrank0;
#pragma unroll
        for (int q = 0; q < VV; ++q)
            if ((lm >> q) & 1) {
                P.LK[r] = lk[q];
                P.LS[r] = 0;
                ++r;
            }
    }
    __syncthreads();

    // ---- heavies in rounds of at most HCAP ranks
    u64 jcur = J0;
    u64 gcur = O.hchunk[u];
    u32 lfirst = 0;  // first light not yet resolved
    while (jcur < J1) {
        // enumerate CB chunks from gcur with the heavy rank of their first heavy
        if (wid == 0) {
            const u64 g = gcur + lane;
            u64 hb = ~0ull;
            u32 hcnt = 0;
            if (g < nt * NW) {
                const u64 t = g / NW;
                const int c = (int)(g % NW);
                hcnt = chunk_valid(n, g) - W.mcl[g];
                u32 pre = 0;
                for (int k = 0; k < c; ++k) pre += chunk_valid(n, t * NW + k) - W.mcl[t * NW + k];
                hb = heavies_before_tile(W, n, t) + pre;
            }
            P.cbase[lane] = hb;
            const u64 last = __shfl_sync(0xffffffffu, hb == ~0ull ? ~0ull : hb + hcnt, 31);
            if (lane == 0) {
                P.cbase[CB] = last;
                P.next_item = NONE64;
            }
        }
        __syncthreads();
        u64 jend = J1 < jcur + HCAP ? J1 : jcur + HCAP;
        if (P.cbase[CB] < jend) jend = P.cbase[CB];
        const u32 nH = (u32)(jend - jcur);
        const bool last_round = jend >= J1;
        // rebuild the chunks covering ranks [jcur, jend], own frame
        for (int ci = wid; ci < CB; ci += NW) {
            const u64 hb = P.cbase[ci], hn = P.cbase[ci + 1];
            if (hb == ~0ull || hb > jend || hn <= jcur) continue;
            const u64 g = gcur + ci;
            const u64 t = g / NW;
            const int c = (int)(g % NW);
            const double base = c ? W.mE[g - 1] : 0.0, bound = W.mE[g];
            const dd D = dd_sub(W.DHb[t], own);
            double v[VV], k[VV], ex, tot;
            u32 m;
            load8(w, n, g * CH + (u64)lane * VV, v);
            lane_class<false>(v, avg, k, m, ex, tot, lane);
            class_keys(k, ex, base, bound, lane);
            u32 tc;
            u64 rr = hb + warp_excl_count(__popc(m), tc, lane);
#pragma unroll
            for (int q = 0; q < VV; ++q)
                if ((m >> q) & 1) {
                    const u32 item = (u32)(g * CH + (u64)lane * VV + q);
                    if (rr >= jcur && rr < jend) {
                        const u32 s = (u32)(rr - jcur);
                        P.HK[s] = add_dd_d(D, k[q]);
                        P.HI[s] = item;
                    } else if (rr == jend) {
                        P.next_item = item;
                    }
                    ++rr;
                }
        }
        __syncthreads();
        if (!last_round && wid == 0 && P.next_item == NONE64) {
            // rank jend lies past the enumerated chunks
            const u64 gl = gcur + CB - 1;
            const u64 nx = next_heavy_after(W, gl / NW, (int)(gl % NW), lane);
            if (lane == 0) P.next_item = nx;
        }
        // merge path: lights [lfirst, nL) with heavies [0, nH); heavy first on ties
        {
            const u32 na = nL - lfirst;
            const u32 total = na + nH;
            const u32 per = (total + TB - 1) / TB;
            const u32 d0 = threadIdx.x * per;
            if (d0 < total) {
                u32 lo = d0 > nH ? d0 - nH : 0, hi = d0 < na ? d0 : na;
                while (lo < hi) {
                    const u32 mid = (lo + hi) >> 1;
                    if (!le_dd_d(P.HK[d0 - mid - 1], P.LK[lfirst + mid])) lo = mid + 1;
                    else hi = mid;
                }
                u32 i = lo, j = d0 - lo;
                const u32 d1 = d0 + per < total ? d0 + per : total;
                for (u32 d = d0; d < d1; ++d) {
                    const bool light = i < na && (j >= nH || !le_dd_d(P.HK[j], P.LK[lfirst + i]));
                    if (light) {
                        if (j < nH) P.LS[lfirst + i] = P.HI[j] + 1;
                        ++i;
                    } else {
                        P.SL[j] = (unsigned short)(lfirst + i);
                        ++j;
                    }
                }
            }
        }
        __syncthreads();
        // heavy rows of this round
        const u64 nxt = last_round ? after : P.next_item;
        for (u32 j = threadIdx.x; j < nH; j += TB) {
            const u32 item = P.HI[j];
            const u32 sl = P.SL[j];
            const double DL = sl < nL ? P.LK[sl] : secbound;
            const dd tw = dd_add_d(add_dd_d(P.HK[j], -DL), avg);
            u64 al;
            if (j + 1 < nH) al = (u64)P.HI[j + 1] + 1;
            else al = nxt == NONE64 ? (u64)item + 1 : nxt + 1;
            RowT row;
            row.tw = tw_store<T>(tw.hi + tw.lo, avg);
            row.alias = (AliasT)al;
            rows[item] = row;
        }
        // the resolved lights form a prefix: the next round starts after it
        if (!last_round && threadIdx.x == 0) {
            u32 a = lfirst, b = nL;
            while (a < b) {
                const u32 mid = (a + b) >> 1;
                if (P.LS[mid] != 0) a = mid + 1;
                else b = mid;
            }
            P.lfirst = a;
        }
        u64 gnext = gcur;
        for (int ci = 0; ci < CB; ++ci) {
            const u64 hb = P.cbase[ci];
            if (hb != ~0ull && hb <= jend) gnext = gcur + ci;
        }
        __syncthreads();
        if (!last_round) lfirst = P.lfirst;
        gcur = gnext;
        jcur = jend;
    }
    // lights: rows written by their owning lanes; unresolved ones alias the
    // first heavy past the section (or themselves)
    if (u < nt) {
        u32 r = lrank0;
#pragma unroll
        for (int q = 0; q < VV; ++q)
            if ((lm >> q) & 1) {
                const u64 item = u * TILE + (u64)wid * CH + (u64)lane * VV + q;
                const u32 s = P.LS[r];
                const u64 al = s ? (u64)s : (after == NONE64 ? item + 1 : after + 1);
                RowT row;
                row.tw = (TwT)lv[q];
                row.alias = (AliasT)al;
                rows[item] = row;
                ++r;
            }
    }
}

template <typename T>
int run_build(const void *wv, u64 n, double total, void *rows, void *ws, cudaStream_t st)
{
    const T *w = (const T *)wv;
    BuildWs W = carve(ws, n);
    const double avg = total / (double)n;
    SplitOut O;
    {
        char *tail = (char *)ws + ws_bytes_for(n) - split_bytes(n);
        O.hrank = (u64 *)tail;
        O.hchunk = O.hrank + (W.nt + 2);
        O.hitem = O.hchunk + (W.nt + 2);
    }
    AK_CUDA_TRY(cudaMemsetAsync(W.counter, 0, 256, st));
    AK_CUDA_TRY(cudaMemsetAsync(W.status, 0, W.nst * 4, st));
    k_build_scan<T><<<(unsigned)W.nst, TB, 0, st>>>(w, n, avg, W);
    AK_LAUNCH_CHECK("k_build_scan");
    k_build_coarse<<<(unsigned)((W.nt + 1 + 255) / 256), 256, 0, st>>>(W, n);
    AK_LAUNCH_CHECK("k_build_coarse");
    k_build_split<T><<<(unsigned)((W.nt + 1 + NW - 1) / NW), TB, 0, st>>>(w, n, avg, W, O);
    AK_LAUNCH_CHECK("k_build_split");
    const size_t smem = sizeof(SecSmem<T>);
    AK_CUDA_TRY(cudaFuncSetAttribute(k_build_pack<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    k_build_pack<T><<<(unsigned)(W.nt + 1), TB, smem, st>>>(w, n, avg, W, O,
                                                           (typename RowOf<T>::type *)rows);
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
