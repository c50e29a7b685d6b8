// ak_build.cu — fused PSA construction (psa_construct, pack.py:255-277).
//
// Formulation.  Let d = avg - w (light deficit) and e = w - avg (heavy
// excess).  The sequential construction (seqbuild.py:33-58) is a merge of
// two sorted key sequences: light k has key DL(k) = sum of the deficits of
// the lights before it, heavy j has key DH(j) = sum of the excess of the
// heavies up to and including it; heavy j closes before light k iff
// DH(j) <= DL(k).  Hence
//   light k:  alias = first heavy (item order) with DH > DL(k), else itself;
//   heavy j:  tw = avg + DH(j) - DL(first light with DL >= DH(j)),
//             alias = next heavy, or itself when it is the last;
// and the reference's split predicate L[n-h] + H[h] <= n*avg (split.py:69-77)
// is exactly DH(h) <= DL(n-h).  Every row follows from prefix sums.
//
// Exact fixed-point keys.  With e_avg = ilogb(avg), u0 = 2^(e_avg-53) and
// A = avg/u0 (an integer in [2^53, 2^54)), every weight becomes the integer
// v = w/u0 (exact for f32 weights >= 2^-30 avg and f64 weights >= avg/2,
// rounded half up below), a light contributes A - v < 2^54 and a heavy
// v - A.  Keys are exact integer sums, hence associative: any kernel
// recomputes any key bit-identically from a chunk base plus an in-chunk
// prefix, with no canonical-scan or compensated-sum machinery, and the table
// equals Vose's sequential order carried out in exact arithmetic (oracle
// diagnostic ako_vose_fixed; f64 thresholds rounded once).
//
// Pipeline (three kernels; a chunk is 512 items = one warp, 16 per lane):
//  1. k_b2_scan   one read of the weights: per chunk the light count, the
//                 light deficit sum (u64) and the heavy excess sum (u128);
//                 CTA tiles of 64 chunks with a single-pass decoupled
//                 look-back; writes the exclusive chunk bases DLb, DHb
//                 (u128), the light counts kL and each chunk's first heavy.
//  2. k_b2_split  PSA split at every segment of 16 chunks: the first chunk
//                 each partner finder starts from (binary search of bases).
//  3. k_b2_pack   one warp per segment (dynamic order), per own chunk r:
//                 - own keys from the chunk's weights (registers);
//                 - merge A: every own light's successor heavy, from a
//                   partner-heavy list (one chunk's heavies: keys + items in
//                   shared memory) that advances through the heavy sequence;
//                 - merge B: every own heavy's successor light key, from a
//                   partner-light list advancing through the light sequence;
//                 - every row of the chunk written by its owner lane as full
//                   32-byte sectors (STG.256).  A partially written sector
//                   costs the L2 a fill read (2.2-4.5x slower writes,
//                   measured: tools/ubench/ops.cu), so no row is written by
//                   anyone but its owner.
//  DRAM traffic: the weights twice (scan; own chunk — partner chunks are
//  re-read from L2, being the neighbours of chunks in flight) and every row
//  once = the algorithmic bytes.
#include <cstring>

#include "ak_common.cuh"

namespace {

typedef unsigned __int128 u128;
typedef __int128 i128;

constexpr int CH = 512;                    // items per chunk = section = partner chunk
constexpr int LV = CH / 32;                // items per lane of the warp that owns a chunk
constexpr int SC_WARPS = 8;                // scan CTA warps (one chunk per warp at a time)
constexpr int SC_CPW = 4;                  // chunks per scan warp per tile
constexpr int SC_TCH = SC_WARPS * SC_CPW;  // chunks per scan tile (one per lane of warp 0)
static_assert(SC_TCH == 32, "the tile scan gives each lane of warp 0 one chunk");
constexpr int SEG = 4;                     // sections per pack segment
constexpr int PK_WARPS = 4;                // warps per pack CTA (independent)
constexpr u64 SAT = ~0ull;
constexpr u64 NOITEM = ~0ull;
constexpr unsigned short NOFH = 0xFFFF;

// ---------------------------------------------------------------------------
// fixed-point parameters
// ---------------------------------------------------------------------------
struct Keys {
    u64 A;       // avg / u0
    int K;       // v = m << (E - K)
    u32 avgf;    // f32: bits of the largest float <= avg
    u64 avgd;    // f64: bits of avg
    double avg;
    double u0;     // 2^(e_avg - 53)
    double scale;  // 2^(53 - e_avg) = 1 / u0
};

Keys make_keys(double avg, bool f32)
{
    Keys P;
    const int e = ilogb(avg);
    P.A = (u64)ldexp(avg, 53 - e);
    P.K = f32 ? 97 + e : 1022 + e;
    float af = (float)avg;
    while ((double)af > avg) af = nextafterf(af, 0.0f);
    u32 ab;
    memcpy(&ab, &af, 4);
    P.avgf = ab;
    memcpy(&P.avgd, &avg, 8);
    P.avg = avg;
    P.u0 = ldexp(1.0, e - 53);
    P.scale = ldexp(1.0, 53 - e);
    return P;
}

template <typename T> struct WT;
template <> struct WT<float> {
    typedef u32 B;
    typedef RowF32 Row;
};
template <> struct WT<double> {
    typedef u64 B;
    typedef RowF64 Row;
};

// v = w / u0 from the weight's bits, rounded to the nearest integer with ties
// to even (exact for every f32 weight >= 2^-30 avg, f64 weight >= avg/2);
// `wide`: v >= 2^64 (the returned value is then invalid)
__device__ __forceinline__ u64 fixv(u32 b, const Keys &P, bool &wide)
{
    u32 E = b >> 23;  // weights are positive and finite (validated upstream)
    u32 m = b & 0x7FFFFFu;
    if (E) m |= 0x800000u;
    else E = 1;
    const int sh = (int)E - P.K;
    if (sh >= 0) {
        wide = sh > 40;
        return (u64)m << (sh & 63);
    }
    const int r = -sh;
    if (r > 24) return 0ull;  // below half a unit
    const u64 q = (u64)m >> r, rem = (u64)m & ((1ull << r) - 1), half = 1ull << (r - 1);
    return q + (rem > half || (rem == half && (q & 1)));
}
// f64: exact scaling, then a round-to-nearest-even conversion
__device__ __forceinline__ u64 fixv(u64 b, const Keys &P, bool &wide)
{
    const double x = __longlong_as_double((long long)b) * P.scale;
    wide = x >= 18446744073709551616.0;
    return __double2ull_rn(x);
}

// the general f32 decode (tiny weights rounded, wide ones flagged), out of
// line: it is rare and the pack's hot code must stay small
__device__ __noinline__ void decode_slow(const u32 (&b)[LV], u32 valid, const Keys &P, u64 (&v)[LV])
{
    for (int q = 0; q < LV; ++q) {
        bool wd = false;
        v[q] = ((valid >> q) & 1) ? fixv(b[q], P, wd) : 0ull;
    }
}

// v for the lane's LV items (valid ones; others 0): f32 takes an integer
// fast path when every item of the warp has 0 <= E - K <= 40 (no rounding,
// no overflow), f64 one multiply and one conversion per item
__device__ __forceinline__ void decode(const u32 (&b)[LV], u32 valid, const Keys &P, u64 (&v)[LV])
{
    int emin = 255, emax = 0;
#pragma unroll
    for (int q = 0; q < LV; ++q) {
        const int E = ((valid >> q) & 1) ? (int)(b[q] >> 23) : P.K;
        emin = E < emin ? E : emin;
        emax = E > emax ? E : emax;
    }
    if (__all_sync(0xffffffffu, emin >= P.K && emin >= 1 && emax <= P.K + 40)) {
#pragma unroll
        for (int q = 0; q < LV; ++q) {
            const u64 m = (b[q] & 0x7FFFFFu) | 0x800000u;
            v[q] = ((valid >> q) & 1) ? m << ((int)(b[q] >> 23) - P.K) : 0ull;
        }
    } else {
        decode_slow(b, valid, P, v);
    }
}
__device__ __forceinline__ void decode(const u64 (&b)[LV], u32 valid, const Keys &P, u64 (&v)[LV])
{
#pragma unroll
    for (int q = 0; q < LV; ++q) {
        bool wd = false;
        v[q] = ((valid >> q) & 1) ? fixv(b[q], P, wd) : 0ull;
    }
}

// the exact excess v - A of any heavy
__device__ __forceinline__ u128 excess_exact(u32 b, const Keys &P)
{
    const int sh = (int)(b >> 23) - P.K;  // heavies: sh >= 30
    return ((u128)((b & 0x7FFFFFu) | 0x800000u) << sh) - P.A;
}
__device__ __forceinline__ u128 excess_exact(u64 b, const Keys &P)
{
    const int sh = (int)(u32)(b >> 52) - P.K;  // heavies: sh >= 1
    return ((u128)((b & ((1ull << 52) - 1)) | (1ull << 52)) << sh) - P.A;
}
__device__ __forceinline__ bool is_light(u32 b, const Keys &P) { return b <= P.avgf; }
__device__ __forceinline__ bool is_light(u64 b, const Keys &P) { return b <= P.avgd; }

// ---------------------------------------------------------------------------
// workspace
// ---------------------------------------------------------------------------
struct Tab {
    u64 n, nc, ntiles, nseg;
    unsigned *tile_ctr, *seg_ctr;
    u32 *status;                      // [ntiles] 0 none, 1 aggregate, 2 inclusive
    u128 *aggL, *aggH, *incL, *incH;  // [ntiles]
    u32 *aggK, *incK;                 // [ntiles]
    u128 *DLb, *DHb;                  // [nc + 1] exclusive chunk bases
    u32 *kL;                          // [nc + 1] lights before the chunk
    unsigned short *fh;               // [nc] first heavy offset, NOFH if none
    u32 *hstart;                      // [nseg] heavy finder's first chunk
    u32 *cnt;                         // [nc] arrival counts of the pack
    u32 *LAg;                         // [n] light answers by item (L2 scratch)
    void *HTg;                        // [n] heavy thresholds (row bits) by heavy rank
};

inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

template <typename F> void layout(u64 n, size_t tw_bytes, F &&take)
{
    const u64 nc = (n + CH - 1) / CH;
    const u64 nt = (nc + SC_TCH - 1) / SC_TCH;
    const u64 ns = (nc + SEG - 1) / SEG;
    const size_t sz[16] = {256,           nt * 4,       nt * 16, nt * 16, nt * 16,
                           nt * 16,       nt * 4,       nt * 4,  (nc + 1) * 16,
                           (nc + 1) * 16, (nc + 1) * 4, nc * 2,  ns * 4,
                           nc * 4,        n * 4,        n * tw_bytes};
    for (int i = 0; i < 16; ++i) take(i, sz[i]);
}

size_t ws_bytes_for(u64 n, size_t tw_bytes)
{
    size_t off = 0;
    layout(n, tw_bytes, [&](int, size_t b) { off += al256(b); });
    return off;
}

Tab carve(void *ws, u64 n, size_t tw_bytes)
{
    Tab t;
    t.n = n;
    t.nc = (n + CH - 1) / CH;
    t.ntiles = (t.nc + SC_TCH - 1) / SC_TCH;
    t.nseg = (t.nc + SEG - 1) / SEG;
    char *p[16];
    size_t off = 0;
    layout(n, tw_bytes, [&](int i, size_t b) {
        p[i] = (char *)ws + off;
        off += al256(b);
    });
    t.tile_ctr = (unsigned *)p[0];
    t.seg_ctr = (unsigned *)p[0] + 1;
    t.status = (u32 *)p[1];
    t.aggL = (u128 *)p[2];
    t.aggH = (u128 *)p[3];
    t.incL = (u128 *)p[4];
    t.incH = (u128 *)p[5];
    t.aggK = (u32 *)p[6];
    t.incK = (u32 *)p[7];
    t.DLb = (u128 *)p[8];
    t.DHb = (u128 *)p[9];
    t.kL = (u32 *)p[10];
    t.fh = (unsigned short *)p[11];
    t.hstart = (u32 *)p[12];
    t.cnt = (u32 *)p[13];
    t.LAg = (u32 *)p[14];
    t.HTg = (void *)p[15];
    return t;
}

// ---------------------------------------------------------------------------
// loads and stores
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ldg256(const void *p, u64 &a, u64 &b, u64 &c, u64 &d)
{
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p));
}
__device__ __forceinline__ void ldcg256(const void *p, u64 &a, u64 &b, u64 &c, u64 &d)
{
    asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p)
                 : "memory");
}
__device__ __forceinline__ void stg256(void *p, u64 a, u64 b, u64 c, u64 d)
{
    asm volatile("st.global.L1::no_allocate.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(a), "l"(b),
                 "l"(c), "l"(d)
                 : "memory");
}

// 8 consecutive weights from item i0 as raw bits; returns the mask of items < n
__device__ __forceinline__ u32 load8(const float *w, u64 n, u64 i0, u32 (&b)[8])
{
    if (i0 + 8 <= n) {
        u64 x[4];
        ldg256(w + i0, x[0], x[1], x[2], x[3]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            b[2 * k] = (u32)x[k];
            b[2 * k + 1] = (u32)(x[k] >> 32);
        }
        return 0xFFu;
    }
    u32 valid = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const bool ok = i0 + q < n;
        b[q] = ok ? __float_as_uint(w[i0 + q]) : 0u;
        valid |= (u32)ok << q;
    }
    return valid;
}
__device__ __forceinline__ u32 load8(const double *w, u64 n, u64 i0, u64 (&b)[8])
{
    if (i0 + 8 <= n) {
        ldg256(w + i0, b[0], b[1], b[2], b[3]);
        ldg256(w + i0 + 4, b[4], b[5], b[6], b[7]);
        return 0xFFu;
    }
    u32 valid = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const bool ok = i0 + q < n;
        b[q] = ok ? (u64)__double_as_longlong(w[i0 + q]) : 0ull;
        valid |= (u32)ok << q;
    }
    return valid;
}

// the lane's LV consecutive weights of chunk c as raw bits (mask of items < n)
template <typename T>
__device__ __forceinline__ u32 load_lane(const T *w, u64 n, u64 c, int lane,
                                         typename WT<T>::B (&b)[LV])
{
    const u64 i0 = c * CH + (u64)lane * LV;
    u32 valid = 0;
#pragma unroll
    for (int g = 0; g < LV / 8; ++g) {
        typename WT<T>::B t[8];
        valid |= load8(w, n, i0 + 8 * g, t) << (8 * g);
#pragma unroll
        for (int q = 0; q < 8; ++q) b[8 * g + q] = t[q];
    }
    return valid;
}

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64 shfl_u64(u64 x, int src)
{
    return ((u64)__shfl_sync(0xffffffffu, (u32)(x >> 32), src) << 32) |
           __shfl_sync(0xffffffffu, (u32)x, src);
}
__device__ __forceinline__ u64 shfl_up_u64(u64 x, int d)
{
    return ((u64)__shfl_up_sync(0xffffffffu, (u32)(x >> 32), d) << 32) |
           __shfl_up_sync(0xffffffffu, (u32)x, d);
}
__device__ __forceinline__ u64 shfl_xor_u64(u64 x, int m)
{
    return ((u64)__shfl_xor_sync(0xffffffffu, (u32)(x >> 32), m) << 32) |
           __shfl_xor_sync(0xffffffffu, (u32)x, m);
}
__device__ __forceinline__ u128 shfl_u128(u128 x, int src)
{
    return ((u128)shfl_u64((u64)(x >> 64), src) << 64) | shfl_u64((u64)x, src);
}
__device__ __forceinline__ u128 shfl_up_u128(u128 x, int d)
{
    return ((u128)shfl_up_u64((u64)(x >> 64), d) << 64) | shfl_up_u64((u64)x, d);
}
__device__ __forceinline__ u128 shfl_xor_u128(u128 x, int m)
{
    return ((u128)shfl_xor_u64((u64)(x >> 64), m) << 64) | shfl_xor_u64((u64)x, m);
}

// exclusive warp scans (sums that cannot overflow their type)
__device__ __forceinline__ u64 warp_excl_u64(u64 x, int lane, u64 &total)
{
    u64 inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u64 y = shfl_up_u64(inc, d);
        if (lane >= d) inc += y;
    }
    total = shfl_u64(inc, 31);
    return inc - x;
}
__device__ __forceinline__ u128 warp_excl_u128(u128 x, int lane, u128 &total)
{
    u128 inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u128 y = shfl_up_u128(inc, d);
        if (lane >= d) inc += y;
    }
    total = shfl_u128(inc, 31);
    return inc - x;
}
__device__ __forceinline__ u32 warp_excl_u32(u32 x, int lane, u32 &total)
{
    u32 inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
    }
    total = __shfl_sync(0xffffffffu, inc, 31);
    return inc - x;
}

// u128 table entries: written by other CTAs (the scan's look-back, the
// previous kernel): read from L2 so no stale L1 line is ever seen
__device__ __forceinline__ u128 ld_u128(const u128 *p)
{
    u64 lo, hi;
    asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
    return ((u128)hi << 64) | lo;
}
__device__ __forceinline__ void st_u128(u128 *p, u128 x)
{
    *reinterpret_cast<uint4 *>(p) =
        make_uint4((u32)x, (u32)((u64)x >> 32), (u32)(x >> 64), (u32)(x >> 96));
}

// max c in [lo, hi] with pred(c), given pred(lo) and pred monotone
// (true..true false..false): one probe per lane per round, a window of 32
// after lo first (the finder usually moves by a chunk or two).  Warp-collective.
template <typename F>
__device__ __forceinline__ u64 warp_last_true(u64 lo, u64 hi, int lane, F &&pred)
{
    {
        const u64 h1 = hi < lo + 32 ? hi : lo + 32;
        const u64 pos = lo + 1 + (u64)lane;
        const unsigned b = __ballot_sync(0xffffffffu, pos <= h1 && pred(pos));
        const u64 c = lo + (u64)__popc(b);
        if (c < h1 || h1 == hi) return c;
        lo = h1;
    }
    while (lo < hi) {
        const u64 st = (hi - lo + 31) / 32;
        const u64 pos = lo + st * (u64)(lane + 1);
        const unsigned b = __ballot_sync(0xffffffffu, pos <= hi && pred(pos));
        lo += st * (u64)__popc(b);
        const u64 h2 = lo + st - 1;
        hi = h2 < hi ? h2 : hi;
    }
    return lo;
}

// ---------------------------------------------------------------------------
// 1. scan + decoupled look-back
// ---------------------------------------------------------------------------
// One warp per chunk (32 items per lane, read as four 256-bit loads each),
// per chunk: light count, light deficit sum (< 2^64), heavy excess sum (u128).
// Sums are formed from S_all = sum v and S_light = sum over lights of v when
// every v < 2^58 (no 64-bit overflow); else exactly in 128 bits (rare).
template <typename T>
__global__ void __launch_bounds__(SC_WARPS * 32) k_b2_scan(const T *__restrict__ w, Keys P, Tab tb)
{
    typedef typename WT<T>::B B;
    __shared__ u64 sL[SC_TCH];
    __shared__ u128 sH[SC_TCH];
    __shared__ u32 sK[SC_TCH];
    __shared__ unsigned short sF[SC_TCH];
    __shared__ unsigned s_tile;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(tb.tile_ctr, 1u);
    __syncthreads();
    const u64 tile = s_tile;
    const u64 c0 = tile * SC_TCH;
    const u64 nct = (c0 + SC_TCH <= tb.nc) ? SC_TCH : tb.nc - c0;
    const u64 n = tb.n;

    for (int k = 0; k < SC_CPW; ++k) {
        const u64 j = (u64)wid + (u64)k * SC_WARPS;
        if (j >= nct) break;
        B b[LV];
        const u32 valid = load_lane(w, n, c0 + j, lane, b);
        u64 v[LV];
        decode(b, valid, P, v);
        u32 lm = 0;
        u64 sall = 0, slight = 0, vor = 0;
        bool anywide = false;
#pragma unroll
        for (int q = 0; q < LV; ++q) {
            const bool ok = (valid >> q) & 1;
            const bool li = ok && is_light(b[q], P);
            lm |= (u32)li << q;
            sall += v[q];
            slight += li ? v[q] : 0ull;
            vor |= v[q];
        }
        if (sizeof(B) == 4) {
            // an f32 heavy with E - K > 40 is wide (v >= 2^64, not representable)
#pragma unroll
            for (int q = 0; q < LV; ++q) anywide |= ((valid >> q) & 1) && (int)((u32)b[q] >> 23) - P.K > 40;
        } else {
#pragma unroll
            for (int q = 0; q < LV; ++q)
                anywide |= ((valid >> q) & 1) && __longlong_as_double((long long)b[q]) * P.scale >= 18446744073709551616.0;
        }
        const u32 hm = valid & ~lm;
        const u32 nl = __popc(lm), nh = __popc(hm);
        u64 sl = (u64)nl * P.A - slight;
        u128 sh;
        if (!__any_sync(0xffffffffu, anywide || (vor >> 58) != 0)) {
            sh = (u128)(sall - slight) - (u128)nh * P.A;  // heavies' v sum >= nh * A
        } else {
            u128 s = 0;
#pragma unroll
            for (int q = 0; q < LV; ++q)
                if ((hm >> q) & 1) s += excess_exact(b[q], P);
            sh = s;
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            sl += shfl_xor_u64(sl, m);
            sh += shfl_xor_u128(sh, m);
        }
        const u32 cnt = __reduce_add_sync(0xffffffffu, nl);
        const unsigned hb = __ballot_sync(0xffffffffu, hm != 0);
        unsigned short f = NOFH;
        if (hb) {
            const int fl = __ffs(hb) - 1;
            const u32 fm = __shfl_sync(0xffffffffu, hm, fl);
            f = (unsigned short)(fl * LV + __ffs(fm) - 1);
        }
        if (lane == 0) {
            sL[j] = sl;
            sH[j] = sh;
            sK[j] = cnt;
            sF[j] = f;
        }
    }
    __syncthreads();
    if (wid != 0) return;

    // warp 0: inclusive scan of the tile's chunk totals (one chunk per lane)
    const u64 ja = (u64)lane;
    const u128 la = ja < nct ? (u128)sL[ja] : 0;
    const u128 ha = ja < nct ? sH[ja] : 0;
    const u32 ka = ja < nct ? sK[ja] : 0;
    u128 xl = la, xh = ha;
    u32 xk = ka;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u128 yl = shfl_up_u128(xl, d), yh = shfl_up_u128(xh, d);
        const u32 yk = __shfl_up_sync(0xffffffffu, xk, d);
        if (lane >= d) {
            xl += yl;
            xh += yh;
            xk += yk;
        }
    }
    const u128 aL = shfl_u128(xl, 31), aH = shfl_u128(xh, 31);
    const u32 aK = __shfl_sync(0xffffffffu, xk, 31);
    if (lane == 0) {
        if (tile == 0) {
            st_u128(&tb.incL[0], aL);
            st_u128(&tb.incH[0], aH);
            tb.incK[0] = aK;
        } else {
            st_u128(&tb.aggL[tile], aL);
            st_u128(&tb.aggH[tile], aH);
            tb.aggK[tile] = aK;
        }
        __threadfence();
        st_release_u32(&tb.status[tile], tile == 0 ? 2u : 1u);
    }
    // decoupled look-back, 32 predecessors at a time (exact integer sums:
    // the association order does not matter)
    u128 eL = 0, eH = 0;
    u32 eK = 0;
    i64 pred = (i64)tile - 1;
    while (pred >= 0) {
        const i64 p = pred - lane;
        u32 s = 2;
        if (p >= 0) {
            do {
                s = ld_acquire_u32(&tb.status[p]);
            } while (s == 0);
        }
        const unsigned incm = __ballot_sync(0xffffffffu, p >= 0 && s == 2);
        const int stop = incm ? __ffs(incm) - 1 : 32;
        u128 cL = 0, cH = 0;
        u32 cK = 0;
        if (p >= 0 && lane < stop) {
            cL = ld_u128(&tb.aggL[p]);
            cH = ld_u128(&tb.aggH[p]);
            cK = __ldcg(&tb.aggK[p]);
        } else if (p >= 0 && lane == stop) {
            cL = ld_u128(&tb.incL[p]);
            cH = ld_u128(&tb.incH[p]);
            cK = __ldcg(&tb.incK[p]);
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            cL += shfl_xor_u128(cL, m);
            cH += shfl_xor_u128(cH, m);
            cK += __shfl_xor_sync(0xffffffffu, cK, m);
        }
        eL += cL;
        eH += cH;
        eK += cK;
        if (stop < 32 || pred - 32 < 0) break;
        pred -= 32;
    }
    if (lane == 0 && tile > 0) {
        st_u128(&tb.incL[tile], eL + aL);
        st_u128(&tb.incH[tile], eH + aH);
        tb.incK[tile] = eK + aK;
        __threadfence();
        st_release_u32(&tb.status[tile], 2u);
    }
    // exclusive chunk bases
    if (ja < nct) {
        const u64 c = c0 + ja;
        st_u128(&tb.DLb[c], eL + xl - la);
        st_u128(&tb.DHb[c], eH + xh - ha);
        tb.kL[c] = eK + xk - ka;
        tb.fh[c] = sF[ja];
    }
    if (c0 + nct == tb.nc && ja + 1 == nct) {
        st_u128(&tb.DLb[tb.nc], eL + xl);
        st_u128(&tb.DHb[tb.nc], eH + xh);
        tb.kL[tb.nc] = eK + xk;
    }
}

// ---------------------------------------------------------------------------
// 2. split: where each segment's heavy finder starts
// ---------------------------------------------------------------------------
// max c in [0, nc] with a[c] <= x (a non-decreasing, a[0] = 0)
__device__ __forceinline__ u64 last_le(const u128 *a, u64 nc, u128 x)
{
    u64 lo = 0, hi = nc;
    while (lo < hi) {
        const u64 mid = (lo + hi + 1) >> 1;
        if (ld_u128(&a[mid]) <= x) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// PSA split at every segment boundary (split.py:69-77): the first heavy with
// DH > DLb[r0] lies in chunk max{c : DHb[c] <= DLb[r0]}.
__global__ void k_b2_split(Tab tb)
{
    const u64 s = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= tb.nseg) return;
    tb.hstart[s] = (u32)last_le(tb.DHb, tb.nc, ld_u128(&tb.DLb[s * SEG]));
}

// ---------------------------------------------------------------------------
// 3. pack
// ---------------------------------------------------------------------------
// A section is one chunk's lights (key range (DLb[s], DLb[s+1]]) together
// with the heavies whose keys fall in that range (other chunks), one warp per
// section.  A merge path over both gives every light its successor heavy and
// every heavy its successor light, hence its threshold.  The rows of chunk c
// need section c's light answers and the thresholds of c's heavies, made by
// the sections their keys fall in; each contributor writes its part to L2
// scratch (LAg by item, HTg by heavy rank), fences and adds to cnt[c]; the
// contributor that completes the count writes the chunk's rows as full
// 32-byte sectors (k2_rows).  Nothing ever waits on another warp.
struct WSmem {
    u64 LK[CH];       // section lights: keys DL - DLb[s], by light rank
    u64 CK[CH];       // partner list: heavy keys relative to cbase (clamped)
    u32 CI[CH];       // partner list: heavy items
    u32 RES[2 * CH];  // merge results: [light rank] successor list index (then item + 1,
                      // 0 = itself); [CH + list index] successor light rank
};

// warp-cooperative searches over sorted u64 (n <= 1024): two 32-way levels
__device__ __forceinline__ u32 coop_count_le(const u64 *a, u32 n, u64 x, int lane)
{
    const u32 p1 = (u32)(lane + 1) * 32 - 1;
    const u32 c1 = __popc(__ballot_sync(0xffffffffu, p1 < n && a[p1] <= x));
    const u32 p2 = c1 * 32 + (u32)lane;
    return c1 * 32 + __popc(__ballot_sync(0xffffffffu, p2 < n && a[p2] <= x));
}
__device__ __forceinline__ u32 coop_count_lt(const u64 *a, u32 n, u64 x, int lane)
{
    const u32 p1 = (u32)(lane + 1) * 32 - 1;
    const u32 c1 = __popc(__ballot_sync(0xffffffffu, p1 < n && a[p1] < x));
    const u32 p2 = c1 * 32 + (u32)lane;
    return c1 * 32 + __popc(__ballot_sync(0xffffffffu, p2 < n && a[p2] < x));
}
// first index whose key exceeds the signed threshold t
__device__ __forceinline__ u32 coop_first_above(const u64 *a, u32 n, i128 t, int lane)
{
    if (t < 0) return 0;
    if ((u128)t >> 64) return n;
    return coop_count_le(a, n, (u64)t, lane);
}

__device__ __forceinline__ u64 items_in(const Tab &tb, u64 c)
{
    const u64 a = c * CH, b = a + CH;
    return (b < tb.n ? b : tb.n) - a;
}
__device__ __forceinline__ u64 heavies_before(const Tab &tb, u64 c)
{
    return (c * CH < tb.n ? c * CH : tb.n) - tb.kL[c];
}

// threshold row bits of a heavy: T = A + DH - DL(successor light) in units u0
__device__ __forceinline__ u32 tw_bits(float, u64 T, const Keys &P)
{
    return __float_as_uint(tw_to_f32((double)T * P.u0, P.avg));
}
__device__ __forceinline__ u64 tw_bits(double, u64 T, const Keys &P)
{
    return (u64)__double_as_longlong((double)T * P.u0);
}

// the rows of chunk c from its weights, its lights' answers (LAg) and its
// heavies' thresholds (HTg); run by the warp that completes cnt[c]
template <typename T>
__device__ __noinline__ void k2_rows(const T *__restrict__ w, const Keys P, const Tab tb,
                                     const u32 *LAg, const typename WT<T>::B *HTg,
                                     typename WT<T>::Row *rows, u64 c)
{
    typedef typename WT<T>::B B;
    typedef typename WT<T>::Row RowT;
    const int lane = threadIdx.x & 31;
    const u64 n = tb.n, nc = tb.nc;
    const u64 i0 = c * CH + (u64)lane * LV;
    B b[LV];
    const u32 valid = load_lane(w, n, c, lane, b);
    u32 lm = 0;
#pragma unroll
    for (int q = 0; q < LV; ++q) lm |= (u32)is_light(b[q], P) << q;
    lm &= valid;
    const u32 hm = valid & ~lm;
    u32 la[LV];
    if (valid == (1u << LV) - 1) {
#pragma unroll
        for (int g = 0; g < LV / 8; ++g) {
            u64 x[4];
            ldcg256(LAg + i0 + 8 * g, x[0], x[1], x[2], x[3]);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                la[8 * g + 2 * k] = (u32)x[k];
                la[8 * g + 2 * k + 1] = (u32)(x[k] >> 32);
            }
        }
    } else {
#pragma unroll
        for (int q = 0; q < LV; ++q) la[q] = ((valid >> q) & 1) ? __ldcg(LAg + i0 + q) : 0u;
    }
    u32 hcnt;
    const u32 hoff = warp_excl_u32((u32)__popc(hm), lane, hcnt);
    const B *ht = HTg + heavies_before(tb, c) + hoff;
    // the first heavy after this lane's items
    const unsigned hbal = __ballot_sync(0xffffffffu, hm != 0);
    const unsigned later = hbal & ~((2u << lane) - 1u);
    const int nlane = later ? __ffs(later) - 1 : 0;
    const int nf = __shfl_sync(0xffffffffu, hm ? __ffs(hm) - 1 : 0, nlane);
    u64 next = NOITEM;
    if (later) {
        next = c * CH + (u64)nlane * LV + nf;
    } else if (hbal) {
        const u64 r2 = c + 1;
        if (r2 < nc && tb.fh[r2] != NOFH) {
            next = r2 * CH + tb.fh[r2];
        } else if (r2 < nc) {
            const u64 h0 = heavies_before(tb, r2);
            if (heavies_before(tb, nc) > h0) {
                const u64 cc = warp_last_true(r2, nc, lane, [&](u64 p) { return heavies_before(tb, p) == h0; });
                next = cc * CH + tb.fh[cc];
            }
        }
    }
    constexpr int WORDS = LV * (int)sizeof(RowT) / 8;
    u64 wd[WORDS];
    u32 k = __popc(hm);
#pragma unroll
    for (int q = LV - 1; q >= 0; --q) {
        const u64 item = i0 + q;
        u64 twb, al;
        if ((hm >> q) & 1) {
            --k;
            if constexpr (sizeof(B) == 4) twb = __ldcg(reinterpret_cast<const unsigned *>(ht) + k);
            else twb = __ldcg(reinterpret_cast<const unsigned long long *>(ht) + k);
            al = next == NOITEM ? item + 1 : next + 1;
            next = item;
        } else {
            twb = (u64)b[q];  // a light keeps its weight (seqbuild.py:39)
            al = la[q] ? (u64)la[q] : item + 1;
        }
        if constexpr (sizeof(T) == 4) {
            wd[q] = (al << 32) | (u32)twb;
        } else {
            wd[2 * q] = twb;
            wd[2 * q + 1] = al;
        }
    }
    // the scratch of chunk c is dead now: drop its L2 lines without a write-back
    // (the LA block is 128-byte aligned; only HT lines wholly inside c's range)
    __syncwarp();
    if (lane < (int)(CH * 4 / 128))
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(LAg + c * CH + lane * 32) : "memory");
    {
        const uintptr_t h0 = (uintptr_t)(HTg + heavies_before(tb, c)), h1 = h0 + (uintptr_t)hcnt * sizeof(B);
        const uintptr_t a0 = (h0 + 127) & ~(uintptr_t)127;
        for (uintptr_t a = a0 + (uintptr_t)lane * 128; a + 128 <= h1; a += 32 * 128)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
    }
    u64 *dst = reinterpret_cast<u64 *>(rows + i0);
    if (valid == (1u << LV) - 1) {
#pragma unroll
        for (int j = 0; j < WORDS; j += 4) stg256(dst + j, wd[j], wd[j + 1], wd[j + 2], wd[j + 3]);
    } else {
#pragma unroll
        for (int q = 0; q < LV; ++q) {
            if ((valid >> q) & 1) {
                if constexpr (sizeof(T) == 4) {
                    dst[q] = wd[q];
                } else {
                    dst[2 * q] = wd[2 * q];
                    dst[2 * q + 1] = wd[2 * q + 1];
                }
            }
        }
    }
}

// rare: a partner chunk whose excess needs 64 bits or more: exact 128-bit
// sums, keys relative to the section's base clamped into [0, SAT]
template <typename B>
__device__ __noinline__ void build_list_wide(const B (&pb)[LV], u32 hm, const Keys &P, WSmem &S,
                                             u32 slot, u32 item0, u128 hb0, u128 DLs, int lane)
{
    u128 esum = 0;
    for (int q = 0; q < LV; ++q)
        if ((hm >> q) & 1) esum += excess_exact(pb[q], P);
    u128 t128;
    u128 rr = warp_excl_u128(esum, lane, t128);
    const i128 off = (i128)hb0 - (i128)DLs;
    for (int q = 0; q < LV; ++q) {
        if ((hm >> q) & 1) {
            rr += excess_exact(pb[q], P);
            const i128 kk = off + (i128)rr;
            S.CK[slot] = kk < 0 ? 0ull : (((u128)kk >> 64) ? SAT : (u64)kk);
            S.CI[slot] = item0 + q;
            ++slot;
        }
    }
}

// the partner list of chunk cc: every heavy's key (relative to cbase) and
// item, in item (= rank) order
template <typename T>
__device__ __forceinline__ void build_list(const T *__restrict__ w, const Keys &P, const Tab &tb,
                                           WSmem &S, u64 cc, u128 DLs, u128 &cbase, u64 &cfor,
                                           u32 &cn, u64 sec, int lane)
{
    typedef typename WT<T>::B B;
    B pb[LV];
    const u32 pvalid = load_lane(w, tb.n, cc, lane, pb);
    const u128 hb0 = ld_u128(&tb.DHb[cc]);
    const bool wide = (ld_u128(&tb.DHb[cc + 1]) - hb0) >> 64 != 0;
    u32 hm = 0;
#pragma unroll
    for (int q = 0; q < LV; ++q) hm |= (u32)!is_light(pb[q], P) << q;
    hm &= pvalid;
    u32 tot;
    u32 slot = warp_excl_u32((u32)__popc(hm), lane, tot);
    const u32 item0 = (u32)(cc * CH + (u64)lane * LV);
    if (!wide) {
        // keys = the chunk-local inclusive excess prefix (exact u64)
        u64 v[LV], esum = 0;
        decode(pb, pvalid, P, v);
#pragma unroll
        for (int q = 0; q < LV; ++q) {
            v[q] = ((hm >> q) & 1) ? v[q] - P.A : 0ull;
            esum += v[q];
        }
        u64 etot;
        u64 erun = warp_excl_u64(esum, lane, etot);
#pragma unroll
        for (int q = 0; q < LV; ++q) {
            erun += v[q];
            if ((hm >> q) & 1) {
                S.CK[slot] = erun;
                S.CI[slot] = item0 + q;
                ++slot;
            }
        }
        cbase = hb0;
        cfor = NOITEM;
    } else {
        build_list_wide(pb, hm, P, S, slot, item0, hb0, DLs, lane);
        cbase = DLs;
        cfor = sec;
    }
    cn = tot;
    __syncwarp();
}

template <typename T>
__global__ void __launch_bounds__(PK_WARPS * 32, 4) k_b2_pack(const T *__restrict__ w, Keys P, Tab tb,
                                                           u32 *LAg, typename WT<T>::B *HTg,
                                                           typename WT<T>::Row *__restrict__ rows)
{
    typedef typename WT<T>::B B;
    extern __shared__ __align__(16) unsigned char pk_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WSmem &S = reinterpret_cast<WSmem *>(pk_smem)[wid];
    const u64 n = tb.n, nc = tb.nc;
    const u128 DHtot = ld_u128(&tb.DHb[nc]);

    // this warp's contribution to chunk cc's arrival count; the completing
    // contribution writes the chunk's rows
    auto arrive = [&](u64 cc, u32 k) {
        __threadfence();  // every lane's scratch writes, device-wide, before the count
        __syncwarp();
        u32 last = 0;
        if (lane == 0) {
            const u32 expect = (u32)(items_in(tb, cc) - (tb.kL[cc + 1] - tb.kL[cc])) + 1u;
            last = atomicAdd(&tb.cnt[cc], k) + k == expect;
        }
        if (__shfl_sync(0xffffffffu, last, 0)) {
            __threadfence();
#ifdef AK_BUILD_STATS
            if (lane == 0) atomicAdd(tb.tile_ctr + 4, 1u);
#endif
            k2_rows<T>(w, P, tb, LAg, HTg, rows, cc);
        }
    };

    for (;;) {
        u64 sg = 0;
        if (lane == 0) sg = atomicAdd(tb.seg_ctr, 1u);
        sg = __shfl_sync(0xffffffffu, (u32)sg, 0);
        if (sg >= tb.nseg) break;
        const u64 s0 = sg * SEG, s1 = s0 + SEG < nc ? s0 + SEG : nc;
        // the heavy finder: chunk c; the list of chunk `cached` in S.CK/S.CI,
        // keys relative to cbase (DHb of the chunk; or a section's base when
        // the chunk's excess needs more than 64 bits: cfor = that section)
        u64 c = tb.hstart[sg];
        u64 cached = NOITEM, cfor = NOITEM;
        u128 cbase = 0;
        u32 cn = 0, cdone = 0;  // list entries below cdone belong to earlier sections

        for (u64 s = s0; s < s1; ++s) {
            // ---- the section's lights: keys DL - DLb[s], compacted by rank
            B b[LV];
            const u32 valid = load_lane(w, n, s, lane, b);
            const u128 DLs = ld_u128(&tb.DLb[s]);
            const bool last_sec = s + 1 == nc;
            u64 v[LV];
            decode(b, valid, P, v);
            u32 lm = 0;
            u64 lsum = 0;
#pragma unroll
            for (int q = 0; q < LV; ++q) {
                const bool li = ((valid >> q) & 1) && is_light(b[q], P);
                lm |= (u32)li << q;
                v[q] = li ? P.A - v[q] : 0ull;  // deficits
                lsum += v[q];
            }
            u64 span;
            u64 run = warp_excl_u64(lsum, lane, span);
            u32 nl;
            const u32 rank0 = warp_excl_u32((u32)__popc(lm), lane, nl);
            {
                u32 rk = rank0;
#pragma unroll
                for (int q = 0; q < LV; ++q) {
                    if ((lm >> q) & 1) S.LK[rk++] = run;
                    run += v[q];
                }
            }
            __syncwarp();

            // ---- rounds: one partner chunk each
            u32 l0 = 0;
            for (;;) {
                if (DHtot <= DLs || c >= nc) {
                    // no heavy closes after these lights: they alias themselves
                    for (u32 i = l0 + lane; i < nl; i += 32) S.RES[i] = 0;
                    break;
                }
                // the chunk holding the first heavy with DH > DLb[s]
                if (!(ld_u128(&tb.DHb[c + 1]) > DLs))
                    c = warp_last_true(c, nc, lane, [&](u64 p) { return ld_u128(&tb.DHb[p]) <= DLs; });
                if (cached != c || (cfor != NOITEM && cfor != s)) {
#ifdef AK_BUILD_STATS
                    if (lane == 0) atomicAdd(tb.tile_ctr + 5, 1u);
#endif
                    build_list(w, P, tb, S, c, DLs, cbase, cfor, cn, s, lane);
                    cached = c;
                    cdone = 0;
                }
                const i128 off = (i128)cbase - (i128)DLs;  // list key + off = DH - DLb[s]
                const u64 offlo = (u64)off;
                const u32 e0 = cdone + coop_first_above(S.CK + cdone, cn - cdone, -off, lane);
                const u32 e1 = last_sec ? cn : e0 + coop_first_above(S.CK + e0, cn - e0, (i128)span - off, lane);
                const bool more = ld_u128(&tb.DHb[c + 1]) < DHtot;
                const bool fin = e1 < cn || !more;
                const u32 next_code = e1 < cn ? S.CI[e1] + 1 : 0u;
                // lights past the list's last heavy wait for the next round
                const u32 l1 = fin ? nl : l0 + coop_count_lt(S.LK + l0, nl - l0, S.CK[cn - 1] + offlo, lane);
                const u32 nA = l1 - l0, nB = e1 - e0;
                // merge path: lights [l0, l1) with heavies [e0, e1), heavy first
                // on ties (DH <= DL)
                const u32 tot = nA + nB;
#ifdef AK_BUILD_STATS
                if (lane == 0) {
                    atomicAdd(tb.tile_ctr + 2, 1u);
                    atomicAdd(tb.tile_ctr + 3, tot);
                }
#endif
                if (tot) {
                    const u32 per = (tot + 31) >> 5;
                    const u32 d0 = (u32)lane * per < tot ? (u32)lane * per : tot;
                    const u32 d1 = d0 + per < tot ? d0 + per : tot;
                    const u64 *LKr = S.LK + l0;
                    const u64 *CKr = S.CK + e0;
                    u32 lo = d0 > nB ? d0 - nB : 0, hi = d0 < nA ? d0 : nA;
                    while (lo < hi) {
                        const u32 mid = (lo + hi + 1) >> 1;
                        if (LKr[mid - 1] < CKr[d0 - mid] + offlo) lo = mid;
                        else hi = mid - 1;
                    }
                    u32 i = lo, j = d0 - lo;
                    u64 av = i < nA ? LKr[i] : SAT;
                    u64 bv = j < nB ? CKr[j] + offlo : SAT;
                    // branch-free steps: one result store and one key load each
                    for (u32 dd = d0; dd < d1; ++dd) {
                        const bool hv = j < nB && (i >= nA || bv <= av);
                        const u32 at = hv ? CH + e0 + j : l0 + i;
                        const u32 val = hv ? l0 + i : (j < nB ? e0 + j : 0xFFFFFFFFu);
                        S.RES[at] = val;
                        i += hv ? 0u : 1u;
                        j += hv ? 1u : 0u;
                        const bool inb = hv ? j < nB : i < nA;
                        const u64 *src = hv ? CKr + j : LKr + i;
                        const u64 x = inb ? *src : SAT;
                        if (hv) bv = inb ? x + offlo : SAT;
                        else av = x;
                    }
                }
                __syncwarp();
                // heavies: thresholds -> HTg (coalesced by rank); a heavy
                // closes at its successor light, or at the next section's first
                if (nB) {
                    B *dst = HTg + heavies_before(tb, c);
                    for (u32 e = e0 + lane; e < e1; e += 32) {
                        const u32 sr = S.RES[CH + e];
                        const u64 dl = sr < nl ? S.LK[sr] : span;
                        dst[e] = tw_bits((T)0, P.A + (S.CK[e] + offlo) - dl, P);
                    }
                }
                // lights: list index -> item + 1
                for (u32 i = l0 + lane; i < l1; i += 32) {
                    const u32 x = S.RES[i];
                    S.RES[i] = x == 0xFFFFFFFFu ? next_code : S.CI[x] + 1;
                }
                cdone = e1;  // the next section's heavies start at e1
                if (nB) arrive(c, nB);
                __syncwarp();
                l0 = l1;
                if (fin) break;
                // the next chunk with heavies
                const u128 hnext = ld_u128(&tb.DHb[c + 1]);
                c = warp_last_true(c + 1, nc, lane, [&](u64 p) { return ld_u128(&tb.DHb[p]) <= hnext; });
            }

            // ---- the section's own light answers -> LAg (by item)
            {
                u32 la[LV];
                u32 rk = rank0;
#pragma unroll
                for (int q = 0; q < LV; ++q) la[q] = ((lm >> q) & 1) ? S.RES[rk++] : 0u;
                const u64 i0 = s * CH + (u64)lane * LV;
                if (valid == (1u << LV) - 1) {
#pragma unroll
                    for (int g = 0; g < LV / 8; ++g)
                        stg256(LAg + i0 + 8 * g, ((u64)la[8 * g + 1] << 32) | la[8 * g],
                               ((u64)la[8 * g + 3] << 32) | la[8 * g + 2],
                               ((u64)la[8 * g + 5] << 32) | la[8 * g + 4],
                               ((u64)la[8 * g + 7] << 32) | la[8 * g + 6]);
                } else {
#pragma unroll
                    for (int q = 0; q < LV; ++q)
                        if ((valid >> q) & 1) LAg[i0 + q] = la[q];
                }
            }
            arrive(s, 1u);
        }
    }
}

template <typename T>
int run_build(const void *wv, u64 n, double avg, void *rows, void *ws, cudaStream_t st)
{
    typedef typename WT<T>::B B;
    const T *w = (const T *)wv;
    const Tab tb = carve(ws, n, sizeof(B));
    const Keys P = make_keys(avg, sizeof(T) == 4);
    AK_CUDA_TRY(cudaMemsetAsync(tb.tile_ctr, 0, 256, st));
    AK_CUDA_TRY(cudaMemsetAsync(tb.status, 0, tb.ntiles * 4, st));
    AK_CUDA_TRY(cudaMemsetAsync(tb.cnt, 0, tb.nc * 4, st));
    k_b2_scan<T><<<(unsigned)tb.ntiles, SC_WARPS * 32, 0, st>>>(w, P, tb);
    AK_LAUNCH_CHECK("k_b2_scan");
    k_b2_split<<<(unsigned)((tb.nseg + 255) / 256), 256, 0, st>>>(tb);
    AK_LAUNCH_CHECK("k_b2_split");
    const size_t smem = PK_WARPS * sizeof(WSmem);
    AK_SMEM_ATTR(k_b2_pack<T>, smem);
    int per_sm = 0;
    AK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_b2_pack<T>, PK_WARPS * 32, smem));
    if (per_sm < 1) per_sm = 1;
    u64 grid = (u64)ak_num_sms() * per_sm;
    const u64 need = (tb.nseg + PK_WARPS - 1) / PK_WARPS;
    if (grid > need) grid = need;
    k_b2_pack<T><<<(unsigned)grid, PK_WARPS * 32, smem, st>>>(w, P, tb, tb.LAg, (B *)tb.HTg,
                                                              (typename WT<T>::Row *)rows);
    AK_LAUNCH_CHECK("k_b2_pack");
    return AK_OK;
}

}  // namespace

extern "C" {

size_t ak_build_workspace_bytes(uint64_t n, int dtype)
{
    return ws_bytes_for(n, dtype == AK_F32 ? 4 : 8);
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
    if (dtype != AK_F32 && dtype != AK_F64) return AK_ERR_VALUE;
    if (ws_bytes < ws_bytes_for(n, dtype == AK_F32 ? 4 : 8)) return AK_ERR_WORKSPACE;
    // 256-bit weight loads and row stores
    if (((uintptr_t)w & 31) != 0 || ((uintptr_t)rows & 31) != 0) return AK_ERR_VALUE;
    if (!(avg > 0.0) || !std::isfinite(avg)) return AK_ERR_VALUE;
    // u32 aliases in f32 rows, u32 item ids in the partner lists
    if (n >= 0xFFFFFFFFull) return AK_ERR_VALUE;
    cudaStream_t st = ak_stream(stream);
    if (dtype == AK_F32) return run_build<float>(w, n, avg, rows, ws, st);
    if (dtype == AK_F64) return run_build<double>(w, n, avg, rows, ws, st);
    return AK_ERR_VALUE;
}

int ak_build_stats(const void *ws, uint64_t n, uint64_t *nl, uint64_t *nh, uint64_t *tiles,
                   void *stream)
{
    const Tab tb = carve(const_cast<void *>(ws), n, 4);  // the table prefix does not depend on it
    u32 k = 0;
    cudaStream_t st = ak_stream(stream);
    AK_CUDA_TRY(cudaMemcpyAsync(&k, tb.kL + tb.nc, sizeof(u32), cudaMemcpyDeviceToHost, st));
    AK_CUDA_TRY(cudaStreamSynchronize(st));
    *nl = k;
    *nh = n - k;
    *tiles = tb.nc;
    return AK_OK;
}

}  // extern "C"
