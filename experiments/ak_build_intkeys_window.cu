// ak_build.cu — fused PSA construction (psa_construct, pack.py:255-277).
//
// Formulation.  Let d_i = avg - w_i (light deficit) and e_i = w_i - avg (heavy
// excess).  The sequential construction (seqbuild.py:33-58) is a merge of two
// sorted key sequences: light k has key DL(k) = sum of the deficits of the
// lights before it, heavy j has key DH(j) = sum of the excess of the heavies
// up to and including it; heavy j closes before light k iff DH(j) <= DL(k)
// (the loop's `wcur > avg` test, seqbuild.py:38).  Hence
//   light k:  alias = first heavy with DH > DL(k), else itself;
//   heavy j:  tw = avg + DH(j) - DL(first light with DL >= DH(j)),
//             alias = next heavy, or itself when it is the last;
// and the reference's split predicate L[n-h] + H[h] <= n*avg
// (split.py:69-77) is exactly DH(h) <= DL(n-h).
//
// Exact integer keys.  avg = A * 2^ea with A in [2^52, 2^53) (the f64
// mantissa of avg).  Every weight becomes an integer number of units u = 2^ea
// (exact for f32 weights >= 2^-29 avg and for every heavy; the rest round to
// nearest, half up), so deficits A - W and excesses W - A are integers and all
// keys are exact integer prefix sums: monotone by construction, identical in
// every kernel that recomputes them, with no clamps, running maxima or
// double-double frames.  Tile bases are 128-bit; inside a section every key
// that takes part in a decision lies in [0, 2^64) of the section's own frame,
// so the pack runs entirely in u64 (heavy keys modulo 2^64, whose true values
// are known to be in range).  A row's threshold is avg + (key difference)*u,
// rounded once.
//
// Pipeline (three kernels):
//  1. k_build_scan   one pass over the weights, streamed chunk by chunk
//                    through a per-warp ring of shared-memory slots filled by
//                    1-D bulk async copies (TMA): classify, per-tile light
//                    deficit (u64) and light count, per-chunk heavy excess
//                    (u128); a single-pass decoupled look-back over super-
//                    tiles gives the exclusive tile bases DLb[t], DHb[t]
//                    (u128) and light counts kL[t].
//  2. k_build_split  the PSA split (split.py:69-77): for every section (light
//                    tile) boundary X = DLb[u], the first heavy with DH > X:
//                    its item hitem[u] and the key base KB[u] = DH(prev) - X
//                    (mod 2^64) of the window that starts at it.  32 tile
//                    searches per warp in parallel (lane per boundary), then
//                    the chunk from the chunk excess sums, then one chunk.
//  3. k_build_pack   CTA per section u: the tile's lights (keys = exact
//                    in-tile deficit prefixes) and the heavy window
//                    [hitem[u], hitem[u+1]) — exactly the heavies the
//                    section's lights pair with, one contiguous item range —
//                    scanned in rounds of up to 2304 items; per round one
//                    merge path (heavy first on ties) over the resolved
//                    lights; heavy rows written per round, light rows by
//                    position (coalesced) at the end.
//  DRAM traffic ~ read w twice + write the rows once = the algorithmic bytes.
#include "ak_common.cuh"

namespace {

constexpr int TB = 256;            // threads per pack CTA
constexpr int VV = 8;              // items per lane
constexpr int CH = 32 * VV;        // items per chunk (one warp)
constexpr int NW = TB / 32;        // chunks per tile
constexpr int TILE = TB * VV;      // items per tile (= one section's lights)
constexpr int SUPER = 32;          // max tiles per scan CTA (look-back granularity)
constexpr int XG = 32;             // extra window groups per round (warp 0)
constexpr int HCAP = (TB + XG) * VV;  // window items (so heavies) per round: 2304
constexpr u64 NONE64 = ~0ull;
constexpr u64 KEY_INF = ~0ull;

// ---------------------------------------------------------------------------
// 128-bit unsigned integers
// ---------------------------------------------------------------------------
struct u128 {
    u64 lo, hi;
};
__host__ __device__ __forceinline__ u128 mk128(u64 lo, u64 hi = 0)
{
    u128 r;
    r.lo = lo;
    r.hi = hi;
    return r;
}
__device__ __forceinline__ u128 add128(u128 a, u128 b)
{
    u128 r;
    asm("add.cc.u64 %0, %2, %4;\n\taddc.u64 %1, %3, %5;"
        : "=l"(r.lo), "=l"(r.hi)
        : "l"(a.lo), "l"(a.hi), "l"(b.lo), "l"(b.hi));
    return r;
}
__device__ __forceinline__ u128 sub128(u128 a, u128 b)
{
    u128 r;
    asm("sub.cc.u64 %0, %2, %4;\n\tsubc.u64 %1, %3, %5;"
        : "=l"(r.lo), "=l"(r.hi)
        : "l"(a.lo), "l"(a.hi), "l"(b.lo), "l"(b.hi));
    return r;
}
__device__ __forceinline__ bool le128(u128 a, u128 b)
{
    return a.hi < b.hi || (a.hi == b.hi && a.lo <= b.lo);
}
__device__ __forceinline__ u128 shfl128(u128 x, int src)
{
    return mk128(__shfl_sync(0xffffffffu, x.lo, src), __shfl_sync(0xffffffffu, x.hi, src));
}
__device__ __forceinline__ u128 shfl_up128(u128 x, int d)
{
    return mk128(__shfl_up_sync(0xffffffffu, x.lo, d), __shfl_up_sync(0xffffffffu, x.hi, d));
}
__device__ __forceinline__ u128 shfl_xor128(u128 x, int m)
{
    return mk128(__shfl_xor_sync(0xffffffffu, x.lo, m), __shfl_xor_sync(0xffffffffu, x.hi, m));
}

// shifts with PTX semantics: amounts >= 64 give 0 (no C++ undefined behaviour)
__device__ __forceinline__ u64 shl64(u64 x, u32 s)
{
    u64 r;
    asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "r"(s));
    return r;
}
__device__ __forceinline__ u64 shr64(u64 x, u32 s)
{
    u64 r;
    asm("shr.b64 %0, %1, %2;" : "=l"(r) : "l"(x), "r"(s));
    return r;
}

// ---------------------------------------------------------------------------
// weights as integer units of u = 2^ea
// ---------------------------------------------------------------------------
struct Quant {
    double avg;   // A * 2^ea exactly
    double u;     // 2^ea
    double scale; // 2^-ea when representable (f64 fast decode), else 0
    u64 A;        // in [2^52, 2^53)
    int ea;
    int sh32;     // 150 + ea (f32 fast decode)
};

inline Quant make_quant(double avg)
{
    Quant q;
    int e = 0;
    const double f = frexp(avg, &e);  // avg = f * 2^e, f in [0.5, 1)
    q.avg = avg;
    q.A = (u64)ldexp(f, 53);
    q.ea = e - 53;
    q.u = ldexp(1.0, q.ea);
    q.scale = (-q.ea <= 1023 && -q.ea >= -1022) ? ldexp(1.0, -q.ea) : 0.0;
    q.sh32 = 150 + q.ea;
    return q;
}

// mantissa m and exponent e0 with w = m * 2^e0 (w > 0 finite)
__device__ __forceinline__ void split_fp(float w, u64 &m, int &e0)
{
    const u32 b = __float_as_uint(w);
    const int E = (int)(b >> 23);
    m = (u64)((b & 0x7FFFFFu) | (E ? 0x800000u : 0u));
    e0 = (E ? E : 1) - 150;
}
__device__ __forceinline__ void split_fp(double w, u64 &m, int &e0)
{
    const u64 b = (u64)__double_as_longlong(w);
    const int E = (int)(b >> 52);
    m = (b & 0xFFFFFFFFFFFFFull) | (E ? (1ull << 52) : 0ull);
    e0 = (E ? E : 1) - 1075;
}

// W = w / u as an integer (128-bit), rounded to nearest even: exact whenever
// w is a multiple of u (every heavy, every f32 weight >= 2^-29 avg).  The
// generic shift-based decode; the fast paths below equal it wherever they
// apply and defer to it elsewhere.
template <typename T> __device__ __noinline__ u128 units_generic(T w, int ea)
{
    u64 m;
    int e0;
    split_fp(w, m, e0);
    const int s = e0 - ea;
    if (s >= 0) {
        const u64 lo = shl64(m, (u32)s);
        const u64 hi = s >= 64 ? shl64(m, (u32)(s - 64)) : shr64(m, (u32)(64 - s));
        return mk128(lo, hi);
    }
    const u32 r = (u32)(-s);
    if (r >= 54) return mk128(0);  // m < 2^53 <= 2^(r-1): rounds to 0
    const u64 q = shr64(m, r), rem = m - shl64(q, r), half = shl64(1ull, r - 1);
    return mk128(q + ((rem > half || (rem == half && (q & 1))) ? 1 : 0), 0);
}

// Fast class-specific decodes.  f32: w = m * 2^(E-150), W = m << s with
// s = E - 150 - ea; a light has s <= 29 and a heavy s >= 29 (w > avg >=
// 2^52 u), so each class is a couple of clamped 32-bit (funnel) shifts.
// f64: W = RNE(w * 2^-ea), one multiply and one conversion.  Each decode
// folds its item into a per-group check `chk`; the group is redone by
// units_generic when the check fails (tiny or subnormal lights, weights
// >= 2^64 units, unrepresentable scale): see group_slow().
__device__ __forceinline__ u32 shl32c(u32 x, u32 s)
{
    u32 r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
    return r;
}
__device__ __forceinline__ u32 shf_hi(u32 x, u32 s)  // upper word of ((u64)x << s), s <= 32
{
    u32 r;
    asm("shf.l.clamp.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(0u), "r"(s));
    return r;
}

struct Chk {
    u32 smax;    // f32: max over items of (u32)s (lights need s < 32, heavies s < 64)
    double xmax; // f64: max scaled weight (must be < 2^64)
};
__device__ __forceinline__ void chk_init(Chk &c)
{
    c.smax = 0;
    c.xmax = 0.0;
}

// light units (f32, the pack's light pass): needs s in [0, 32)
__device__ __forceinline__ u64 light_W(float w, const Quant &Q, bool use, Chk &c)
{
    const u32 b = __float_as_uint(w);
    const u32 s = (u32)((int)(b >> 23) - Q.sh32);
    c.smax = max(c.smax, use ? s << 1 : 0u);  // s >= 32 or s < 0 -> >= 64
    const u32 m = (b & 0x7FFFFFu) | 0x800000u;
    return ((u64)shf_hi(m, s) << 32) | shl32c(m, s);
}
// units mod 2^64 of either class (f32), bits >= 64 into hi; the class's
// condition (light: s < 32, heavy: s < 64) is folded into c when `use`
__device__ __forceinline__ u64 any_W(float w, const Quant &Q, bool light, bool use, Chk &c, u32 &hi)
{
    const u32 b = __float_as_uint(w);
    const u32 s = (u32)((int)(b >> 23) - Q.sh32);
    c.smax = max(c.smax, use ? (light ? s << 1 : s) : 0u);
    const u32 m = (b & 0x7FFFFFu) | 0x800000u;
    const bool big = s >= 32u;
    const u32 t = s - 32u;
    const u32 lo = shl32c(m, s);  // 0 when s >= 32
    const u32 hw = big ? shl32c(m, t) : shf_hi(m, s);
    hi = big ? shf_hi(m, t) : 0u;
    return ((u64)hw << 32) | lo;
}
__device__ __forceinline__ u64 light_W(double w, const Quant &Q, bool use, Chk &c)
{
    const double x = w * Q.scale;
    c.xmax = use ? fmax(c.xmax, x) : c.xmax;
    return __double2ull_rn(x);
}
__device__ __forceinline__ u64 any_W(double w, const Quant &Q, bool, bool use, Chk &c, u32 &hi)
{
    const double x = w * Q.scale;
    c.xmax = use ? fmax(c.xmax, x) : c.xmax;
    hi = 0;
    return __double2ull_rn(x);
}
__device__ __forceinline__ bool group_slow(const Chk &c, const Quant &Q, float)
{
    return c.smax >= 64u || Q.sh32 < 1;  // sh32 < 1: subnormal weights may pass the shift test
}
__device__ __forceinline__ bool group_slow(const Chk &c, const Quant &Q, double)
{
    return !(c.xmax < 18446744073709551616.0) || Q.scale == 0.0;
}

// the largest T not above avg: (double)v <= avg  <=>  v <= avg_floor(avg)
template <typename T> __device__ __forceinline__ T avg_floor(double avg);
template <> __device__ __forceinline__ float avg_floor<float>(double avg)
{
    return __double2float_rd(avg);
}
template <> __device__ __forceinline__ double avg_floor<double>(double avg) { return avg; }

// ---------------------------------------------------------------------------
// loads
// ---------------------------------------------------------------------------
// 8 consecutive values from 16-byte aligned global memory (read-only path)
template <typename T> __device__ __forceinline__ void ldg8(const T *p, T v[VV])
{
    if (sizeof(T) == 4) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
        const float4 b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
        const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int q = 0; q < VV; ++q) v[q] = (T)f[q];
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 a = __ldg(reinterpret_cast<const double2 *>(p) + q);
            v[2 * q] = (T)a.x;
            v[2 * q + 1] = (T)a.y;
        }
    }
}
// the same from shared memory
template <typename T> __device__ __forceinline__ void lds8(const T *p, T v[VV])
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
// items [i0, i0 + 8) with i0 % 8 == 0; items outside [lo, hi) are marked by
// the returned mask bit being clear (their values are unspecified)
template <typename T>
__device__ __forceinline__ u32 load_group(const T *__restrict__ w, u64 i0, u64 lo, u64 hi, T v[VV],
                                          T fill)
{
    if (i0 >= lo && i0 + VV <= hi) {
        ldg8(w + i0, v);
        return 0xFFu;
    }
    u32 m = 0;
#pragma unroll
    for (int q = 0; q < VV; ++q) {
        const bool in = i0 + q >= lo && i0 + q < hi;
        v[q] = in ? w[i0 + q] : fill;  // a light value the fast decodes accept
        m |= (u32)in << q;
    }
    return m;
}

// ---------------------------------------------------------------------------
// workspace layout
// ---------------------------------------------------------------------------
struct BuildWs {
    u64 nt, nst;  // tiles, super-tiles
    u32 super;    // tiles per scan CTA
    unsigned int *counter;
    u32 *status;            // [nst] 0 none, 1 aggregate, 2 inclusive
    u128 *agg_D, *agg_H;    // [nst] super-tile aggregates (write once)
    u64 *agg_k;
    u128 *inc_D, *inc_H;    // [nst] inclusive prefixes (write once)
    u64 *inc_k;
    u128 *DLb, *DHb;        // [nt+1] exclusive tile bases (exact)
    u64 *kL;                // [nt+1] lights before tile
    u128 *cE;               // [nt*NW] heavy excess of each chunk
    u64 *hitem;             // [nt+1] first heavy past section boundary u (NONE64: none)
    u64 *KB;                // [nt+1] key base of the window that starts there
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// tiles per scan CTA: 32, or fewer (multiples of 4, one per warp) so that
// small inputs still spread over ~2 CTAs per SM
inline u32 super_for(u64 nt)
{
    const u64 s = nt / 296;
    return (u32)(s >= SUPER ? SUPER : (s < 4 ? 4 : s & ~3ull));
}

constexpr int NBUF = 15;
template <typename F> inline void layout(u64 n, F &&take)
{
    const u64 nt = (n + TILE - 1) / TILE;
    const u64 nst = (nt + super_for(nt) - 1) / super_for(nt);
    const size_t sizes[NBUF] = {256,          nst * 4,       nst * 16,      nst * 16,     nst * 8,
                                nst * 16,     nst * 16,      nst * 8,       (nt + 1) * 16, (nt + 1) * 16,
                                (nt + 1) * 8, nt * NW * 16,  (nt + 1) * 8,  (nt + 1) * 8, 0};
    for (int i = 0; i < NBUF; ++i) take(i, sizes[i]);
}

inline BuildWs carve(void *ws, u64 n)
{
    BuildWs W;
    W.nt = (n + TILE - 1) / TILE;
    W.super = super_for(W.nt);
    W.nst = (W.nt + W.super - 1) / W.super;
    char *base = (char *)ws;
    size_t off = 0;
    char *p[NBUF];
    layout(n, [&](int i, size_t b) {
        p[i] = base + off;
        off += align256(b);
    });
    W.counter = (unsigned int *)p[0];
    W.status = (u32 *)p[1];
    W.agg_D = (u128 *)p[2];
    W.agg_H = (u128 *)p[3];
    W.agg_k = (u64 *)p[4];
    W.inc_D = (u128 *)p[5];
    W.inc_H = (u128 *)p[6];
    W.inc_k = (u64 *)p[7];
    W.DLb = (u128 *)p[8];
    W.DHb = (u128 *)p[9];
    W.kL = (u64 *)p[10];
    W.cE = (u128 *)p[11];
    W.hitem = (u64 *)p[12];
    W.KB = (u64 *)p[13];
    return W;
}

size_t ws_bytes_for(u64 n)
{
    size_t off = 0;
    layout(n, [&](int, size_t b) { off += align256(b); });
    return off + 256;
}

// ---------------------------------------------------------------------------
// 1. scan + super-tile decoupled look-back
// ---------------------------------------------------------------------------
constexpr int SC_WARPS = 4;  // warps per scan CTA; each owns SUPER / SC_WARPS tiles
template <typename T> struct ScanBuf {
    // per warp a ring of NW chunk slots (chunk c of successive tiles in slot
    // c), then the per-lane heavy sums of the warp's current tile
    static constexpr size_t RING = (size_t)SC_WARPS * NW * CH * sizeof(T);
    static constexpr size_t SUMS = (size_t)SC_WARPS * NW * 32 * sizeof(u128);
    static constexpr size_t BYTES = RING + SUMS;
};

// One pass over the weights.  Each warp streams its tiles chunk by chunk
// through a ring of shared-memory slots filled by 1-D bulk async copies (the
// TMA engine; 8 chunks in flight per warp).  Per lane: the units W of its 8
// items, summed by class (lights: u64, heavies: u128).  Per chunk: the heavy
// excess sum(W) - nh*A (u128, exact).  Per tile: the light deficit
// nl*A - sum(W) (u64, exact) and light count.  Warp 0 then scans the
// super-tile's tile totals, publishes the aggregate, runs the decoupled
// look-back and writes the exclusive tile bases.
template <typename T>
__global__ void __launch_bounds__(SC_WARPS * 32) k_build_scan(const T *__restrict__ w, u64 n,
                                                              Quant Q, BuildWs W)
{
    extern __shared__ __align__(128) unsigned char scan_smem[];
    __shared__ __align__(8) u64 bars[SC_WARPS][NW];
    __shared__ u64 s_tD[SUPER];
    __shared__ u128 s_tE[SUPER];
    __shared__ u32 s_tL[SUPER];
    __shared__ unsigned int s_st;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_st = atomicAdd(W.counter, 1u);
    if (lane == 0) {
#pragma unroll
        for (int c = 0; c < NW; ++c) mbar_init(&bars[wid][c], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const u64 st = s_st;
    const u64 t0 = st * W.super;
    const u64 tn = (t0 + W.super <= W.nt) ? W.super : W.nt - t0;
    T *ring = reinterpret_cast<T *>(scan_smem) + (size_t)wid * NW * CH;
    u128 *sums = reinterpret_cast<u128 *>(scan_smem + ScanBuf<T>::RING) + (size_t)wid * NW * 32;
    const T avgT = avg_floor<T>(Q.avg);
    const u64 A = Q.A;
    auto full_chunk = [&](u64 g) { return (g + 1) * CH <= n; };
    auto issue = [&](u64 j, int c) {  // chunk c of the super-tile's tile j into slot c
        const u64 g = (t0 + j) * NW + c;
        if (lane == 0 && j < tn && full_chunk(g)) {
            mbar_expect_tx(&bars[wid][c], CH * sizeof(T));
            bulk_g2s(ring + c * CH, w + g * CH, CH * sizeof(T), &bars[wid][c]);
        }
    };
#pragma unroll
    for (int c = 0; c < NW; ++c) issue((u64)wid, c);
    u32 phase = 0;  // all slots complete once per tile: one parity for all

    for (u64 j = wid; j < tn; j += SC_WARPS) {
        const u64 t = t0 + j;
        u64 sLW = 0;   // lane's light units
        u32 nl = 0;    // lane's lights
        u32 nhc = 0;   // heavies of chunk (lane & 7) (lanes 0..7 after the loop)
#pragma unroll 1
        for (int c = 0; c < NW; ++c) {
            const u64 g = t * NW + c;
            T v[VV];
            u32 vm;
            if (full_chunk(g)) {
                mbar_wait(&bars[wid][c], phase);
                lds8(ring + c * CH + lane * VV, v);
                vm = 0xFFu;
                // the slot's reads are done and ordered before the async-proxy
                // refill of the next tile's chunk c
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                issue(j + SC_WARPS, c);
            } else {
                vm = load_group(w, g * CH + (u64)lane * VV, 0, n, v, avgT);
            }
            u64 Wq[VV];
            u32 Hq[VV];
            u32 lm = 0;
            Chk ck;
            chk_init(ck);
#pragma unroll
            for (int q = 0; q < VV; ++q) {
                const bool li = v[q] <= avgT;
                lm |= (u32)li << q;
                Wq[q] = any_W(v[q], Q, li, true, ck, Hq[q]);
            }
            if (group_slow(ck, Q, T())) {
#pragma unroll
                for (int q = 0; q < VV; ++q) {
                    const u128 g = units_generic(v[q], Q.ea);
                    Wq[q] = g.lo;
                    Hq[q] = (u32)g.hi;
                }
            }
            if (vm != 0xFFu) {
#pragma unroll
                for (int q = 0; q < VV; ++q)
                    if (!((vm >> q) & 1)) Wq[q] = 0, Hq[q] = 0;
                lm &= vm;
            }
            // all valid units (96-bit) and the lights' (u64); heavies = all - lights
            u64 tlo = 0, lsum = 0;
            u32 thi = 0;
#pragma unroll
            for (int q = 0; q < VV; ++q) {
                asm("add.cc.u64 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+l"(tlo), "+r"(thi) : "l"(Wq[q]), "r"(Hq[q]));
                if ((lm >> q) & 1) lsum += Wq[q];
            }
            sLW += lsum;
            u64 hlo;
            u32 hhi;
            asm("sub.cc.u64 %0, %2, %4;\n\tsubc.u32 %1, %3, 0;" : "=l"(hlo), "=r"(hhi) : "l"(tlo), "r"(thi), "l"(lsum));
            const u128 hW = mk128(hlo, hhi);
            lm &= vm;
            nl += __popc(lm);
            const u32 nh = __reduce_add_sync(0xffffffffu, (u32)__popc(vm & ~lm));
            if (lane == c) nhc = nh;
            sums[c * 32 + lane] = hW;
        }
        phase ^= 1;
        __syncwarp();
        // chunk heavy sums: lane l adds lanes 8q..8q+7 of chunk l>>2 (q = l&3)
        const int cc = lane >> 2, qq = lane & 3;
        u128 s = mk128(0);
#pragma unroll
        for (int k = 0; k < 8; ++k) s = add128(s, sums[cc * 32 + qq * 8 + k]);
        s = add128(s, shfl_xor128(s, 1));
        s = add128(s, shfl_xor128(s, 2));
        const u32 nh_c = __shfl_sync(0xffffffffu, nhc, cc);
        const u128 ex = sub128(s, mk128((u64)nh_c * A));  // chunk cc's excess
        if (qq == 0) W.cE[t * NW + cc] = ex;
        // tile excess: sum over the chunk lanes (qq == 0 lanes hold distinct chunks)
        u128 te = qq == 0 ? ex : mk128(0);
        te = add128(te, shfl_xor128(te, 4));
        te = add128(te, shfl_xor128(te, 8));
        te = add128(te, shfl_xor128(te, 16));
        // tile light deficit
        u64 lw = sLW;
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) lw += __shfl_xor_sync(0xffffffffu, lw, d);
        const u32 tl = __reduce_add_sync(0xffffffffu, nl);
        if (lane == 0) {
            s_tD[j] = (u64)tl * A - lw;
            s_tE[j] = te;
            s_tL[j] = tl;
        }
        __syncwarp();  // sums[] reads done before the next tile overwrites them
    }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    // warp 0: inclusive scan of the tile totals (exact)
    u128 xD = mk128((u64)lane < tn ? s_tD[lane] : 0ull);
    u128 xH = (u64)lane < tn ? s_tE[lane] : mk128(0);
    u64 xK = (u64)lane < tn ? s_tL[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u128 yD = shfl_up128(xD, d), yH = shfl_up128(xH, d);
        const u64 yK = __shfl_up_sync(0xffffffffu, xK, d);
        if (lane >= d) {
            xD = add128(xD, yD);
            xH = add128(xH, yH);
            xK += yK;
        }
    }
    const u128 aD = shfl128(xD, 31), aH = shfl128(xH, 31);
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
    u128 eD = mk128(0), eH = mk128(0);
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
        u128 cD = mk128(0), cH = mk128(0);
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
            cD = add128(cD, shfl_xor128(cD, m));
            cH = add128(cH, shfl_xor128(cH, m));
            cK += __shfl_xor_sync(0xffffffffu, cK, m);
        }
        eD = add128(eD, cD);
        eH = add128(eH, cH);
        eK += cK;
        if (stop < 32 || pred - 32 < 0) break;
        pred -= 32;
    }
    if (lane == 0 && st > 0) {
        W.inc_D[st] = add128(eD, aD);
        W.inc_H[st] = add128(eH, aH);
        W.inc_k[st] = eK + aK;
        __threadfence();
        st_release_u32(&W.status[st], 2u);
    }
    // exclusive bases of the super-tile's tiles
    const u128 pD = shfl_up128(xD, 1), pH = shfl_up128(xH, 1);
    const u64 pK = __shfl_up_sync(0xffffffffu, xK, 1);
    if ((u64)lane < tn) {
        const u64 t = t0 + lane;
        W.DLb[t] = lane ? add128(eD, pD) : eD;
        W.DHb[t] = lane ? add128(eH, pH) : eH;
        W.kL[t] = eK + (lane ? pK : 0);
        if (t + 1 == W.nt) {
            W.DLb[W.nt] = add128(eD, xD);
            W.DHb[W.nt] = add128(eH, xH);
            W.kL[W.nt] = eK + xK;
        }
    }
}

// ---------------------------------------------------------------------------
// 2. PSA split: the first heavy past every section boundary
// ---------------------------------------------------------------------------
// Section u holds the lights of tile u and the heavies with keys in
// (DLb[u], DLb[u+1]] — the reference's split (split.py:69-77: the greatest h
// with H[h] <= cap - L[n-h]).  For X = DLb[u] the boundary heavy J is the
// first with DH(J) > X: tile t = max{t : DHb[t] <= X} (binary search, one
// lane per boundary, 32 boundaries per warp), chunk c = the first whose
// inclusive excess passes X (8 lanes), J inside the chunk from its exact keys.
// hitem[u] = J's item; KB[u] = DH(J-1) - X (mod 2^64) so that the window key
// of any heavy from J on is KB[u] + (excess prefix from J).
template <typename T>
__global__ void __launch_bounds__(TB) k_build_split(const T *__restrict__ w, u64 n, Quant Q,
                                                    BuildWs W)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u64 nt = W.nt;
    const u64 b0 = ((u64)blockIdx.x * NW + wid) * 32;
    if (b0 > nt) return;
    const u64 mb = b0 + lane;
    u128 X = mb <= nt ? W.DLb[mb] : mk128(0);
    u64 tt = 0;
    if (mb <= nt) {
        u64 lo = 0, hi = nt;
        while (lo < hi) {
            const u64 mid = (lo + hi + 1) >> 1;
            if (le128(W.DHb[mid], X)) lo = mid;
            else hi = mid - 1;
        }
        tt = lo;
    }
    const T avgT = avg_floor<T>(Q.avg);
    const u128 A = mk128(Q.A);
    const int cnt = (int)(nt - b0 + 1 < 32 ? nt - b0 + 1 : 32);
    for (int i = 0; i < cnt; ++i) {
        const u64 b = b0 + i;
        const u64 t = __shfl_sync(0xffffffffu, tt, i);
        const u128 x = shfl128(X, i);
        if (t >= nt) {
            if (lane == 0) {
                W.hitem[b] = NONE64;
                W.KB[b] = 0;
            }
            continue;
        }
        const u128 rel = sub128(x, W.DHb[t]);
        // chunk: the first whose inclusive excess (within the tile) passes rel
        u128 e = lane < NW ? W.cE[t * NW + lane] : mk128(0);
        u128 inc = e;
#pragma unroll
        for (int d = 1; d < NW; d <<= 1) {
            const u128 y = shfl_up128(inc, d);
            if (lane >= d) inc = add128(inc, y);
        }
        const unsigned pm = __ballot_sync(0xffffffffu, lane < NW && !le128(inc, rel));
        const int c = __ffs(pm) - 1;  // exists: rel < tile excess
        const u128 excl = sub128(shfl128(inc, c), shfl128(e, c));
        const u128 r = sub128(rel, excl);
        // exact keys of the chunk's heavies (chunk frame)
        const u64 g = t * NW + c;
        const u64 i0 = g * CH + (u64)lane * VV;
        T v[VV];
        const u32 vm = load_group(w, i0, 0, n, v, avgT);
        u64 Wq[VV];
        u32 Hq[VV];
        Chk ck;
        chk_init(ck);
#pragma unroll
        for (int q = 0; q < VV; ++q) {
            const bool h = ((vm >> q) & 1) && !(v[q] <= avgT);
            Wq[q] = any_W(v[q], Q, false, h, ck, Hq[q]);
        }
        if (group_slow(ck, Q, T())) {
#pragma unroll
            for (int q = 0; q < VV; ++q) {
                const u128 g2 = units_generic(v[q], Q.ea);
                Wq[q] = g2.lo;
                Hq[q] = (u32)g2.hi;
            }
        }
        u128 ex[VV];
        u128 s = mk128(0);
        u32 hm = 0;
#pragma unroll
        for (int q = 0; q < VV; ++q) {
            const bool h = ((vm >> q) & 1) && !(v[q] <= avgT);
            hm |= (u32)h << q;
            ex[q] = h ? sub128(mk128(Wq[q], Hq[q]), A) : mk128(0);
            s = add128(s, ex[q]);
        }
        u128 li = s;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u128 y = shfl_up128(li, d);
            if (lane >= d) li = add128(li, y);
        }
        u128 k = sub128(li, s);  // lane's exclusive base
        int fq = -1;
        u64 kb = 0;
#pragma unroll
        for (int q = 0; q < VV; ++q) {
            k = add128(k, ex[q]);
            if (fq < 0 && ((hm >> q) & 1) && !le128(k, r)) {
                fq = q;
                kb = k.lo - ex[q].lo - r.lo;  // DH(J-1) - X, mod 2^64
            }
        }
        const unsigned fl = __ballot_sync(0xffffffffu, fq >= 0);
        const int src = __ffs(fl) - 1;  // exists: the chunk's last heavy key = its excess > r
        const int q0 = __shfl_sync(0xffffffffu, fq, src);
        const u64 kb0 = __shfl_sync(0xffffffffu, kb, src);
        if (lane == 0) {
            W.hitem[b] = g * CH + (u64)src * VV + q0;
            W.KB[b] = kb0;
        }
    }
}

// ---------------------------------------------------------------------------
// 3. section pack
// ---------------------------------------------------------------------------
struct ScanCell {
    u64 v;
    u32 c;
    u32 pad;
};
constexpr int LAP = TILE + TILE / 32;  // padded light-alias slots
__device__ __forceinline__ u32 lslot(u32 p) { return p + (p >> 5); }  // conflict-free both ways

struct SecSmem {
    u64 LK[TILE];                  // light keys (exclusive deficit prefixes, tile frame), rank order
    u64 HK[HCAP + 2];              // round's heavy keys (section frame), slot order; KEY_INF sentinel (+1 pad: LA 16-B aligned)
    u32 LA[LAP];                   // light alias + 1 by tile position (lslot); 0: not a light
    unsigned short LP[TILE];       // light rank -> tile position
    unsigned short HI[HCAP];       // round's heavy items, offset from the round start
    unsigned short SR[HCAP];       // round's heavy -> rank of its successor light
    ScanCell sw[NW];               // CTA scan: warp totals
    ScanCell sb[NW + 1];           // CTA scan: warp bases, [NW] = total
    ScanCell xtot;                 // extra groups (warp 0): totals
    u64 xv[XG];                    // extra groups: exclusive sums / counts
    u32 xc[XG];
    u32 lres;                      // first light not resolved by the round
    u64 pend_item;                 // last heavy of the previous round (alias pending), NONE64
    double pend_tw;
};

// exclusive CTA scan of (u64, u32) pairs: warp Kogge-Stone, warp 0 scans the
// warp totals (two barriers)
__device__ __forceinline__ void cta_scan(SecSmem &P, u64 v, u32 c, int lane, int wid, u64 &ev,
                                         u32 &ec, u64 &tv, u32 &tc)
{
    u64 x = v;
    u32 y = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u64 a = __shfl_up_sync(0xffffffffu, x, d);
        const u32 b = __shfl_up_sync(0xffffffffu, y, d);
        if (lane >= d) {
            x += a;
            y += b;
        }
    }
    if (lane == 31) {
        ScanCell z;
        z.v = x;
        z.c = y;
        z.pad = 0;
        P.sw[wid] = z;
    }
    __syncthreads();
    if (wid == 0) {
        const ScanCell z = P.sw[lane & (NW - 1)];
        u64 a = lane < NW ? z.v : 0ull;
        u32 b = lane < NW ? z.c : 0u;
#pragma unroll
        for (int d = 1; d < NW; d <<= 1) {
            const u64 a2 = __shfl_up_sync(0xffffffffu, a, d);
            const u32 b2 = __shfl_up_sync(0xffffffffu, b, d);
            if (lane >= d) {
                a += a2;
                b += b2;
            }
        }
        if (lane < NW) {
            ScanCell e;
            e.v = a - z.v;
            e.c = b - z.c;
            e.pad = 0;
            P.sb[lane] = e;
            if (lane == NW - 1) {
                e.v = a;
                e.c = b;
                P.sb[NW] = e;
            }
        }
    }
    __syncthreads();
    const ScanCell bw = P.sb[wid], bt = P.sb[NW];
    ev = bw.v + x - v;
    ec = bw.c + y - c;
    tv = bt.v;
    tc = bt.c;
}

// heavy group: class mask, inclusive excess prefixes (mod 2^64)
template <typename T>
__device__ __forceinline__ u64 heavy_group(const T *__restrict__ w, u64 i0, u64 a, u64 b, T avgT,
                                           const Quant &Q, u64 loc[VV], u32 &hm)
{
    T v[VV];
    const u32 vm = load_group(w, i0, a, b, v, avgT);
    u64 Wq[VV];
    Chk ck;
    chk_init(ck);
    hm = 0;
#pragma unroll
    for (int q = 0; q < VV; ++q) {
        const bool h = ((vm >> q) & 1) && !(v[q] <= avgT);
        hm |= (u32)h << q;
        u32 hq;
        Wq[q] = any_W(v[q], Q, false, h, ck, hq);
    }
    if (group_slow(ck, Q, T())) {
#pragma unroll
        for (int q = 0; q < VV; ++q) Wq[q] = units_generic(v[q], Q.ea).lo;
    }
    u64 s = 0;
#pragma unroll
    for (int q = 0; q < VV; ++q) {
        s += ((hm >> q) & 1) ? Wq[q] - Q.A : 0ull;
        loc[q] = s;
    }
    return s;
}

template <typename T>
__global__ void __launch_bounds__(TB, 4) k_build_pack(const T *__restrict__ w, u64 n, Quant Q,
                                                      BuildWs W,
                                                      typename RowOf<T>::type *__restrict__ rows)
{
    typedef typename RowOf<T>::type RowT;
    typedef decltype(RowT::alias) AliasT;
    extern __shared__ __align__(16) unsigned char sec_smem[];
    SecSmem &P = *reinterpret_cast<SecSmem *>(sec_smem);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const u64 nt = W.nt;
    const u64 u = blockIdx.x;  // section; u == nt: the heavies past every light
    const T avgT = avg_floor<T>(Q.avg);
    const u64 ha = W.hitem[u];
    const u64 a = ha == NONE64 ? n : ha;                       // window [a, b)
    const u64 after = u < nt ? W.hitem[u + 1] : NONE64;        // first heavy past the section
    const u64 b = after == NONE64 ? n : after;
    const u64 t0 = u * TILE;
    u64 kb = W.KB[u];

    // ---- lights of tile u: exact exclusive deficit prefixes (tile frame)
    u32 nL = 0;
    u64 Lu = 0;  // the tile's light deficit = the next section's first key
    if (u < nt) {
        for (int i = tid; i < LAP / 4; i += TB) reinterpret_cast<uint4 *>(P.LA)[i] = make_uint4(0, 0, 0, 0);
        const u64 i0 = t0 + (u64)tid * VV;
        T v[VV];
        const u32 vm = t0 + TILE <= n ? (ldg8(w + i0, v), 0xFFu) : load_group(w, i0, 0, n, v, avgT);
        u64 Wq[VV];
        Chk ck;
        chk_init(ck);
        u32 lm = 0;
#pragma unroll
        for (int q = 0; q < VV; ++q) {
            const bool li = ((vm >> q) & 1) && v[q] <= avgT;
            lm |= (u32)li << q;
            Wq[q] = light_W(v[q], Q, li, ck);
        }
        if (group_slow(ck, Q, T())) {
#pragma unroll
            for (int q = 0; q < VV; ++q) Wq[q] = units_generic(v[q], Q.ea).lo;
        }
        u64 loc[VV];
        u64 s = 0;
#pragma unroll
        for (int q = 0; q < VV; ++q) {
            loc[q] = s;
            s += ((lm >> q) & 1) ? Q.A - Wq[q] : 0ull;
        }
        u64 ev, tv;
        u32 ec, tc;
        cta_scan(P, s, __popc(lm), lane, wid, ev, ec, tv, tc);
        nL = tc;
        Lu = tv;
#pragma unroll
        for (int q = 0; q < VV; ++q) {
            if ((lm >> q) & 1) {
                const u32 r = ec + __popc(lm & ((1u << q) - 1));
                P.LK[r] = ev + loc[q];
                P.LP[r] = (unsigned short)(tid * VV + q);
            }
        }
    }
    if (tid == 0) P.pend_item = NONE64;

    // ---- heavy window in rounds
    u32 lfirst = 0;  // first light not yet resolved
    u64 pos = a & ~(u64)(VV - 1);
    while (pos < b) {
        const u64 grem = (b - pos + VV - 1) / VV;
        const u32 G = grem <= (u64)(TB + XG) ? (u32)grem : (u32)TB;
        // primary group tid, extra group TB + lane (warp 0)
        u64 loc[VV];
        u32 hm = 0;
        u64 s = 0;
        if ((u32)tid < G) s = heavy_group(w, pos + (u64)tid * VV, a, b, avgT, Q, loc, hm);
        u64 xloc[VV];
        u32 xhm = 0;
        if (wid == 0 && G > (u32)TB) {
            u64 xs = 0;
            if ((u32)(TB + lane) < G) xs = heavy_group(w, pos + (u64)(TB + lane) * VV, a, b, avgT, Q, xloc, xhm);
            u64 x = xs;
            u32 y = __popc(xhm);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const u64 t1 = __shfl_up_sync(0xffffffffu, x, d);
                const u32 t2 = __shfl_up_sync(0xffffffffu, y, d);
                if (lane >= d) {
                    x += t1;
                    y += t2;
                }
            }
            P.xv[lane] = x - xs;
            P.xc[lane] = y - __popc(xhm);
            if (lane == 31) {
                P.xtot.v = x;
                P.xtot.c = y;
            }
        }
        u64 ev, tv;
        u32 ec, tc;
        cta_scan(P, s, __popc(hm), lane, wid, ev, ec, tv, tc);
        const u64 kb0 = kb + ev;
#pragma unroll
        for (int q = 0; q < VV; ++q) {
            if ((hm >> q) & 1) {
                const u32 sl = ec + __popc(hm & ((1u << q) - 1));
                P.HK[sl] = kb0 + loc[q];
                P.HI[sl] = (unsigned short)(tid * VV + q);
            }
        }
        u32 nH = tc;
        u64 tot = tv;
        if (G > (u32)TB) {
            if (wid == 0) {
                const u64 xb = kb + tv + P.xv[lane];
                const u32 xr = tc + P.xc[lane];
#pragma unroll
                for (int q = 0; q < VV; ++q) {
                    if ((xhm >> q) & 1) {
                        const u32 sl = xr + __popc(xhm & ((1u << q) - 1));
                        P.HK[sl] = xb + xloc[q];
                        P.HI[sl] = (unsigned short)((TB + lane) * VV + q);
                    }
                }
            }
            nH += P.xtot.c;
            tot += P.xtot.v;
        }
        kb += tot;
        const bool last_round = pos + (u64)G * VV >= b;
        __syncthreads();  // HK, HI complete
        if (wid == 0) {
            // lights resolved this round: [lfirst, lres), lres = the first light
            // with key >= the round's last heavy key (32-ary search)
            u32 lo = lfirst, hi = nL;  // answer in [lo, hi]
            if (nH > 0) {
                const u64 hl = P.HK[nH - 1];
                while (hi > lo) {
                    const u32 step = (hi - lo + 31) >> 5;
                    const u32 idx = lo + (u32)lane * step;
                    const bool below = idx < hi && P.LK[idx] < hl;
                    const u32 c = __popc(__ballot_sync(0xffffffffu, below));
                    if (c == 0) {
                        hi = lo;
                    } else {
                        const u32 nlo = lo + (c - 1) * step + 1;
                        hi = lo + c * step < hi ? lo + c * step : hi;
                        lo = nlo;
                    }
                }
            }
            if (lane == 0) {
                P.lres = lo;
                P.HK[nH] = KEY_INF;
                if (nH > 0 && P.pend_item != NONE64) {
                    // the previous round's last heavy: its successor is this round's first
                    RowT row;
                    row.tw = tw_store<T>(P.pend_tw, Q.avg);
                    row.alias = (AliasT)(pos + P.HI[0] + 1);
                    rows[P.pend_item] = row;
                    P.pend_item = NONE64;
                }
            }
        }
        __syncthreads();
        const u32 lres = P.lres;
        // merge path: lights [lfirst, lres) with heavies [0, nH); heavy first
        // on ties.  A taken heavy records its successor light's rank; a taken
        // light writes its alias (the heavy's item) at its tile position.
        {
            const u64 *LKp = P.LK + lfirst;
            const unsigned short *LPp = P.LP + lfirst;
            const u32 na = lres - lfirst;
            const u32 total = na + nH;
            const u32 per = (total + TB - 1) / TB;
            const u32 d0 = (u32)tid * per;
            if (d0 < total) {
                u32 lo = d0 > nH ? d0 - nH : 0, hi = d0 < na ? d0 : na;
                while (lo < hi) {
                    const u32 mid = (lo + hi + 1) >> 1;
                    if (LKp[mid - 1] < P.HK[d0 - mid]) lo = mid;
                    else hi = mid - 1;
                }
                u32 i = lo, j = d0 - lo;
                const u32 steps = d0 + per < total ? per : total - d0;
                u64 lk = i < na ? LKp[i] : KEY_INF;
                u64 hk = P.HK[j];
                const u32 ibase = (u32)pos + 1;
                // branch-free walk: both candidates are read, one is written
                for (u32 d = 0; d < steps; ++d) {
                    const bool th = hk <= lk;
                    const u32 hij = P.HI[j < nH ? j : 0];
                    const u32 lpi = LPp[i < na ? i : 0];
                    unsigned short *srp = P.SR + j;
                    u32 *lap = P.LA + lslot(lpi);
                    if (th) *srp = (unsigned short)(lfirst + i);
                    else *lap = ibase + hij;
                    j += th ? 1u : 0u;
                    i += th ? 0u : 1u;
                    hk = P.HK[j];
                    lk = i < na ? LKp[i] : KEY_INF;
                }
            }
        }
        __syncthreads();
        // heavy rows of this round
        for (u32 j = tid; j < nH; j += TB) {
            const u32 sr = P.SR[j];
            const u64 dl = sr < nL ? P.LK[sr] : Lu;
            const double tw = Q.avg + (double)(i64)(P.HK[j] - dl) * Q.u;
            const u64 item = pos + P.HI[j];
            if (j + 1 < nH || last_round) {
                u64 al;
                if (j + 1 < nH) al = pos + P.HI[j + 1] + 1;
                else al = after == NONE64 ? item + 1 : after + 1;
                RowT row;
                row.tw = tw_store<T>(tw, Q.avg);
                row.alias = (AliasT)al;
                rows[item] = row;
            } else {
                P.pend_item = item;
                P.pend_tw = tw;
            }
        }
        lfirst = lres;
        pos += (u64)G * VV;
        __syncthreads();  // HK/HI/SR reads done before the next round
    }
    if (tid == 0 && P.pend_item != NONE64) {  // window ended after a heavy-free round
        RowT row;
        row.tw = tw_store<T>(P.pend_tw, Q.avg);
        row.alias = (AliasT)(after == NONE64 ? P.pend_item + 1 : after + 1);
        rows[P.pend_item] = row;
    }
    // ---- light rows by position (consecutive threads, consecutive rows)
    if (u < nt) {
        __syncthreads();  // LP/LA complete (also when the window had no round)
        // unresolved lights: the first heavy past the section, or themselves
        for (u32 r = lfirst + tid; r < nL; r += TB) {
            const u32 p = P.LP[r];
            P.LA[lslot(p)] = (u32)(after == NONE64 ? t0 + p + 1 : after + 1);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < TILE / TB; ++k) {
            const u32 p = k * TB + tid;
            const u32 al = P.LA[lslot(p)];
            if (al) {
                RowT row;
                row.tw = w[t0 + p];
                row.alias = (AliasT)al;
                rows[t0 + p] = row;
            }
        }
    }
}

template <typename T>
int run_build(const void *wv, u64 n, double avg, void *rows, void *ws, cudaStream_t st)
{
    const T *w = (const T *)wv;
    BuildWs W = carve(ws, n);
    const Quant Q = make_quant(avg);
    AK_CUDA_TRY(cudaMemsetAsync(W.counter, 0, 256, st));
    AK_CUDA_TRY(cudaMemsetAsync(W.status, 0, W.nst * 4, st));
    AK_SMEM_ATTR(k_build_scan<T>, (int)ScanBuf<T>::BYTES);
    k_build_scan<T><<<(unsigned)W.nst, SC_WARPS * 32, ScanBuf<T>::BYTES, st>>>(w, n, Q, W);
    AK_LAUNCH_CHECK("k_build_scan");
    const u64 nb = W.nt + 1;
    k_build_split<T><<<(unsigned)((nb + NW * 32 - 1) / (NW * 32)), TB, 0, st>>>(w, n, Q, W);
    AK_LAUNCH_CHECK("k_build_split");
    const size_t smem = sizeof(SecSmem);
    AK_SMEM_ATTR(k_build_pack<T>, (int)smem);
    k_build_pack<T><<<(unsigned)(W.nt + 1), TB, smem, st>>>(w, n, Q, W,
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
    return ak_build_psa_avg(w, dtype, n, total / (double)n, rows, ws, ws_bytes, stream);
}

int ak_build_psa_avg(const void *w, int dtype, uint64_t n, double avg, void *rows, void *ws,
                     size_t ws_bytes, void *stream)
{
    if (n == 0) return AK_ERR_EMPTY_INPUT;
    if (ws_bytes < ws_bytes_for(n)) return AK_ERR_WORKSPACE;
    if (((uintptr_t)w & 15) != 0 || ((uintptr_t)rows & 15) != 0) return AK_ERR_VALUE;
    if (!(avg > 0.0) || !isfinite(avg)) return AK_ERR_VALUE;
    // u32 aliases (f32 rows) and u32 light-successor items in the pack
    if (n >= 0xFFFFFFFFull) return AK_ERR_VALUE;
    cudaStream_t st = ak_stream(stream);
    if (dtype == AK_F32) return run_build<float>(w, n, avg, rows, ws, st);
    if (dtype == AK_F64) return run_build<double>(w, n, avg, rows, ws, st);
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
