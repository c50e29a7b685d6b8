// ak_sample.cu — counter-based RNG and the two samplers (sample.py, rng.py).
//
//   ak_fill_uniform        uniform_block (rng.py:153-164), bit-exact
//   ak_sample_naive        _fill_samples over the whole table (sample.py:73-84)
//   ak_sample_from_uniforms  the bucket rule fed explicit uniforms
//   ak_sample_sectioned    sectioned_sample (sample.py:243-267): one CTA per
//                          SM, each a balanced slice of the pass's draw space;
//                          a section's rows staged in shared memory by a bulk
//                          async copy (cp.async.bulk + mbarrier), every draw
//                          served from shared memory; the fast-RNG interior
//                          keeps three Philox calls in flight per thread with
//                          the round keys in the constant bank.
//
// Draws use Philox2x64-10 word 0 (AK_RNG_REFERENCE, bit-exact with the
// reference) or the GPU-native Philox4x32-10 (AK_RNG_PHILOX4X32: one call
// yields the 53-bit uniforms of two consecutive counters; statistically gated
// by the chi-square tests, not bit-compatible with the reference).
#include "ak_common.cuh"


namespace {

// ---------------------------------------------------------------------------
// uniform generation
// ---------------------------------------------------------------------------
__global__ void k_fill_uniform(u64 seed, u64 strm, u64 ctr0, u64 m, double *out)
{
    u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride)
        out[i] = ak_uniform_ref(ctr0 + i, strm, seed);
}

__global__ void k_philox_raw(const u64 *ctr, const u64 *strm, const u64 *key, u64 m, u64 *w0,
                             u64 *w1)
{
    u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    u64 b;
    w0[i] = ak_philox2x64_10(ctr[i], strm[i], key[i], &b);
    w1[i] = b;
}

// Philox4x32-10 for known-answer tests, through each formulation the
// samplers use: the generic round loop (ak_philox4x32_10), round keys formed
// inline (philox4x32_key) and round keys as a precomputed table
// (philox4x32_rk).  out holds 12 words per input: generic, inline, table.
__global__ void k_philox4x32_raw(const u32 *ctr, const u32 *key, u64 m, u32 *out);

// Fast mode: the uniform of counter v (64-bit) is word (v & 1) of
// Philox4x32-10(counter = (v >> 1, stream), key = seed).
__device__ __forceinline__ void ph4_pair(u64 call, u64 strm, u64 seed, double &u0, double &u1)
{
    uint4 c = make_uint4((u32)call, (u32)(call >> 32), (u32)strm, (u32)(strm >> 32));
    uint2 k = make_uint2((u32)seed, (u32)(seed >> 32));
    uint4 r = ak_philox4x32_10(c, k);
    u64 a = ((u64)r.y << 32) | r.x;
    u64 b = ((u64)r.w << 32) | r.z;
    u0 = ak_u53(a);
    u1 = ak_u53(b);
}

__device__ __forceinline__ double ph4_single(u64 v, u64 strm, u64 seed)
{
    double u0, u1;
    ph4_pair(v >> 1, strm, seed, u0, u1);
    return (v & 1) ? u1 : u0;
}

// ---------------------------------------------------------------------------
// naive sampler (sample.py:73-84): one counter per draw, random row gather
// ---------------------------------------------------------------------------
template <typename RowT, int MODE, typename OutT>
__global__ void __launch_bounds__(256) k_sample_naive(const RowT *__restrict__ rows, double avg,
                                                      i64 lo, i64 span, u64 seed, u64 strm,
                                                      u64 ctr0, u64 m, OutT *__restrict__ out)
{
    constexpr int U = 4;  // draws in flight per thread
    const u64 nthr = (u64)gridDim.x * blockDim.x;
    const u64 tid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    for (u64 base = (u64)blockIdx.x * blockDim.x * U; base < m; base += nthr * U) {
        double u[U];
        u64 idx[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            idx[j] = base + (u64)j * blockDim.x + threadIdx.x;
            u64 v = ctr0 + idx[j];
            if (MODE == AK_RNG_REFERENCE) u[j] = ak_uniform_ref(v, strm, seed);
            else u[j] = ph4_single(v, strm, seed);
        }
        RowT r[U];
        i64 k[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            k[j] = ak_rule_row_index(u[j], span);
            if (idx[j] < m) r[j] = ld_row(&rows[lo + k[j]]);
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            if (idx[j] < m) {
                double x = u[j] * (double)span;
                out[idx[j]] = (OutT)(((x - (double)k[j]) * avg < (double)r[j].tw) ? (lo + k[j] + 1)
                                                                                   : (i64)r[j].alias);
            }
        }
        (void)tid;
    }
}

template <typename RowT>
__global__ void k_rule_uniforms(const RowT *__restrict__ rows, double avg, i64 lo, i64 span,
                                const double *__restrict__ u, u64 m, i64 *__restrict__ out)
{
    u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        double uu = u[i];
        i64 k = ak_rule_row_index(uu, span);
        RowT r = rows[lo + k];
        double x = uu * (double)span;
        out[i] = ((x - (double)k) * avg < (double)r.tw) ? (lo + k + 1) : (i64)r.alias;
    }
}

// ---------------------------------------------------------------------------
// sectioned sampler
// ---------------------------------------------------------------------------

// The bucket rule from a raw 64-bit word.  For a power-of-two span 2^b the
// reference's f64 steps x = u*span, k = trunc(x), x - k (span >= 2) are exact bit
// manipulations: k = word >> (64-b), x - k = low 53-b bits of (word >> 11)
// scaled by 2^(b-53) (built as 1.f - 1.0, exact) — bit-identical results
// with four fewer double operations.  Other spans use the f64 rule.
template <typename RowT>
__device__ __forceinline__ i64 rule_word(const RowT &tab, u64 word, i64 span, int b, bool pow2,
                                         i64 lo, double avg)
{
    i64 k;
    double frac;
    if (pow2) {
        k = (i64)(word >> (64 - b));
        const u64 f = (word >> 11) & ((1ull << (53 - b)) - 1);  // 53-b fraction bits
        frac = __longlong_as_double((long long)(0x3FF0000000000000ull | (f << (b - 1)))) - 1.0;
    } else {
        const double x = ak_u53(word) * (double)span;
        k = (i64)x;
        if (k >= span) k = span - 1;
        frac = x - (double)k;
    }
    const auto r = tab[k];
    return (frac * avg < (double)r.tw) ? (lo + k + 1) : (i64)r.alias;
}

// A staged f64 section laid out as separate threshold / alias arrays (12
// bytes per row), so 2^14-row sections of f64 tables fit in shared memory.
struct SoA64View {
    const double *tw;
    const u32 *al;
    __device__ __forceinline__ RowF64 operator[](i64 k) const
    {
        RowF64 r;
        r.tw = tw[k];
        r.alias = al[k];
        return r;
    }
};

// Draw pair (d0, d1) of output slots (o0, o0 + 1) written with 16-byte
// stores where possible.  `par` = 1 when o0 is not 16-byte aligned: then
// lane t stores (d1 of t, d0 of t+1) as one vector and the warp's two end
// elements with 8-byte stores.  v0/v1: whether each draw of the pair is in
// range.  All lanes of the warp must call this (shuffles).
template <typename OutT> struct Pair2;
template <> struct Pair2<i64> {
    typedef longlong2 V;
    static __device__ __forceinline__ V mk(i64 a, i64 b) { return make_longlong2(a, b); }
};
template <> struct Pair2<int32_t> {
    typedef int2 V;
    static __device__ __forceinline__ V mk(i64 a, i64 b) { return make_int2((int)a, (int)b); }
};
template <typename OutT>
__device__ __forceinline__ void store_pair(OutT *o0, i64 d0, i64 d1, bool v0, bool v1, int par,
                                           int lane)
{
    typedef typename Pair2<OutT>::V V;
    if (par == 0) {
        if (v0 && v1) {
            *reinterpret_cast<V *>(o0) = Pair2<OutT>::mk(d0, d1);
        } else {
            if (v0) o0[0] = (OutT)d0;
            if (v1) o0[1] = (OutT)d1;
        }
        return;
    }
    const i64 nx = __shfl_down_sync(0xffffffffu, d0, 1);
    const bool nv = __shfl_down_sync(0xffffffffu, (int)v0, 1) != 0;
    const bool vec = lane < 31 && v1 && nv;
    const bool prev_vec = __shfl_up_sync(0xffffffffu, (int)vec, 1) != 0 && lane > 0;
    if (vec) *reinterpret_cast<V *>(o0 + 1) = Pair2<OutT>::mk(d1, nx);
    else if (v1) o0[1] = (OutT)d1;
    if (v0 && !prev_vec) o0[0] = (OutT)d0;
}

// Philox4x32-10 with the round keys formed from the (warp-uniform) seed
// words inline, so they live in uniform registers rather than per thread.
__device__ __forceinline__ uint4 philox4x32_key(uint4 c, u32 k0, u32 k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const u32 hi0 = __umulhi(AK_PH4_M0, c.x), lo0 = AK_PH4_M0 * c.x;
        const u32 hi1 = __umulhi(AK_PH4_M1, c.z), lo1 = AK_PH4_M1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ (k0 + (u32)r * AK_PH4_W0), lo1, hi0 ^ c.w ^ (k1 + (u32)r * AK_PH4_W1), lo0);
    }
    return c;
}

// Philox4x32-10 round keys (k0 + r W0, k1 + r W1), precomputed on the host
// and passed by value: they sit in the kernel's constant bank and are used
// as direct operands of the round XORs, so they take no registers.
struct Ph4Keys {
    u32 k[20];
};

Ph4Keys ph4_keys(u64 seed)
{
    Ph4Keys rk;
    for (int r = 0; r < 10; ++r) {
        rk.k[2 * r] = (u32)seed + (u32)r * AK_PH4_W0;
        rk.k[2 * r + 1] = (u32)(seed >> 32) + (u32)r * AK_PH4_W1;
    }
    return rk;
}

__device__ __forceinline__ uint4 philox4x32_rk(uint4 c, const Ph4Keys &rk)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const u32 hi0 = __umulhi(AK_PH4_M0, c.x), lo0 = AK_PH4_M0 * c.x;
        const u32 hi1 = __umulhi(AK_PH4_M1, c.z), lo1 = AK_PH4_M1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ rk.k[2 * r], lo1, hi0 ^ c.w ^ rk.k[2 * r + 1], lo0);
    }
    return c;
}

__global__ void k_philox4x32_raw(const u32 *ctr, const u32 *key, u64 m, u32 *out)
{
    const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint4 c = make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]);
    const u32 k0 = key[2 * i], k1 = key[2 * i + 1];
    Ph4Keys rk;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        rk.k[2 * r] = k0 + (u32)r * AK_PH4_W0;
        rk.k[2 * r + 1] = k1 + (u32)r * AK_PH4_W1;
    }
    const uint4 a = ak_philox4x32_10(c, make_uint2(k0, k1));
    const uint4 b = philox4x32_key(c, k0, k1);
    const uint4 d = philox4x32_rk(c, rk);
    const uint4 r3[3] = {a, b, d};
#pragma unroll
    for (int v = 0; v < 3; ++v) {
        out[12 * i + 4 * v] = r3[v].x;
        out[12 * i + 4 * v + 1] = r3[v].y;
        out[12 * i + 4 * v + 2] = r3[v].z;
        out[12 * i + 4 * v + 3] = r3[v].w;
    }
}

// the bucket rule for one 64-bit word on a staged f32 section of span 2^b
__device__ __forceinline__ u32 rule_f32_pow2(const RowF32 *tab, u32 wl, u32 wh, int sk, int b,
                                             u64 fmask, u32 lo1, double avg)
{
    // the 53-b fraction bits (word bits 11 .. 63-b) as the mantissa of a
    // double in [1, 2): ((word & ~0x7ff) << b) >> 12, in 32-bit halves
    const u32 k = wh >> sk;
    const u32 l = wl & ~0x7FFu;
    const u32 vh = __funnelshift_l(l, wh, b), vl = l << b;
    const double frac = __hiloint2double((int)((vh >> 12) + 0x3FF00000u), (int)__funnelshift_r(vl, vh, 12)) - 1.0;
    const uint2 row = *reinterpret_cast<const uint2 *>(tab + k);
    return (frac * avg < (double)__uint_as_float(row.x)) ? lo1 + k : row.y;
}

// Fast-mode interior of a section (f32 rows staged in shared memory, span
// 2^b): pairs q in [qa, qb) with qb - qa a multiple of the CTA size, every
// draw in range.  Pair q is one Philox4x32-10 call (counter low word
// cl0 + q, high word ch), its two 64-bit words are draws 2q and 2q + 1 of
// ob.  Indices fit 32 bits (u32 aliases); outputs are int64.  PAR = 0: ob
// is 16-byte aligned and each pair is one 16-byte store; PAR = 1: two 8-byte
// stores (twice the store requests, but no shuffle or lane branch, which
// cost 14% on the half of the sections whose output is misaligned).  The
// store-request count matters: all-8-byte stores back up the LSU queue and
// lose 30% (profiles/r1_summary.md).
template <int PAR>
__device__ __forceinline__ void store_fast(i64 *p, u32 d0, u32 d1, int lane)
{
    if (PAR == 0) {
        *reinterpret_cast<uint4 *>(p) = make_uint4(d0, 0u, d1, 0u);
    } else {
        *reinterpret_cast<uint2 *>(p) = make_uint2(d0, 0u);
        *reinterpret_cast<uint2 *>(p + 1) = make_uint2(d1, 0u);
    }
}
// int32 outputs (opt-in): one 8-byte store per aligned pair
template <int PAR>
__device__ __forceinline__ void store_fast(int32_t *p, u32 d0, u32 d1, int lane)
{
    if (PAR == 0) {
        *reinterpret_cast<uint2 *>(p) = make_uint2(d0, d1);
    } else {
        reinterpret_cast<u32 *>(p)[0] = d0;
        reinterpret_cast<u32 *>(p)[1] = d1;
    }
}

template <int PAR, typename OutT, int U = 3>
__device__ __forceinline__ void fast_pairs_f32_p(const RowF32 *tab, u32 cl0, u32 ch, u64 strm,
                                                 const Ph4Keys &rk, OutT *ob, u32 qa, u32 qb, int b,
                                                 u32 lo1, double avg, int lane)
{
    const u32 sl = (u32)strm, sh = (u32)(strm >> 32);
    const int sk = 32 - b;
    const u64 fmask = (1ull << (53 - b)) - 1;
    const u32 step = blockDim.x;
    OutT *p = ob + 2 * (u64)(qa + threadIdx.x);
    u32 q = qa + threadIdx.x;
    // U independent calls in flight per thread: the rounds are a serial
    // multiply-xor chain and 32 warps per SM alone leave it latency bound
    // (U = 1 -> 2: +5%, 3: +1% more, 4 slower; tools/time_sectioned.py).
    for (; q + (U - 1) * step < qb; q += U * step, p += 2 * U * (u64)step) {
        uint4 c[U];
#pragma unroll
        for (int z = 0; z < U; ++z) c[z] = philox4x32_rk(make_uint4(cl0 + q + z * step, ch, sl, sh), rk);
#pragma unroll
        for (int z = 0; z < U; ++z)
            store_fast<PAR>(p + 2 * z * (u64)step, rule_f32_pow2(tab, c[z].x, c[z].y, sk, b, fmask, lo1, avg),
                            rule_f32_pow2(tab, c[z].z, c[z].w, sk, b, fmask, lo1, avg), lane);
    }
    for (; q < qb; q += step, p += 2 * (u64)step) {
        const uint4 c0 = philox4x32_rk(make_uint4(cl0 + q, ch, sl, sh), rk);
        store_fast<PAR>(p, rule_f32_pow2(tab, c0.x, c0.y, sk, b, fmask, lo1, avg),
                        rule_f32_pow2(tab, c0.z, c0.w, sk, b, fmask, lo1, avg), lane);
    }
}

template <typename OutT>
__device__ __forceinline__ void fast_pairs_f32(const RowF32 *tab, u32 cl0, u32 ch, u64 strm,
                                               const Ph4Keys &rk, OutT *ob, u32 qa, u32 qb,
                                               int b, u32 lo1, double avg, int par, int lane)
{
    if (par) fast_pairs_f32_p<1, OutT>(tab, cl0, ch, strm, rk, ob, qa, qb, b, lo1, avg, lane);
    else fast_pairs_f32_p<0, OutT>(tab, cl0, ch, strm, rk, ob, qa, qb, b, lo1, avg, lane);
}

// The same interior loop for f64 tables staged in shared memory, either as
// rows (V = const RowF64 *) or as threshold / alias arrays (V = SoA64View);
// indices fit 32 bits (n < 2^32 is checked by the caller).
template <class V>
__device__ __forceinline__ u32 rule_f64_pow2(const V &tab, u32 wl, u32 wh, int sk, int b, u32 lo1,
                                             double avg)
{
    const u32 k = wh >> sk;
    const u32 l = wl & ~0x7FFu;
    const u32 vh = __funnelshift_l(l, wh, b), vl = l << b;
    const double frac = __hiloint2double((int)((vh >> 12) + 0x3FF00000u), (int)__funnelshift_r(vl, vh, 12)) - 1.0;
    const RowF64 row = tab[k];
    return (frac * avg < row.tw) ? lo1 + k : (u32)row.alias;
}

template <class V, int PAR, typename OutT, int U = 3>
__device__ __forceinline__ void fast_pairs_f64_p(const V &tab, u32 cl0, u32 ch, u64 strm,
                                                 const Ph4Keys &rk, OutT *ob, u32 qa, u32 qb, int b,
                                                 u32 lo1, double avg, int lane)
{
    const u32 sl = (u32)strm, sh = (u32)(strm >> 32);
    const int sk = 32 - b;
    const u32 step = blockDim.x;
    OutT *p = ob + 2 * (u64)(qa + threadIdx.x);
    u32 q = qa + threadIdx.x;
    for (; q + (U - 1) * step < qb; q += U * step, p += 2 * U * (u64)step) {
        uint4 c[U];
#pragma unroll
        for (int z = 0; z < U; ++z) c[z] = philox4x32_rk(make_uint4(cl0 + q + z * step, ch, sl, sh), rk);
#pragma unroll
        for (int z = 0; z < U; ++z)
            store_fast<PAR>(p + 2 * z * (u64)step, rule_f64_pow2(tab, c[z].x, c[z].y, sk, b, lo1, avg),
                            rule_f64_pow2(tab, c[z].z, c[z].w, sk, b, lo1, avg), lane);
    }
    for (; q < qb; q += step, p += 2 * (u64)step) {
        const uint4 c0 = philox4x32_rk(make_uint4(cl0 + q, ch, sl, sh), rk);
        store_fast<PAR>(p, rule_f64_pow2(tab, c0.x, c0.y, sk, b, lo1, avg),
                        rule_f64_pow2(tab, c0.z, c0.w, sk, b, lo1, avg), lane);
    }
}

// Sectioned sampling.  The draws of sections [first, first+count) form one
// section-major index space (offsets = exclusive prefix of counts); CTA b
// takes the contiguous slice [D*b/G, D*(b+1)/G) of it, so every CTA does the
// same number of draws whatever the section sizes.  Walking its slice, a CTA
// stages each section's rows in shared memory once (cp.async.bulk +
// mbarrier) and serves every draw from there.  Each thread produces two
// consecutive draws per step (one Philox4x32-10 call in the fast mode) and
// the warp writes them as 16-byte stores where aligned.  SMODE 0 reads rows from
// global memory (sections too large for shared memory).
template <typename RowT, int MODE, int SMODE, typename OutT>
__global__ void __launch_bounds__(1024, 1) k_sample_sectioned(
    const RowT *__restrict__ rows, u64 n, double avg, u64 S, const i64 *__restrict__ counts,
    const i64 *__restrict__ offsets, u64 first, u64 count, u64 seed, u64 stream_id, u64 ctr0,
    OutT *__restrict__ out, i64 out_base, const Ph4Keys rk)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) u64 bar;
    // SMODE 0: rows read from global memory; 1: raw rows staged by a bulk
    // async copy; 2: f64 rows staged as threshold / alias arrays
    constexpr bool STAGE = SMODE != 0;
    RowT *srows = reinterpret_cast<RowT *>(smem_raw);
    double *stw = reinterpret_cast<double *>(smem_raw);
    u32 *sal = reinterpret_cast<u32 *>(stw + S);
    const int lane = threadIdx.x & 31;
    u32 phase = 0;
    if (SMODE == 1 && threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // this CTA's slice of the pass's draw space
    const u64 last = first + count - 1;
    const i64 Dbeg = offsets[first];
    const i64 Dend = offsets[last] + counts[last];
    const u64 D = (u64)(Dend - Dbeg);
    const i64 s0 = Dbeg + (i64)(((unsigned __int128)D * blockIdx.x) / gridDim.x);
    const i64 s1 = Dbeg + (i64)(((unsigned __int128)D * (blockIdx.x + 1)) / gridDim.x);
    if (s0 >= s1) return;
    // the section holding draw s0: greatest j with offsets[j] <= s0
    u64 a = first, b = last;
    while (a < b) {
        const u64 mid = (a + b + 1) >> 1;
        if (offsets[mid] <= s0) a = mid;
        else b = mid - 1;
    }
    for (u64 j = a; j <= last; ++j) {
        const i64 oj = offsets[j];
        if (oj >= s1) break;
        const i64 mj = counts[j];
        if (mj <= 0) continue;
        // draws [ia, ib) of section j belong to this CTA
        const i64 ia = s0 > oj ? s0 - oj : 0;
        const i64 ib = s1 < oj + mj ? s1 - oj : mj;
        if (ia >= ib) continue;
        const u64 lo = j * S;
        const u64 hi = lo + S < n ? lo + S : n;
        const i64 span = (i64)(hi - lo);
        const bool pow2 = span >= 2 && (span & (span - 1)) == 0;
        const int bb = pow2 ? __ffsll(span) - 1 : 0;
        const RowT *src = rows + lo;
        if (SMODE == 1) {
            // the previous section's rows are no longer read (generic proxy)
            // before the async-proxy copy overwrites them
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            const u32 bytes = (u32)(span * sizeof(RowT));
            if ((((uintptr_t)src) & 15) == 0 && (bytes & 15) == 0) {
                if (threadIdx.x == 0) {
                    mbar_expect_tx(&bar, bytes);
                    bulk_g2s(srows, src, bytes, &bar);
                }
                mbar_wait(&bar, phase);
                phase ^= 1;
            } else {
                for (i64 r = threadIdx.x; r < span; r += blockDim.x) srows[r] = src[r];
                __syncthreads();
            }
        } else if (SMODE == 2) {
            __syncthreads();
            for (i64 r = threadIdx.x; r < span; r += blockDim.x) {
                const RowF64 x = ld_row(reinterpret_cast<const RowF64 *>(src) + r);
                stw[r] = x.tw;
                sal[r] = (u32)x.alias;
            }
            __syncthreads();
        }
        const RowT *tabp = SMODE == 1 ? srows : src;
        const u64 strm = ak_derive(seed, stream_id, j, AK_SALT_SECTION);
        OutT *o = out + (oj - out_base);
        // pairs: pair p holds draws (2p - poff, 2p - poff + 1).  The fast RNG
        // pairs draws on its call boundary (counter ctr0 + i even); the
        // reference RNG pairs them on the pair-aligned output boundary.
        const int obit = (int)(((uintptr_t)o / sizeof(OutT)) & 1);
        const i64 poff = MODE == AK_RNG_REFERENCE ? (i64)obit : (i64)(ctr0 & 1);
        const int par = MODE == AK_RNG_REFERENCE ? 0 : (int)((obit + (int)poff) & 1);
        const i64 p0 = (ia + poff) >> 1, p1 = (ib - 1 + poff) >> 1;  // inclusive
        // checked pairs [ps, pe] (every lane of the CTA iterates together)
        auto generic_on = [&](const auto &tab, i64 ps, i64 pe) {
            for (i64 pb = ps; pb <= pe; pb += blockDim.x) {
                const i64 p = pb + threadIdx.x;
                const i64 i0 = 2 * p - poff;
                const bool v0 = p <= pe && i0 >= ia && i0 < ib;
                const bool v1 = p <= pe && i0 + 1 >= ia && i0 + 1 < ib;
                u64 w0, w1;
                if (MODE == AK_RNG_REFERENCE) {
                    w0 = ak_philox2x64_10(ctr0 + (u64)i0, strm, seed, nullptr);
                    w1 = ak_philox2x64_10(ctr0 + (u64)i0 + 1, strm, seed, nullptr);
                } else {
                    const u64 call = (ctr0 + (u64)i0) >> 1;
                    const uint4 c = philox4x32_key(make_uint4((u32)call, (u32)(call >> 32), (u32)strm,
                                                              (u32)(strm >> 32)),
                                                   (u32)seed, (u32)(seed >> 32));
                    w0 = ((u64)c.y << 32) | c.x;
                    w1 = ((u64)c.w << 32) | c.z;
                }
                const i64 d0 = rule_word(tab, w0, span, bb, pow2, (i64)lo, avg);
                const i64 d1 = rule_word(tab, w1, span, bb, pow2, (i64)lo, avg);
                store_pair(o + i0, d0, d1, v0, v1, par, lane);
            }
        };
        auto generic = [&](i64 ps, i64 pe) {
            if constexpr (SMODE == 2) generic_on(SoA64View{stw, sal}, ps, pe);
            else generic_on(tabp, ps, pe);
        };
        // the fast path counts calls linearly from cb: a section whose draw
        // counters wrap past 2^64 (ctr0 + ib overflows) keeps the generic
        // per-draw definition, call = (ctr0 + i) mod 2^64 >> 1
        const bool ctr_wraps = (u64)ib > ~ctr0;
        if (MODE == AK_RNG_PHILOX4X32 && SMODE != 0 && pow2 && !ctr_wraps &&
            (sizeof(RowT) == 8 || n <= 0xFFFFFFFFull)) {
            // interior pairs q = p - p0 in [qa, qa + nfast): both draws in
            // range, the call counter's high word constant, whole CTA steps
            const i64 np = p1 - p0 + 1;
            const i64 qa = (2 * p0 - poff >= ia) ? 0 : 1;
            const i64 qb = np - ((2 * p1 - poff + 1 < ib) ? 0 : 1);
            const u64 cb = (ctr0 + (u64)(2 * p0 - poff)) >> 1;
            i64 nfast = qb > qa ? ((qb - qa) / (i64)blockDim.x) * (i64)blockDim.x : 0;
            if ((u64)(u32)cb + (u64)(qa + nfast) > 0xFFFFFFFFull) nfast = 0;
            if (nfast > 0) {
                if (qa > 0) generic(p0, p0 + qa - 1);
                OutT *ob = o + (2 * p0 - poff);
                const u32 fa = (u32)qa, fb = (u32)(qa + nfast), l1 = (u32)(lo + 1);
                if constexpr (sizeof(RowT) == 8) {
                    fast_pairs_f32(reinterpret_cast<const RowF32 *>(tabp), (u32)cb, (u32)(cb >> 32),
                                   strm, rk, ob, fa, fb, bb, l1, avg, par, lane);
                } else if constexpr (SMODE == 2) {
                    const SoA64View v{stw, sal};
                    if (par) fast_pairs_f64_p<SoA64View, 1, OutT>(v, (u32)cb, (u32)(cb >> 32), strm, rk, ob, fa, fb, bb, l1, avg, lane);
                    else fast_pairs_f64_p<SoA64View, 0, OutT>(v, (u32)cb, (u32)(cb >> 32), strm, rk, ob, fa, fb, bb, l1, avg, lane);
                } else {
                    const RowF64 *v = reinterpret_cast<const RowF64 *>(tabp);
                    if (par) fast_pairs_f64_p<const RowF64 *, 1, OutT>(v, (u32)cb, (u32)(cb >> 32), strm, rk, ob, fa, fb, bb, l1, avg, lane);
                    else fast_pairs_f64_p<const RowF64 *, 0, OutT>(v, (u32)cb, (u32)(cb >> 32), strm, rk, ob, fa, fb, bb, l1, avg, lane);
                }
                if (qa + nfast < np) generic(p0 + qa + nfast, p1);
                continue;
            }
        }
        generic(p0, p1);
    }
}

int grid_for(u64 work, int threads, int per_sm = 8)
{
    u64 g = (work + threads - 1) / threads;
    u64 cap = (u64)ak_num_sms() * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

template <typename RowT, typename OutT>
int launch_naive(const void *rows, double avg, u64 lo, u64 span, u64 seed, u64 strm, u64 ctr0,
                 u64 m, OutT *out, int mode, cudaStream_t st)
{
    int g = grid_for((m + 3) / 4, 256, 16);
    if (mode == AK_RNG_REFERENCE)
        k_sample_naive<RowT, AK_RNG_REFERENCE, OutT><<<g, 256, 0, st>>>(
            (const RowT *)rows, avg, (i64)lo, (i64)span, seed, strm, ctr0, m, out);
    else
        k_sample_naive<RowT, AK_RNG_PHILOX4X32, OutT><<<g, 256, 0, st>>>(
            (const RowT *)rows, avg, (i64)lo, (i64)span, seed, strm, ctr0, m, out);
    AK_LAUNCH_CHECK("k_sample_naive");
    return AK_OK;
}

template <typename RowT, int MODE, int SMODE, typename OutT>
int launch_sectioned_t(const void *rows, u64 n, double avg, u64 S, const i64 *counts,
                       const i64 *offsets, u64 first, u64 count, u64 seed, u64 sid, u64 ctr0,
                       OutT *out, i64 out_base, cudaStream_t st)
{
    size_t smem = SMODE == 1 ? S * sizeof(RowT) : (SMODE == 2 ? S * 12 : 0);
    auto kern = k_sample_sectioned<RowT, MODE, SMODE, OutT>;
    if (SMODE) AK_SMEM_ATTR(kern, (int)smem);
    int per_sm = SMODE ? (smem > 110 * 1024 ? 1 : 2) : 2;
    u64 g = (u64)ak_num_sms() * per_sm;
    kern<<<(unsigned)g, 1024, smem, st>>>((const RowT *)rows, n, avg, S, counts, offsets, first,
                                          count, seed, sid, ctr0, out, out_base, ph4_keys(seed));
    AK_LAUNCH_CHECK("k_sample_sectioned");
    return AK_OK;
}

template <typename RowT, int MODE, typename OutT>
int launch_sectioned_m(const void *rows, u64 n, double avg, u64 S, const i64 *counts,
                       const i64 *offsets, u64 first, u64 count, u64 seed, u64 sid, u64 ctr0,
                       OutT *out, i64 out_base, cudaStream_t st)
{
    if (S * sizeof(RowT) <= 200 * 1024)
        return launch_sectioned_t<RowT, MODE, 1, OutT>(rows, n, avg, S, counts, offsets, first,
                                                       count, seed, sid, ctr0, out, out_base, st);
    if (sizeof(RowT) == 16 && S * 12 <= 200 * 1024 && n < 0xFFFFFFFFull)
        return launch_sectioned_t<RowT, MODE, 2, OutT>(rows, n, avg, S, counts, offsets, first,
                                                       count, seed, sid, ctr0, out, out_base, st);
    return launch_sectioned_t<RowT, MODE, 0, OutT>(rows, n, avg, S, counts, offsets, first, count,
                                                   seed, sid, ctr0, out, out_base, st);
}

template <typename RowT, typename OutT>
int launch_sectioned(const void *rows, u64 n, double avg, u64 S, const i64 *counts,
                     const i64 *offsets, u64 first, u64 count, u64 seed, u64 sid, u64 ctr0,
                     OutT *out, i64 out_base, int mode, cudaStream_t st)
{
    if (mode == AK_RNG_REFERENCE)
        return launch_sectioned_m<RowT, AK_RNG_REFERENCE, OutT>(rows, n, avg, S, counts, offsets,
                                                                first, count, seed, sid, ctr0, out,
                                                                out_base, st);
    return launch_sectioned_m<RowT, AK_RNG_PHILOX4X32, OutT>(rows, n, avg, S, counts, offsets,
                                                             first, count, seed, sid, ctr0, out,
                                                             out_base, st);
}

template <typename OutT>
int naive_rows(const void *rows, int dtype, double avg, u64 lo, u64 span, u64 seed, u64 sid,
               u64 ctr0, u64 m, OutT *out, int mode, cudaStream_t st)
{
    if (dtype == AK_F32) return launch_naive<RowF32, OutT>(rows, avg, lo, span, seed, sid, ctr0, m, out, mode, st);
    if (dtype == AK_F64) return launch_naive<RowF64, OutT>(rows, avg, lo, span, seed, sid, ctr0, m, out, mode, st);
    return AK_ERR_VALUE;
}

template <typename OutT>
int sectioned_rows(const void *rows, int dtype, u64 n, double avg, u64 S, const i64 *counts,
                   const i64 *offsets, u64 first, u64 count, u64 seed, u64 sid, u64 ctr0,
                   OutT *out, i64 out_base, int mode, cudaStream_t st)
{
    if (dtype == AK_F32)
        return launch_sectioned<RowF32, OutT>(rows, n, avg, S, counts, offsets, first, count, seed,
                                              sid, ctr0, out, out_base, mode, st);
    if (dtype == AK_F64)
        return launch_sectioned<RowF64, OutT>(rows, n, avg, S, counts, offsets, first, count, seed,
                                              sid, ctr0, out, out_base, mode, st);
    return AK_ERR_VALUE;
}

}  // namespace

extern "C" {

int ak_fill_uniform(uint64_t seed, uint64_t stream_id, uint64_t ctr0, uint64_t m, double *out,
                    void *stream)
{
    if (m == 0) return AK_OK;
    k_fill_uniform<<<grid_for(m, 256), 256, 0, ak_stream(stream)>>>(seed, stream_id, ctr0, m, out);
    AK_LAUNCH_CHECK("k_fill_uniform");
    return AK_OK;
}

int ak_philox4x32(const uint32_t *ctr, const uint32_t *key, uint64_t m, uint32_t *out,
                  void *stream)
{
    if (m == 0) return AK_OK;
    k_philox4x32_raw<<<(unsigned)((m + 255) / 256), 256, 0, ak_stream(stream)>>>(ctr, key, m, out);
    AK_LAUNCH_CHECK("k_philox4x32_raw");
    return AK_OK;
}

int ak_philox2x64(const uint64_t *ctr, const uint64_t *strm, const uint64_t *key, uint64_t m,
                  uint64_t *out_w0, uint64_t *out_w1, void *stream)
{
    if (m == 0) return AK_OK;
    k_philox_raw<<<(unsigned)((m + 255) / 256), 256, 0, ak_stream(stream)>>>(ctr, strm, key, m,
                                                                            out_w0, out_w1);
    AK_LAUNCH_CHECK("k_philox_raw");
    return AK_OK;
}

int ak_sample_naive_out(const void *rows, int dtype, uint64_t n, double avg, uint64_t lo,
                        uint64_t span, uint64_t seed, uint64_t stream_id, uint64_t ctr0, uint64_t m,
                        void *out, int out_dtype, int rng_mode, void *stream)
{
    if (m == 0) return AK_OK;
    if (span == 0 || lo + span > n) return AK_ERR_VALUE;
    if (rng_mode != AK_RNG_REFERENCE && rng_mode != AK_RNG_PHILOX4X32) return AK_ERR_VALUE;
    if (dtype != AK_F32 && dtype != AK_F64) return AK_ERR_VALUE;
    cudaStream_t st = ak_stream(stream);
    if (out_dtype == AK_I64)
        return naive_rows<i64>(rows, dtype, avg, lo, span, seed, stream_id, ctr0, m, (i64 *)out,
                               rng_mode, st);
    if (out_dtype == AK_I32 && n <= 0x7FFFFFFFull)
        return naive_rows<int32_t>(rows, dtype, avg, lo, span, seed, stream_id, ctr0, m,
                                   (int32_t *)out, rng_mode, st);
    return AK_ERR_VALUE;
}

int ak_sample_naive(const void *rows, int dtype, uint64_t n, double avg, uint64_t lo,
                    uint64_t span, uint64_t seed, uint64_t stream_id, uint64_t ctr0, uint64_t m,
                    int64_t *out, int rng_mode, void *stream)
{
    return ak_sample_naive_out(rows, dtype, n, avg, lo, span, seed, stream_id, ctr0, m, out, AK_I64,
                               rng_mode, stream);
}

int ak_sample_from_uniforms(const void *rows, int dtype, uint64_t n, double avg, uint64_t lo,
                            uint64_t span, const double *u, uint64_t m, int64_t *out,
                            void *stream)
{
    if (m == 0) return AK_OK;
    if (span == 0 || lo + span > n) return AK_ERR_VALUE;
    int g = grid_for(m, 256);
    if (dtype == AK_F32)
        k_rule_uniforms<RowF32><<<g, 256, 0, ak_stream(stream)>>>((const RowF32 *)rows, avg,
                                                                  (i64)lo, (i64)span, u, m, out);
    else if (dtype == AK_F64)
        k_rule_uniforms<RowF64><<<g, 256, 0, ak_stream(stream)>>>((const RowF64 *)rows, avg,
                                                                  (i64)lo, (i64)span, u, m, out);
    else
        return AK_ERR_VALUE;
    AK_LAUNCH_CHECK("k_rule_uniforms");
    return AK_OK;
}

int ak_sample_sectioned_out(const void *rows, int dtype, uint64_t n, double avg, uint64_t S,
                            const int64_t *counts, const int64_t *offsets, uint64_t first,
                            uint64_t count, uint64_t seed, uint64_t stream_id, uint64_t ctr0,
                            void *out, int out_dtype, int64_t out_base, int rng_mode, void *stream)
{
    if (count == 0) return AK_OK;
    if (S < 1) return AK_ERR_INVALID_SECTION_SIZE;
    if (S > n) S = n;
    if (first + count > ak_num_sections(n, S)) return AK_ERR_VALUE;
    if (rng_mode != AK_RNG_REFERENCE && rng_mode != AK_RNG_PHILOX4X32) return AK_ERR_VALUE;
    if (dtype != AK_F32 && dtype != AK_F64) return AK_ERR_VALUE;
    cudaStream_t st = ak_stream(stream);
    if (out_dtype == AK_I64)
        return sectioned_rows<i64>(rows, dtype, n, avg, S, counts, offsets, first, count, seed,
                                   stream_id, ctr0, (i64 *)out, out_base, rng_mode, st);
    if (out_dtype == AK_I32 && n <= 0x7FFFFFFFull)
        return sectioned_rows<int32_t>(rows, dtype, n, avg, S, counts, offsets, first, count, seed,
                                       stream_id, ctr0, (int32_t *)out, out_base, rng_mode, st);
    return AK_ERR_VALUE;
}

int ak_sample_sectioned(const void *rows, int dtype, uint64_t n, double avg, uint64_t S,
                        const int64_t *counts, const int64_t *offsets, uint64_t first,
                        uint64_t count, uint64_t seed, uint64_t stream_id, uint64_t ctr0,
                        int64_t *out, int64_t out_base, int rng_mode, void *stream)
{
    return ak_sample_sectioned_out(rows, dtype, n, avg, S, counts, offsets, first, count, seed,
                                   stream_id, ctr0, out, AK_I64, out_base, rng_mode, stream);
}

}  // extern "C"
