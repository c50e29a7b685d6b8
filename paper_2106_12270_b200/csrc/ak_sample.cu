// ak_sample.cu — counter-based RNG and the two samplers (sample.py, rng.py).
//
//   ak_fill_uniform        uniform_block (rng.py:153-164), bit-exact
//   ak_sample_naive        _fill_samples over the whole table (sample.py:73-84)
//   ak_sample_from_uniforms  the bucket rule fed explicit uniforms
//   ak_sample_sectioned    sectioned_sample (sample.py:243-267): one CTA per
//                          section (persistent, grid = SMs), the section's rows
//                          staged in shared memory by a bulk async copy
//                          (cp.async.bulk + mbarrier), every draw served from
//                          shared memory.
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
template <typename RowT, int MODE>
__global__ void __launch_bounds__(256) k_sample_naive(const RowT *__restrict__ rows, double avg,
                                                      i64 lo, i64 span, u64 seed, u64 strm,
                                                      u64 ctr0, u64 m, i64 *__restrict__ out)
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
                out[idx[j]] = ((x - (double)k[j]) * avg < (double)r[j].tw) ? (lo + k[j] + 1)
                                                                              : (i64)r[j].alias;
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
__device__ __forceinline__ void mbar_init(u64 *bar, u32 count)
{
    u32 a = (u32)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64 *bar, u32 bytes)
{
    u32 a = (u32)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *bar, u32 phase)
{
    u32 a = (u32)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, u32 bytes, u64 *bar)
{
    u32 d = (u32)__cvta_generic_to_shared(dst);
    u32 b = (u32)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(d),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
}

// Philox2x64-10 with a precomputed key schedule (the per-round keys depend
// on the seed only, so they are hoisted out of the draw loop).
struct KeySched64 {
    u64 k[10];
};
__device__ __forceinline__ KeySched64 sched64(u64 key)
{
    KeySched64 s;
#pragma unroll
    for (int r = 0; r < 10; ++r) s.k[r] = key + (u64)r * AK_PHILOX_WEYL;
    return s;
}
__device__ __forceinline__ u64 philox64_sched(u64 x0, u64 x1, const KeySched64 &s)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        u64 hi = __umul64hi(x0, AK_PHILOX_MULT);
        u64 lo = x0 * AK_PHILOX_MULT;
        x0 = hi ^ s.k[r] ^ x1;
        x1 = lo;
    }
    return x0;
}
struct KeySched32 {
    uint2 k[10];
};
__device__ __forceinline__ KeySched32 sched32(u64 seed)
{
    KeySched32 s;
    uint2 k = make_uint2((u32)seed, (u32)(seed >> 32));
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        s.k[r] = k;
        k.x += AK_PH4_W0;
        k.y += AK_PH4_W1;
    }
    return s;
}
__device__ __forceinline__ void philox32_sched(u64 call, u64 strm, const KeySched32 &s, u64 &a, u64 &b)
{
    uint4 c = make_uint4((u32)call, (u32)(call >> 32), (u32)strm, (u32)(strm >> 32));
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        u32 hi0 = __umulhi(AK_PH4_M0, c.x), lo0 = AK_PH4_M0 * c.x;
        u32 hi1 = __umulhi(AK_PH4_M1, c.z), lo1 = AK_PH4_M1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ s.k[r].x, lo1, hi0 ^ c.w ^ s.k[r].y, lo0);
    }
    a = ((u64)c.y << 32) | c.x;
    b = ((u64)c.w << 32) | c.z;
}

// The bucket rule from a raw 64-bit word.  For a power-of-two span 2^b the
// reference's f64 steps x = u*span, k = trunc(x), x - k (span >= 2) are exact bit
// manipulations: k = word >> (64-b), x - k = low 53-b bits of (word >> 11)
// scaled by 2^(b-53) (built as 1.f - 1.0, exact) — bit-identical results
// with four fewer double operations.  Other spans use the f64 rule.
template <typename RowT>
__device__ __forceinline__ i64 rule_word(const RowT *tab, u64 word, i64 span, int b, bool pow2,
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
    const RowT r = tab[k];
    return (frac * avg < (double)r.tw) ? (lo + k + 1) : (i64)r.alias;
}

// One CTA per section (grid-strided over [first, first+count)); the rows of
// the section are copied into shared memory once, then every draw of the
// section reads its row from there.  STAGE=false reads rows from global
// memory (sections too large for shared memory).
template <typename RowT, int MODE, bool STAGE>
__global__ void __launch_bounds__(1024) k_sample_sectioned(
    const RowT *__restrict__ rows, u64 n, double avg, u64 S, const i64 *__restrict__ counts,
    const i64 *__restrict__ offsets, u64 first, u64 count, u64 seed, u64 stream_id, u64 ctr0,
    i64 *__restrict__ out, i64 out_base)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) u64 bar;
    RowT *srows = reinterpret_cast<RowT *>(smem_raw);
    u32 phase = 0;
    if (STAGE && threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const KeySched64 ks64 = sched64(seed);
    const KeySched32 ks32 = sched32(seed);
    for (u64 sj = blockIdx.x; sj < count; sj += gridDim.x) {
        const u64 j = first + sj;
        const i64 mj = counts[j];
        if (mj <= 0) continue;
        const u64 lo = j * S;
        const u64 hi = lo + S < n ? lo + S : n;
        const i64 span = (i64)(hi - lo);
        const bool pow2 = span >= 2 && (span & (span - 1)) == 0;
        const int b = pow2 ? __ffsll(span) - 1 : 0;
        const RowT *src = rows + lo;
        if (STAGE) {
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
        }
        const RowT *tab = STAGE ? srows : src;
        const u64 strm = ak_derive(seed, stream_id, j, AK_SALT_SECTION);
        i64 *o = out + (offsets[j] - out_base);
        const u64 um = (u64)mj;
        if (MODE == AK_RNG_REFERENCE) {
            constexpr int U = 2;
            for (u64 bb = 0; bb < um; bb += (u64)blockDim.x * U) {
                u64 wd[U];
#pragma unroll
                for (int t = 0; t < U; ++t)
                    wd[t] = philox64_sched(ctr0 + bb + (u64)t * blockDim.x + threadIdx.x, strm, ks64);
#pragma unroll
                for (int t = 0; t < U; ++t) {
                    const u64 i = bb + (u64)t * blockDim.x + threadIdx.x;
                    if (i < um) o[i] = rule_word(tab, wd[t], span, b, pow2, (i64)lo, avg);
                }
            }
        } else {
            // counters ctr0+i, paired on even 64-bit counter values: thread t
            // owns pair p -> draws i = 2p - (ctr0 & 1) and i + 1.
            const u64 off = ctr0 & 1;
            const u64 npairs = (um + off + 1) / 2;
            for (u64 p = threadIdx.x; p < npairs; p += blockDim.x) {
                u64 w0, w1;
                philox32_sched((ctr0 >> 1) + p, strm, ks32, w0, w1);
                const i64 i0 = (i64)(2 * p) - (i64)off;
                if (i0 >= 0 && (u64)i0 < um) o[i0] = rule_word(tab, w0, span, b, pow2, (i64)lo, avg);
                if ((u64)(i0 + 1) < um) o[i0 + 1] = rule_word(tab, w1, span, b, pow2, (i64)lo, avg);
            }
        }
        if (STAGE) __syncthreads();  // rows buffer reused by the next section
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

template <typename RowT>
int launch_naive(const void *rows, double avg, u64 lo, u64 span, u64 seed, u64 strm, u64 ctr0,
                 u64 m, i64 *out, int mode, cudaStream_t st)
{
    int g = grid_for((m + 3) / 4, 256, 16);
    if (mode == AK_RNG_REFERENCE)
        k_sample_naive<RowT, AK_RNG_REFERENCE><<<g, 256, 0, st>>>(
            (const RowT *)rows, avg, (i64)lo, (i64)span, seed, strm, ctr0, m, out);
    else
        k_sample_naive<RowT, AK_RNG_PHILOX4X32><<<g, 256, 0, st>>>(
            (const RowT *)rows, avg, (i64)lo, (i64)span, seed, strm, ctr0, m, out);
    AK_LAUNCH_CHECK("k_sample_naive");
    return AK_OK;
}

template <typename RowT, int MODE, bool STAGE>
int launch_sectioned_t(const void *rows, u64 n, double avg, u64 S, const i64 *counts,
                       const i64 *offsets, u64 first, u64 count, u64 seed, u64 sid, u64 ctr0,
                       i64 *out, i64 out_base, cudaStream_t st)
{
    size_t smem = STAGE ? S * sizeof(RowT) : 0;
    auto kern = k_sample_sectioned<RowT, MODE, STAGE>;
    if (STAGE) AK_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = STAGE ? (smem > 110 * 1024 ? 1 : 2) : 2;
    u64 g = (u64)ak_num_sms() * per_sm;
    if (g > count) g = count;
    kern<<<(unsigned)g, 1024, smem, st>>>((const RowT *)rows, n, avg, S, counts, offsets, first,
                                          count, seed, sid, ctr0, out, out_base);
    AK_LAUNCH_CHECK("k_sample_sectioned");
    return AK_OK;
}

template <typename RowT>
int launch_sectioned(const void *rows, u64 n, double avg, u64 S, const i64 *counts,
                     const i64 *offsets, u64 first, u64 count, u64 seed, u64 sid, u64 ctr0,
                     i64 *out, i64 out_base, int mode, cudaStream_t st)
{
    const bool stage = S * sizeof(RowT) <= 200 * 1024;
    if (mode == AK_RNG_REFERENCE) {
        if (stage)
            return launch_sectioned_t<RowT, AK_RNG_REFERENCE, true>(rows, n, avg, S, counts, offsets,
                                                                    first, count, seed, sid, ctr0,
                                                                    out, out_base, st);
        return launch_sectioned_t<RowT, AK_RNG_REFERENCE, false>(rows, n, avg, S, counts, offsets,
                                                                 first, count, seed, sid, ctr0,
                                                                 out, out_base, st);
    }
    if (stage)
        return launch_sectioned_t<RowT, AK_RNG_PHILOX4X32, true>(rows, n, avg, S, counts, offsets,
                                                                 first, count, seed, sid, ctr0,
                                                                 out, out_base, st);
    return launch_sectioned_t<RowT, AK_RNG_PHILOX4X32, false>(rows, n, avg, S, counts, offsets,
                                                              first, count, seed, sid, ctr0, out,
                                                              out_base, st);
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

int ak_philox2x64(const uint64_t *ctr, const uint64_t *strm, const uint64_t *key, uint64_t m,
                  uint64_t *out_w0, uint64_t *out_w1, void *stream)
{
    if (m == 0) return AK_OK;
    k_philox_raw<<<(unsigned)((m + 255) / 256), 256, 0, ak_stream(stream)>>>(ctr, strm, key, m,
                                                                            out_w0, out_w1);
    AK_LAUNCH_CHECK("k_philox_raw");
    return AK_OK;
}

int ak_sample_naive(const void *rows, int dtype, uint64_t n, double avg, uint64_t lo,
                    uint64_t span, uint64_t seed, uint64_t stream_id, uint64_t ctr0, uint64_t m,
                    int64_t *out, int rng_mode, void *stream)
{
    if (m == 0) return AK_OK;
    if (span == 0 || lo + span > n) return AK_ERR_VALUE;
    if (rng_mode != AK_RNG_REFERENCE && rng_mode != AK_RNG_PHILOX4X32) return AK_ERR_VALUE;
    if (dtype == AK_F32)
        return launch_naive<RowF32>(rows, avg, lo, span, seed, stream_id, ctr0, m, out, rng_mode,
                                    ak_stream(stream));
    if (dtype == AK_F64)
        return launch_naive<RowF64>(rows, avg, lo, span, seed, stream_id, ctr0, m, out, rng_mode,
                                    ak_stream(stream));
    return AK_ERR_VALUE;
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

int ak_sample_sectioned(const void *rows, int dtype, uint64_t n, double avg, uint64_t S,
                        const int64_t *counts, const int64_t *offsets, uint64_t first,
                        uint64_t count, uint64_t seed, uint64_t stream_id, uint64_t ctr0,
                        int64_t *out, int64_t out_base, int rng_mode, void *stream)
{
    if (count == 0) return AK_OK;
    if (S < 1) return AK_ERR_INVALID_SECTION_SIZE;
    if (S > n) S = n;
    if (first + count > ak_num_sections(n, S)) return AK_ERR_VALUE;
    if (rng_mode != AK_RNG_REFERENCE && rng_mode != AK_RNG_PHILOX4X32) return AK_ERR_VALUE;
    if (dtype == AK_F32)
        return launch_sectioned<RowF32>(rows, n, avg, S, counts, offsets, first, count, seed,
                                        stream_id, ctr0, out, out_base, rng_mode,
                                        ak_stream(stream));
    if (dtype == AK_F64)
        return launch_sectioned<RowF64>(rows, n, avg, S, counts, offsets, first, count, seed,
                                        stream_id, ctr0, out, out_base, rng_mode,
                                        ak_stream(stream));
    return AK_ERR_VALUE;
}

}  // extern "C"
