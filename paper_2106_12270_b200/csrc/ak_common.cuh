// ak_common.cuh — shared device primitives for libaliaskit_b200 (sm_100a).
//
// Compiled with --fmad=false: the reference (CPython / numba) never contracts
// a multiply and an add, and the double-double routines below rely on exact
// IEEE rounding of every operation.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/aliaskit_b200.h"

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;

#define AK_WARP 32

// ---------------------------------------------------------------------------
// error plumbing (host)
// ---------------------------------------------------------------------------
void ak_set_cuda_error(cudaError_t e, const char *where);
int ak_check_launch(const char *where);

#define AK_CUDA_TRY(expr)                                        \
    do {                                                         \
        cudaError_t _e = (expr);                                 \
        if (_e != cudaSuccess) {                                 \
            ak_set_cuda_error(_e, #expr);                        \
            return AK_ERR_CUDA;                                  \
        }                                                        \
    } while (0)

#define AK_LAUNCH_CHECK(name)                                    \
    do {                                                         \
        int _s = ak_check_launch(name);                          \
        if (_s != AK_OK) return _s;                              \
    } while (0)

static inline cudaStream_t ak_stream(void *s) { return (cudaStream_t)s; }

int ak_num_sms();
unsigned ak_resident_ctas(const void *kernel, int threads, size_t smem);
void *ak_stream_scratch(cudaStream_t st);  // 256 B per (host thread, device, stream)
void *ak_mailbox(cudaStream_t st);         // 256 B mapped pinned host memory, same keying
// Small device results (up to 3 pieces, <= 256 bytes in all) to host memory
// through the mailbox: one-block kernel, then a synchronisation of st only.
int ak_readback(cudaStream_t st, void *dst0, const void *src0, size_t n0, void *dst1 = nullptr,
                const void *src1 = nullptr, size_t n1 = 0, void *dst2 = nullptr,
                const void *src2 = nullptr, size_t n2 = 0);
// A small device fill by a kernel (no copy engine): bytes of value `byte`.
int ak_fill_small(void *p, int byte, size_t bytes, cudaStream_t st);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the launch paths call this instead of the driver on every call
cudaError_t ak_smem_attr_once(const void *kernel, int bytes);
#define AK_SMEM_ATTR(kern, bytes) AK_CUDA_TRY(ak_smem_attr_once((const void *)(kern), (int)(bytes)))

// ---------------------------------------------------------------------------
// table rows
// ---------------------------------------------------------------------------
struct __align__(8) RowF32 {
    float tw;
    u32 alias;
};
struct __align__(16) RowF64 {
    double tw;
    u64 alias;
};

__device__ __forceinline__ RowF32 ld_row(const RowF32 *p)
{
    uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
    RowF32 r;
    r.tw = __uint_as_float(v.x);
    r.alias = v.y;
    return r;
}
__device__ __forceinline__ RowF64 ld_row(const RowF64 *p)
{
    uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
    RowF64 r;
    r.tw = __hiloint2double((int)v.y, (int)v.x);
    r.alias = ((u64)v.w << 32) | v.z;
    return r;
}

// A threshold stored in a row: f64 rows keep the value; f32 rows take the
// nearest float, stepped down when it would exceed avg (a full bucket must
// not read as more than full after rounding).
__host__ __device__ __forceinline__ float tw_to_f32(double t, double avg)
{
    float f = (float)t;
#ifdef __CUDA_ARCH__
    // the walk below ends at the largest float not above avg: one conversion
    // rounding down (avg > 0), no loop and no divergence
    const float cap = __double2float_rd(avg);
    return (double)f > avg ? cap : f;
#else
    while ((double)f > avg && f > 0.0f) f = nextafterf(f, 0.0f);
    return f;
#endif
}
template <typename T> __host__ __device__ __forceinline__ T tw_store(double t, double avg);
template <> __host__ __device__ __forceinline__ float tw_store<float>(double t, double avg)
{
    return tw_to_f32(t, avg);
}
template <> __host__ __device__ __forceinline__ double tw_store<double>(double t, double)
{
    return t;
}

template <typename T> struct RowOf;
template <> struct RowOf<float> { typedef RowF32 type; };
template <> struct RowOf<double> { typedef RowF64 type; };

// ---------------------------------------------------------------------------
// Philox (rng.py)
// ---------------------------------------------------------------------------
#define AK_PHILOX_MULT 0xD2B74407B1CE6E93ULL  // rng.py:22
#define AK_PHILOX_WEYL 0x9E3779B97F4A7C15ULL  // rng.py:23
#define AK_SALT_STREAM 0x6A09E667F3BCC909ULL  // rng.py:27
#define AK_SALT_NODE 0xBB67AE8584CAA73BULL    // rng.py:28
#define AK_SALT_SECTION 0x3C6EF372FE94F82BULL // rng.py:29

// Philox2x64-10 word 0 (rng.py:53-65 / 109-129); both words optionally.
__host__ __device__ __forceinline__ u64 ak_philox2x64_10(u64 ctr, u64 strm, u64 key,
                                                         u64 *w1 = nullptr)
{
    u64 x0 = ctr, x1 = strm, k = key;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
        u64 hi = __umul64hi(x0, AK_PHILOX_MULT);
#else
        u64 hi = (u64)(((unsigned __int128)x0 * AK_PHILOX_MULT) >> 64);
#endif
        u64 lo = x0 * AK_PHILOX_MULT;
        x0 = hi ^ k ^ x1;
        x1 = lo;
        k += AK_PHILOX_WEYL;
    }
    if (w1) *w1 = x1;
    return x0;
}

// (x >> 11) * 2^-53: uniform_nb (rng.py:138-141)
__host__ __device__ __forceinline__ double ak_u53(u64 x)
{
    return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

__host__ __device__ __forceinline__ double ak_uniform_ref(u64 ctr, u64 strm, u64 key)
{
    return ak_u53(ak_philox2x64_10(ctr, strm, key));
}

__host__ __device__ __forceinline__ u64 ak_derive(u64 seed, u64 stream, u64 t0, u64 t1)
{
    return ak_philox2x64_10(t0, t1 ^ stream, seed ^ AK_SALT_STREAM);
}

// GPU-native Philox4x32-10 (Random123 constants): 128 bits per call.
#define AK_PH4_M0 0xD2511F53u
#define AK_PH4_M1 0xCD9E8D57u
#define AK_PH4_W0 0x9E3779B9u
#define AK_PH4_W1 0xBB67AE85u
__device__ __forceinline__ uint4 ak_philox4x32_10(uint4 c, uint2 k)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        u32 hi0 = __umulhi(AK_PH4_M0, c.x), lo0 = AK_PH4_M0 * c.x;
        u32 hi1 = __umulhi(AK_PH4_M1, c.z), lo1 = AK_PH4_M1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += AK_PH4_W0;
        k.y += AK_PH4_W1;
    }
    return c;
}

// The bucket rule (sample.py:76-84): f64 x = u*span, k = trunc clamped,
// keep row+1 iff (x-k)*avg < tw[row], else alias[row] (1-based).
template <typename RowT>
__device__ __forceinline__ i64 ak_rule(const RowT &row, double u, i64 span, i64 lo, double avg,
                                       i64 k_and_row_out[2] = nullptr)
{
    double x = u * (double)span;
    i64 k = (i64)x;
    if (k >= span) k = span - 1;
    double thr = (double)row.tw;
    (void)k_and_row_out;
    return ((x - (double)k) * avg < thr) ? (lo + k + 1) : (i64)row.alias;
}

__device__ __forceinline__ i64 ak_rule_row_index(double u, i64 span)
{
    double x = u * (double)span;
    i64 k = (i64)x;
    return k >= span ? span - 1 : k;
}

// ---------------------------------------------------------------------------
// double-double arithmetic (exact sums for the prefix keys)
// ---------------------------------------------------------------------------
struct dd {
    double hi, lo;
};

__host__ __device__ __forceinline__ dd dd_make(double h, double l = 0.0)
{
    dd r;
    r.hi = h;
    r.lo = l;
    return r;
}

__host__ __device__ __forceinline__ void two_sum(double a, double b, double &s, double &e)
{
    s = a + b;
    double bb = s - a;
    e = (a - (s - bb)) + (b - bb);
}

__host__ __device__ __forceinline__ void fast_two_sum(double a, double b, double &s, double &e)
{
    s = a + b;
    e = b - (s - a);
}

__host__ __device__ __forceinline__ dd dd_add_d(dd x, double y)
{
    double s, e;
    two_sum(x.hi, y, s, e);
    e += x.lo;
    double h, l;
    fast_two_sum(s, e, h, l);
    return dd_make(h, l);
}

__host__ __device__ __forceinline__ dd dd_add(dd x, dd y)
{
    double s1, s2, t1, t2;
    two_sum(x.hi, y.hi, s1, s2);
    two_sum(x.lo, y.lo, t1, t2);
    s2 += t1;
    fast_two_sum(s1, s2, s1, s2);
    s2 += t2;
    fast_two_sum(s1, s2, s1, s2);
    return dd_make(s1, s2);
}

__host__ __device__ __forceinline__ dd dd_neg(dd x) { return dd_make(-x.hi, -x.lo); }
__host__ __device__ __forceinline__ dd dd_sub(dd x, dd y) { return dd_add(x, dd_neg(y)); }

// x <= y / x < y for normalized double-doubles
__host__ __device__ __forceinline__ bool dd_le(dd x, dd y)
{
    return x.hi < y.hi || (x.hi == y.hi && x.lo <= y.lo);
}
__host__ __device__ __forceinline__ bool dd_lt(dd x, dd y)
{
    return x.hi < y.hi || (x.hi == y.hi && x.lo < y.lo);
}

__host__ __device__ __forceinline__ dd two_diff_dd(double a, double b)
{
    double s = a - b;
    double bb = s - a;
    double e = (a - (s - bb)) - (b + bb);
    return dd_make(s, e);
}

// exact comparison of (a - b) against dd t: returns a - b <= t
__host__ __device__ __forceinline__ bool diff_le(double a, double b, dd t)
{
    return dd_le(two_diff_dd(a, b), t);
}


// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double shfl_up_d(double v, int d)
{
    return __shfl_up_sync(0xffffffffu, v, d);
}
__device__ __forceinline__ double shfl_idx_d(double v, int l)
{
    return __shfl_sync(0xffffffffu, v, l);
}

// memory-order helpers for the decoupled look-back
__device__ __forceinline__ u32 ld_acquire_u32(const u32 *p)
{
    u32 v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(u32 *p, u32 v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// mbarrier + 1-D bulk async copy (TMA engine) helpers
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

template <typename T> __device__ __forceinline__ double to_d(T v) { return (double)v; }
