// ops.cu — microbenchmarks that decide the round-2 construction design.
//
//  1. per-SM issue throughput of the ops a fixed-point key costs:
//     F2F.F64.F32, DADD, DMUL, F2I.S64.F64, I2F.F64.S64, 64-bit IADD, REDUX
//  2. row-write patterns for an 8 GB f32 table: fully coalesced 8 B rows vs
//     two complementary half-masked writers (light rows / heavy rows written
//     by different warps), back to back and interleaved.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ops ops.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITER = 4096;

__global__ void k_f2f(const float *in, double *out)
{
    float a = in[threadIdx.x], b = in[threadIdx.x + 1], c = in[threadIdx.x + 2], d = in[threadIdx.x + 3];
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int i = 0; i < ITER; ++i) {
        s0 = (double)a; s1 = (double)b; s2 = (double)c; s3 = (double)d;
        a = __int_as_float(__float_as_int(a) ^ (int)__double2hiint(s0));
        b = __int_as_float(__float_as_int(b) ^ (int)__double2hiint(s1));
        c = __int_as_float(__float_as_int(c) ^ (int)__double2hiint(s2));
        d = __int_as_float(__float_as_int(d) ^ (int)__double2hiint(s3));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}

__global__ void k_dadd(const double *in, double *out)
{
    double a = in[threadIdx.x], b = in[threadIdx.x + 1], c = in[threadIdx.x + 2], d = in[threadIdx.x + 3];
    const double e = in[0];
    for (int i = 0; i < ITER; ++i) {
        a = a + e; b = b + e; c = c + e; d = d + e;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}

__global__ void k_dmul(const double *in, double *out)
{
    double a = in[threadIdx.x], b = in[threadIdx.x + 1], c = in[threadIdx.x + 2], d = in[threadIdx.x + 3];
    const double e = in[0];
    for (int i = 0; i < ITER; ++i) {
        a = a * e; b = b * e; c = c * e; d = d * e;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}

__global__ void k_f2i(const double *in, long long *out)
{
    double a = in[threadIdx.x], b = in[threadIdx.x + 1], c = in[threadIdx.x + 2], d = in[threadIdx.x + 3];
    long long s = 0;
    for (int i = 0; i < ITER; ++i) {
        long long x = __double2ll_rz(a), y = __double2ll_rz(b), z = __double2ll_rz(c), w = __double2ll_rz(d);
        s ^= x ^ y ^ z ^ w;
        a = __longlong_as_double(__double_as_longlong(a) ^ (x & 1));
        b = __longlong_as_double(__double_as_longlong(b) ^ (y & 1));
        c = __longlong_as_double(__double_as_longlong(c) ^ (z & 1));
        d = __longlong_as_double(__double_as_longlong(d) ^ (w & 1));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_i2f(const long long *in, double *out)
{
    long long a = in[threadIdx.x], b = in[threadIdx.x + 1], c = in[threadIdx.x + 2], d = in[threadIdx.x + 3];
    double s = 0;
    for (int i = 0; i < ITER; ++i) {
        double x = (double)a, y = (double)b, z = (double)c, w = (double)d;
        a ^= __double_as_longlong(x) & 1; b ^= __double_as_longlong(y) & 1;
        c ^= __double_as_longlong(z) & 1; d ^= __double_as_longlong(w) & 1;
        s = x + y + z + w;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_iadd64(const unsigned long long *in, unsigned long long *out)
{
    unsigned long long a = in[threadIdx.x], b = in[threadIdx.x + 1], c = in[threadIdx.x + 2], d = in[threadIdx.x + 3];
    const unsigned long long e = in[0];
    for (int i = 0; i < ITER; ++i) {
        a += e; b += e; c += e; d += e;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ b ^ c ^ d;
}

__global__ void k_redux(const unsigned *in, unsigned *out)
{
    unsigned a = in[threadIdx.x], b = in[threadIdx.x + 1], c = in[threadIdx.x + 2], d = in[threadIdx.x + 3];
    for (int i = 0; i < ITER; ++i) {
        a = __reduce_add_sync(0xffffffffu, a) + 1; b = __reduce_add_sync(0xffffffffu, b) + 1;
        c = __reduce_add_sync(0xffffffffu, c) + 1; d = __reduce_add_sync(0xffffffffu, d) + 1;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ b ^ c ^ d;
}

__global__ void k_shfl64(const unsigned long long *in, unsigned long long *out)
{
    unsigned long long a = in[threadIdx.x], b = in[threadIdx.x + 1], c = in[threadIdx.x + 2], d = in[threadIdx.x + 3];
    for (int i = 0; i < ITER; ++i) {
        a += __shfl_up_sync(0xffffffffu, a, 1); b += __shfl_up_sync(0xffffffffu, b, 2);
        c += __shfl_up_sync(0xffffffffu, c, 4); d += __shfl_up_sync(0xffffffffu, d, 8);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ b ^ c ^ d;
}

// ---- row writes -----------------------------------------------------------
__device__ __forceinline__ unsigned hash32(unsigned x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

// every row, consecutive lanes -> consecutive rows
__global__ void k_rows_full(uint2 *rows, unsigned long long n)
{
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x)
        rows[i] = make_uint2((unsigned)i, (unsigned)(i >> 3));
}

// rows of one class only (hash bit == cls): half-masked coalesced stores
__global__ void k_rows_half(uint2 *rows, unsigned long long n, unsigned cls)
{
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x)
        if ((hash32((unsigned)i) & 1u) == cls) rows[i] = make_uint2((unsigned)i, (unsigned)(i >> 3));
}

// both classes in one launch: warp pairs (2w, 2w+1) cover the same 256 B
// span, each writing one class (the two writers of a region run together)
__global__ void k_rows_pair(uint2 *rows, unsigned long long n)
{
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned cls = wid & 1;
    const unsigned long long nwarp_pairs = (unsigned long long)gridDim.x * (blockDim.x / 64);
    for (unsigned long long span = blockIdx.x * (unsigned long long)(blockDim.x / 64) + (wid >> 1);
         span * 32 < n; span += nwarp_pairs) {
        unsigned long long i = span * 32 + lane;
        if (i < n && (hash32((unsigned)i) & 1u) == cls) rows[i] = make_uint2((unsigned)i, (unsigned)(i >> 3));
    }
}

// both classes, with the second writer lagging by `lag` rows (the heavy cursor
// of a section trails/leads the light cursor)
__global__ void k_rows_lag(uint2 *rows, unsigned long long n, unsigned long long lag)
{
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned cls = wid & 1;
    const unsigned long long nwarp_pairs = (unsigned long long)gridDim.x * (blockDim.x / 64);
    for (unsigned long long span = blockIdx.x * (unsigned long long)(blockDim.x / 64) + (wid >> 1);
         span * 32 < n + lag; span += nwarp_pairs) {
        unsigned long long i = span * 32 + lane;
        if (cls) i -= lag;
        if (i < n && (hash32((unsigned)i) & 1u) == cls) rows[i] = make_uint2((unsigned)i, (unsigned)(i >> 3));
    }
}

template <typename K, typename... A>
float time_kernel(K k, dim3 g, dim3 b, A... a)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<g, b>>>(a...);
    cudaEventRecord(e0);
    k<<<g, b>>>(a...);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main()
{
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    void *buf;
    CK(cudaMalloc(&buf, 1 << 24));
    CK(cudaMemset(buf, 0x3f, 1 << 24));
    void *out;
    CK(cudaMalloc(&out, 1 << 26));
    const dim3 g(sms * 8), b(256);
    const double ops = (double)g.x * b.x * ITER * 4;  // 4 independent chains
    auto rep = [&](const char *name, float ms) {
        double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
        printf("%-10s %8.3f ms  %7.1f lane-ops/clk/SM (at %d MHz nominal)\n", name, ms, per_clk_sm, clk / 1000);
    };
    rep("F2F.F64", time_kernel(k_f2f, g, b, (const float *)buf, (double *)out));
    rep("DADD", time_kernel(k_dadd, g, b, (const double *)buf, (double *)out));
    rep("DMUL", time_kernel(k_dmul, g, b, (const double *)buf, (double *)out));
    rep("F2I.S64", time_kernel(k_f2i, g, b, (const double *)buf, (long long *)out));
    rep("I2F.F64", time_kernel(k_i2f, g, b, (const long long *)buf, (double *)out));
    rep("IADD64", time_kernel(k_iadd64, g, b, (const unsigned long long *)buf, (unsigned long long *)out));
    rep("REDUX", time_kernel(k_redux, g, b, (const unsigned *)buf, (unsigned *)out));
    rep("SHFL64+add", time_kernel(k_shfl64, g, b, (const unsigned long long *)buf, (unsigned long long *)out));

    const unsigned long long n = 1000000000ull;  // 8 GB of f32 rows
    uint2 *rows;
    CK(cudaMalloc(&rows, n * 8));
    const dim3 gw(sms * 16), bw(256);
    float t_full = time_kernel(k_rows_full, gw, bw, rows, n);
    float t_h0 = time_kernel(k_rows_half, gw, bw, rows, n, 0u);
    float t_h1 = time_kernel(k_rows_half, gw, bw, rows, n, 1u);
    float t_pair = time_kernel(k_rows_pair, gw, bw, rows, n);
    printf("rows full       %8.3f ms  %7.1f GB/s\n", t_full, n * 8 / (t_full * 1e6));
    printf("rows half x2    %8.3f ms  %7.1f GB/s (two launches, %.3f + %.3f)\n", t_h0 + t_h1,
           n * 8 / ((t_h0 + t_h1) * 1e6), t_h0, t_h1);
    printf("rows pair       %8.3f ms  %7.1f GB/s (complementary warps, same span)\n", t_pair,
           n * 8 / (t_pair * 1e6));
    for (unsigned long long lag : {4096ull, 65536ull, 1048576ull, 8388608ull}) {
        float t = time_kernel(k_rows_lag, gw, bw, rows, n, lag);
        printf("rows lag %8llu %8.3f ms  %7.1f GB/s\n", lag, t, n * 8 / (t * 1e6));
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
