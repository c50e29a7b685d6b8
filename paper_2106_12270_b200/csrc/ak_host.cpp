// ak_host.cpp — host-side parts of libaliaskit_b200: error plumbing, library
// identity, and the communication-free section assignment of sectioned
// sampling (sample.py:152-240).
//
// The assignment stays on the host on purpose: the reference draws each
// node's binomial with CPython floats, i.e. glibc log/sqrt/pow and
// round-half-even (sample.py:163-174, stats.py:56-74).  CUDA's libdevice log
// is not bit-identical to glibc's, so bit-exact counts need the host libm.
// This file is compiled with -ffp-contract=off (CPython never fuses mul+add).
// 61,036 nodes at N=1e9, S=2^14 take well under a millisecond here.
#include <utility>
#include <map>
#include <mutex>
#include <tuple>
#include <cuda_runtime.h>

#include <cfenv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/aliaskit_b200.h"

typedef uint64_t u64;
typedef int64_t i64;

static thread_local char g_last_error[512] = "";

void ak_set_cuda_error(cudaError_t e, const char *where)
{
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s (%s)", where, cudaGetErrorName(e),
             cudaGetErrorString(e));
}

int ak_check_launch(const char *where)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        ak_set_cuda_error(e, where);
        return AK_ERR_CUDA;
    }
    return AK_OK;
}

// 256 bytes of device scratch for the small status words an entry point
// writes and reads back within ONE call (flags, counts).  Keyed by (host
// thread, device, stream): two host threads that share a stream (e.g. both
// on the legacy default stream) never share a buffer, and every call that
// uses it ends with a stream synchronisation, so calls of one thread cannot
// overlap.  Allocated once per key (no allocation on the call path) and
// released when the thread exits.
namespace {
struct ThreadScratch {
    std::map<std::pair<int, cudaStream_t>, void *> bufs;
    ~ThreadScratch()
    {
        for (auto &kv : bufs) cudaFree(kv.second);
    }
};
}  // namespace

void *ak_stream_scratch(cudaStream_t st)
{
    static thread_local ThreadScratch ts;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    auto key = std::make_pair(dev, st);
    auto it = ts.bufs.find(key);
    if (it != ts.bufs.end()) return it->second;
    void *p = nullptr;
    if (cudaMalloc(&p, 256) != cudaSuccess) return nullptr;
    ts.bufs[key] = p;
    return p;
}

// 256 bytes of mapped pinned host memory per (host thread, device, stream):
// the mailbox a one-block kernel stores an entry point's small results into
// (ak_readback).  Kernel stores over PCIe need no copy engine, so a result
// readback does not queue behind bulk host<->device copies other streams
// have in flight on the copy engines (a cudaMemcpyAsync of 8 bytes does).
namespace {
struct ThreadMailbox {
    std::map<std::pair<int, cudaStream_t>, void *> bufs;
    ~ThreadMailbox()
    {
        for (auto &kv : bufs) cudaFreeHost(kv.second);
    }
};
}  // namespace

void *ak_mailbox(cudaStream_t st)
{
    static thread_local ThreadMailbox tm;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    auto key = std::make_pair(dev, st);
    auto it = tm.bufs.find(key);
    if (it != tm.bufs.end()) return it->second;
    void *p = nullptr;
    if (cudaHostAlloc(&p, 256, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) return nullptr;
    tm.bufs[key] = p;
    return p;
}

cudaError_t ak_smem_attr_once(const void *kernel, int bytes)
{
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, int> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    int &have = done[std::make_pair(kernel, dev)];
    if (have >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

int ak_num_sms();

// CTAs of `kernel` resident at once on the whole device (SMs x CTAs per SM)
// for a block size and dynamic shared memory, queried once per (kernel,
// device, threads, smem): the L2-prefetch distance of the construction
// kernels, kept off the per-call path (0 if the query fails)
unsigned ak_resident_ctas(const void *kernel, int threads, size_t smem)
{
    static std::mutex mu;
    static std::map<std::tuple<const void *, int, int, size_t>, unsigned> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    const auto key = std::make_tuple(kernel, dev, threads, smem);
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    int per_sm = 0;
    unsigned v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) == cudaSuccess)
        v = (unsigned)(per_sm * ak_num_sms());
    else
        (void)cudaGetLastError();
    std::lock_guard<std::mutex> g(mu);
    cache[key] = v;
    return v;
}

int ak_num_sms()
{
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

extern "C" {

const char *ak_version(void) { return "aliaskit_b200 0.1.0 (sm_100a)"; }

const char *ak_last_error(void) { return g_last_error; }

size_t ak_row_bytes(int dtype) { return dtype == AK_F32 ? 8 : 16; }

// ---- rng.py -------------------------------------------------------------

static u64 philox_w0(u64 ctr, u64 strm, u64 key)
{
    // _philox_py (rng.py:53-65)
    u64 x0 = ctr, x1 = strm, k = key;
    for (int r = 0; r < 10; ++r) {
        unsigned __int128 p = (unsigned __int128)x0 * 0xD2B74407B1CE6E93ULL;
        x0 = (u64)(p >> 64) ^ k ^ x1;
        x1 = (u64)p;
        k += 0x9E3779B97F4A7C15ULL;
    }
    return x0;
}

uint64_t ak_derive_stream(uint64_t seed, uint64_t stream_id, uint64_t tag0, uint64_t tag1)
{
    // derive_stream (rng.py:167-169)
    return philox_w0(tag0, tag1 ^ stream_id, seed ^ 0x6A09E667F3BCC909ULL);
}

// ---- sample.py: section assignment ---------------------------------------

// stats._probit (stats.py:37-74), Acklam's approximation, evaluated in the
// same operation order as the Python source.
static double probit(double p)
{
    static const double a[6] = {-3.969683028665376e+01, 2.209460984245205e+02,
                                -2.759285104469687e+02, 1.383577518672690e+02,
                                -3.066479806614716e+01, 2.506628277459239e+00};
    static const double b[5] = {-5.447609879822406e+01, 1.615858368580409e+02,
                                -1.556989798598866e+02, 6.680131188771972e+01,
                                -1.328068155288572e+01};
    static const double c[6] = {-7.784894002430293e-03, -3.223964580411365e-01,
                                -2.400758277161838e+00, -2.549732539343734e+00,
                                4.374664141464968e+00,  2.938163982698783e+00};
    static const double d[4] = {7.784695709041462e-03, 3.224671290700398e-01,
                                2.445134137142996e+00, 3.754408661907416e+00};
    const double plow = 0.02425;
    if (p < plow) {
        double q = std::sqrt(-2.0 * std::log(p));
        return (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
               ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
    }
    if (p > 1.0 - plow) {
        double q = std::sqrt(-2.0 * std::log(1.0 - p));
        return -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
               ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
    }
    double q = p - 0.5;
    double r = q * q;
    return (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
           (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
}

// _binom_draw (sample.py:152-174): exact CDF inversion below m = 100, else
// the rounded (half-to-even, like Python's round) clamped normal approximation.
static i64 binom_draw(i64 m, double q, double u)
{
    if (m <= 0 || q <= 0.0) return 0;
    if (q >= 1.0) return m;
    if (m < 100) {
        double ratio = q / (1.0 - q);
        double pmf = std::pow(1.0 - q, (double)m);
        double cdf = pmf;
        i64 k = 0;
        while (u > cdf && k < m) {
            k++;
            pmf *= ratio * (double)(m - k + 1) / (double)k;
            cdf += pmf;
        }
        return k;
    }
    double z = probit(u > 1e-300 ? u : 1e-300);
    double mq = (double)m * q;
    double x = std::nearbyint(mq + z * std::sqrt(mq * (1.0 - q)));
    i64 xi = (i64)x;
    return xi < 0 ? 0 : (xi > m ? m : xi);
}

uint64_t ak_num_sections(uint64_t n_rows, uint64_t S)
{
    if (n_rows == 0 || S == 0) return 0;
    if (S > n_rows) S = n_rows;
    return (n_rows + S - 1) / S;
}

int ak_assign_subtree(uint64_t n_rows, uint64_t S, uint64_t seed, uint64_t stream_id, uint64_t a,
                      uint64_t b, uint64_t m, int64_t *counts_out)
{
    if (S < 1) return AK_ERR_INVALID_SECTION_SIZE;
    if (n_rows < 1) return AK_ERR_VALUE;
    if (S > n_rows) S = n_rows;
    u64 ns = (n_rows + S - 1) / S;
    if (!(a < b && b <= ns)) return AK_ERR_VALUE;
    int old_round = std::fegetround();
    std::fesetround(FE_TONEAREST);
    std::memset(counts_out, 0, (size_t)(b - a) * sizeof(int64_t));
    // _assign_range (sample.py:182-200): DFS over midpoint halving; each node
    // is keyed by its row range, so the visiting order is immaterial.
    struct Node {
        u64 na, nb;
        i64 m;
    };
    std::vector<Node> stack;
    stack.reserve(128);
    stack.push_back({a, b, (i64)m});
    while (!stack.empty()) {
        Node nd = stack.back();
        stack.pop_back();
        if (nd.m == 0) continue;
        if (nd.nb - nd.na == 1) {
            counts_out[nd.na - a] += nd.m;
            continue;
        }
        u64 mid = (nd.na + nd.nb) / 2;
        u64 lo_row = nd.na * S;
        u64 hi_row = nd.nb * S < n_rows ? nd.nb * S : n_rows;
        u64 mid_row = mid * S;
        double q = (double)(mid_row - lo_row) / (double)(hi_row - lo_row);
        u64 sub = ak_derive_stream(seed, stream_id, lo_row, hi_row ^ 0xBB67AE8584CAA73BULL);
        double u = (double)(philox_w0(0, sub, seed) >> 11) * (1.0 / 9007199254740992.0);
        i64 ml = binom_draw(nd.m, q, u);
        stack.push_back({mid, nd.nb, nd.m - ml});
        stack.push_back({nd.na, mid, ml});
    }
    std::fesetround(old_round);
    return AK_OK;
}

}  // extern "C"
