// ak_weights.cu — make_weight_set (model.py:95-108) on the device.
//
// Validation (finite and > 0; the first bad index wins) and the total.  The
// reference takes the total from np.sum, which for a contiguous float64
// vector is numpy's pairwise summation: blocks of <= 128 values summed with 8
// interleaved accumulators, larger ranges split at n/2 rounded down to a
// multiple of 8 (numpy 2.3.5 pairwise_sum; restated in the oracle and pinned
// against np.sum by tests).  The tree depends on n only, so the device
// evaluates exactly the same additions in the same order — the total is
// bit-identical to the reference's — with every subtree of the cut at depth D
// summed by one thread and the top D levels combined by two more launches.
#include "ak_common.cuh"

namespace {

constexpr u64 PW_BLOCK = 128;
constexpr u64 SUBTREE_TARGET = 2048;  // elements per thread at the cut depth

struct Node {
    u64 off, size;
    bool exists;  // false: below an earlier leaf, on a non-leftmost path
    bool leaf;    // size <= 128 (reached at or above this depth)
};

__host__ __device__ __forceinline__ u64 split_point(u64 size)
{
    u64 n2 = size / 2;
    return n2 - n2 % 8;
}

// node at depth d, index idx (bits MSB first: 0 = left, 1 = right)
__host__ __device__ inline Node node_at(u64 n, int d, u64 idx)
{
    Node nd{0, n, true, n <= PW_BLOCK};
    for (int lvl = 0; lvl < d; ++lvl) {
        int bit = (int)((idx >> (d - 1 - lvl)) & 1);
        if (nd.size <= PW_BLOCK) {
            // leaf already: only the all-left path carries it down
            if (bit) {
                nd.exists = false;
                return nd;
            }
            continue;
        }
        u64 n2 = split_point(nd.size);
        if (bit == 0) nd.size = n2;
        else {
            nd.off += n2;
            nd.size -= n2;
        }
    }
    nd.leaf = nd.size <= PW_BLOCK;
    return nd;
}

template <typename T>
__device__ __forceinline__ double ld_val(const T *p, u64 i)
{
    return (double)__ldg(p + i);
}

// numpy pairwise_sum leaf (n <= 128)
template <typename T>
__device__ double leaf_sum(const T *a, u64 off, u64 n)
{
    if (n < 8) {
        double res = 0.0;
        for (u64 i = 0; i < n; ++i) res += ld_val(a, off + i);
        return res;
    }
    double r0 = ld_val(a, off + 0), r1 = ld_val(a, off + 1), r2 = ld_val(a, off + 2),
           r3 = ld_val(a, off + 3), r4 = ld_val(a, off + 4), r5 = ld_val(a, off + 5),
           r6 = ld_val(a, off + 6), r7 = ld_val(a, off + 7);
    u64 i;
    for (i = 8; i < n - (n % 8); i += 8) {
        r0 += ld_val(a, off + i + 0);
        r1 += ld_val(a, off + i + 1);
        r2 += ld_val(a, off + i + 2);
        r3 += ld_val(a, off + i + 3);
        r4 += ld_val(a, off + i + 4);
        r5 += ld_val(a, off + i + 5);
        r6 += ld_val(a, off + i + 6);
        r7 += ld_val(a, off + i + 7);
    }
    double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    for (; i < n; ++i) res += ld_val(a, off + i);
    return res;
}

// full pairwise recursion over [off, off+n) with an explicit stack
template <typename T>
__device__ double subtree_sum(const T *a, u64 off, u64 n)
{
    // post-order evaluation: stack of (off, size, state); values stack
    struct Fr {
        u64 off, size;
        int state;
    };
    Fr st[48];
    double vals[48];
    int sp = 0, vp = 0;
    st[sp++] = {off, n, 0};
    while (sp) {
        Fr &f = st[sp - 1];
        if (f.size <= PW_BLOCK) {
            vals[vp++] = leaf_sum(a, f.off, f.size);
            --sp;
            continue;
        }
        u64 n2 = split_point(f.size);
        if (f.state == 0) {
            f.state = 1;
            st[sp++] = {f.off, n2, 0};
        } else if (f.state == 1) {
            f.state = 2;
            st[sp++] = {f.off + n2, f.size - n2, 0};
        } else {
            double r = vals[--vp];
            double l = vals[--vp];
            vals[vp++] = l + r;
            --sp;
        }
    }
    return vals[0];
}

template <typename T>
__global__ void k_pairwise_leaves(const T *__restrict__ w, u64 n, int D, double *__restrict__ part,
                                  unsigned long long *__restrict__ first_bad)
{
    u64 idx = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (1ull << D)) return;
    Node nd = node_at(n, D, idx);
    if (!nd.exists) return;
    // validation of this node's range: finite and > 0 (model.py:101-104)
    for (u64 i = nd.off; i < nd.off + nd.size; ++i) {
        double v = ld_val(w, i);
        if (!(isfinite(v) && v > 0.0)) {
            atomicMin(first_bad, (unsigned long long)i);
            break;
        }
    }
    part[idx] = nd.leaf ? leaf_sum(w, nd.off, nd.size) : subtree_sum(w, nd.off, nd.size);
}

// Combine levels [d_lo, d_hi) in place: part holds values at depth d_hi in
// slots [0, 2^d_hi); each block folds 2^(d_hi-d_lo) children into one value
// at depth d_lo stored in out[block index].
__global__ void k_pairwise_combine(u64 n, int d_hi, int d_lo, const double *__restrict__ part,
                                   double *__restrict__ out)
{
    extern __shared__ double sv[];
    const int span_lv = d_hi - d_lo;  // levels folded by this block
    const u64 width = 1ull << span_lv;
    const u64 base = (u64)blockIdx.x * width;
    for (u64 t = threadIdx.x; t < width; t += blockDim.x) {
        Node nd = node_at(n, d_hi, base + t);
        sv[t] = nd.exists ? part[base + t] : 0.0;
    }
    __syncthreads();
    for (int lv = d_hi - 1; lv >= d_lo; --lv) {
        u64 cnt = 1ull << (lv - d_lo);
        u64 stride = 1ull << (d_hi - lv);  // slot spacing of this level's nodes
        for (u64 t = threadIdx.x; t < cnt; t += blockDim.x) {
            u64 gidx = ((u64)blockIdx.x << (lv - d_lo)) + t;  // index at depth lv
            Node nd = node_at(n, lv, gidx);
            u64 s = t * stride;
            if (nd.exists && !nd.leaf) sv[s] = sv[s] + sv[s + stride / 2];
            // leaf: value already sits in the leftmost slot
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = sv[0];
}

int cut_depth(u64 n)
{
    int D = 0;
    while ((n >> D) > SUBTREE_TARGET && D < 30) ++D;
    return D;
}

}  // namespace

extern "C" {

size_t ak_weights_workspace_bytes(uint64_t n)
{
    int D = cut_depth(n);
    size_t parts = (size_t)1 << D;
    return 256 + parts * sizeof(double) * 2 + 4096;
}

int ak_weights_validate_total(const void *w, int dtype, uint64_t n, double *total,
                              int64_t *bad_index, void *ws, size_t ws_bytes, void *stream)
{
    *bad_index = -1;
    if (n == 0) return AK_ERR_EMPTY_INPUT;
    if (dtype != AK_F32 && dtype != AK_F64) return AK_ERR_VALUE;
    if (ws_bytes < ak_weights_workspace_bytes(n)) return AK_ERR_WORKSPACE;
    cudaStream_t st = ak_stream(stream);
    const int D = cut_depth(n);
    unsigned char *base = (unsigned char *)ws;
    unsigned long long *bad = (unsigned long long *)base;
    double *part = (double *)(base + 256);
    double *part2 = part + ((size_t)1 << D);
    AK_CUDA_TRY(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
    const u64 nthreads = 1ull << D;
    const int tb = 128;
    const unsigned g = (unsigned)((nthreads + tb - 1) / tb);
    if (dtype == AK_F32)
        k_pairwise_leaves<float><<<g, tb, 0, st>>>((const float *)w, n, D, part, bad);
    else
        k_pairwise_leaves<double><<<g, tb, 0, st>>>((const double *)w, n, D, part, bad);
    AK_LAUNCH_CHECK("k_pairwise_leaves");
    // fold the top D levels, at most 10 levels (1024 slots) per block
    int d = D;
    double *src = part, *dst = part2;
    while (d > 0) {
        int lo = d > 10 ? d - 10 : 0;
        u64 blocks = 1ull << lo;
        size_t smem = ((size_t)1 << (d - lo)) * sizeof(double);
        k_pairwise_combine<<<(unsigned)blocks, 256, smem, st>>>(n, d, lo, src, dst);
        AK_LAUNCH_CHECK("k_pairwise_combine");
        double *t = src;
        src = dst;
        dst = t;
        d = lo;
    }
    double tot = 0.0;
    unsigned long long b = 0;
    AK_CUDA_TRY(cudaMemcpyAsync(&tot, src, sizeof(double), cudaMemcpyDeviceToHost, st));
    AK_CUDA_TRY(cudaMemcpyAsync(&b, bad, sizeof(b), cudaMemcpyDeviceToHost, st));
    AK_CUDA_TRY(cudaStreamSynchronize(st));
    if (b != ~0ull) {
        *bad_index = (int64_t)b;
        return AK_ERR_INVALID_WEIGHT;
    }
    *total = tot;
    return AK_OK;
}

}  // extern "C"
