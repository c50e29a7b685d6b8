// ak_util.cu — small-result plumbing shared by the entry points.
//
// Every entry point that returns scalars to the host (totals, counts, flags)
// used to read them with cudaMemcpyAsync + cudaStreamSynchronize.  A
// device-to-host copy runs on a copy engine in submission order, so those 8
// bytes waited behind any bulk transfer in flight on another stream (the
// e2e pipeline's 16 GB sample copy-out: make_weight_set blocked for the
// whole transfer, tools/e2e_timeline.py).  Here one thread block stores the
// bytes into mapped pinned host memory (ak_mailbox) instead, and only the
// calling stream is synchronised.
#include <cstring>

#include "ak_common.cuh"

namespace {

struct Piece {
    const unsigned char *src;
    u32 off, n;
};

__global__ void k_publish(unsigned char *box, Piece a, Piece b, Piece c)
{
    const Piece ps[3] = {a, b, c};
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (u32 i = threadIdx.x; i < ps[k].n; i += blockDim.x)
            reinterpret_cast<volatile unsigned char *>(box)[ps[k].off + i] = ps[k].src[i];
    __threadfence_system();
}

__global__ void k_fill_small(unsigned char *p, unsigned char v, u64 bytes)
{
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < bytes; i += (u64)gridDim.x * blockDim.x)
        p[i] = v;
}

}  // namespace

int ak_readback(cudaStream_t st, void *dst0, const void *src0, size_t n0, void *dst1,
                const void *src1, size_t n1, void *dst2, const void *src2, size_t n2)
{
    if (n0 + n1 + n2 > 256) return AK_ERR_VALUE;
    unsigned char *box = (unsigned char *)ak_mailbox(st);
    if (!box) return AK_ERR_CUDA;
    Piece a{(const unsigned char *)src0, 0, (u32)n0};
    Piece b{(const unsigned char *)src1, (u32)n0, (u32)n1};
    Piece c{(const unsigned char *)src2, (u32)(n0 + n1), (u32)n2};
    k_publish<<<1, 32, 0, st>>>(box, a, b, c);
    AK_LAUNCH_CHECK("k_publish");
    AK_CUDA_TRY(cudaStreamSynchronize(st));
    if (n0) memcpy(dst0, box, n0);
    if (n1) memcpy(dst1, box + n0, n1);
    if (n2) memcpy(dst2, box + n0 + n1, n2);
    return AK_OK;
}

int ak_fill_small(void *p, int byte, size_t bytes, cudaStream_t st)
{
    if (!bytes) return AK_OK;
    u64 blocks = (bytes + 255) / 256;
    if (blocks > 1024) blocks = 1024;
    k_fill_small<<<(unsigned)blocks, 256, 0, st>>>((unsigned char *)p, (unsigned char)byte, bytes);
    AK_LAUNCH_CHECK("k_fill_small");
    return AK_OK;
}
