// ak_prepack.cu — PSA+ (greedy block-local prepack, partition.py:134-282, and
// psa_plus_construct, pack.py:280-305) on the device.
//
// The reference pairs lights (w < avg) and heavies (w > avg) inside each block
// of `block_size` items with a sequential Vose sweep (exactly-full items
// w == avg fill their own bucket), stops when one side runs out, and forwards
// the leftovers — remaining lights, remaining heavies and the partially
// consumed heavy with its residual — in item order to an ordinary PSA
// construction with the global average.
//
// Here a CTA owns a block.  The block's sweep is the same key merge as the
// fused builder (ak_build.cu): with block-local prefix keys DL(k) (deficits of
// the lights before k) and DH(j) (excess of heavies up to j), light k goes to
// the first heavy with DH > DL(k) and heavy j closes with residual
// DH(j) + avg - DL(#lights with DL < DH(j)).  The sweep ends either when the
// lights run out (the current heavy is the first with DH > DL(nl)) or at the
// last heavy (when DH(nh-1) <= DL(nl)); the terminal heavy closes on itself
// when its residual is exactly avg, else it is forwarded with that residual.
// Keys are block-local doubles (|key| <= block_size * avg), so decisions agree
// with the reference's f64 chain except at ties inside its rounding noise.
//
//   k_prepack_block   classify, compact, keys, write handled rows, per-block
//                     residual summary
//   k_prepack_emit    residual items (index, weight) in global item order
//   k_residual_remap  the residual table (built by the fused builder with the
//                     global average) scattered into the final table
#include "ak_common.cuh"

namespace {

constexpr int PP_TB = 256;

struct BlockInfo {
    u32 nl, nh;     // lights / heavies of the block
    u32 kend;       // lights [0, kend) handled
    int jt;         // terminal heavy (-1: no pairing); heavies (jt, nh) forwarded
    u32 cur;        // 1: heavy jt forwarded with residual curw
    u32 nres;       // forwarded items
    double curw;
    u64 nwritten;   // rows written by the block
};

template <typename T> __device__ __forceinline__ int item_class(T v, double avg)
{
    const double d = (double)v;
    return d == avg ? 2 : (d < avg ? 0 : 1);  // 0 light, 1 heavy, 2 exactly full
}

// exclusive block scan of two counters (PP_TB threads)
__device__ __forceinline__ void block_scan2(u32 a, u32 b, u32 &ea, u32 &eb, u32 &ta, u32 &tb)
{
    __shared__ u32 sa[PP_TB / 32], sb[PP_TB / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u32 ia = a, ib = b;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u32 x = __shfl_up_sync(0xffffffffu, ia, d), y = __shfl_up_sync(0xffffffffu, ib, d);
        if (lane >= d) { ia += x; ib += y; }
    }
    if (lane == 31) { sa[wid] = ia; sb[wid] = ib; }
    __syncthreads();
    u32 oa = 0, ob = 0;
    ta = tb = 0;
    for (int k = 0; k < PP_TB / 32; ++k) {
        if (k < wid) { oa += sa[k]; ob += sb[k]; }
        ta += sa[k];
        tb += sb[k];
    }
    ea = oa + ia - a;
    eb = ob + ib - b;
    __syncthreads();
}

// exclusive block scan of a double (thread-order association, deterministic)
__device__ __forceinline__ double block_scan_d(double x, double &total)
{
    __shared__ double sd[PP_TB / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc = inc + y;
    }
    if (lane == 31) sd[wid] = inc;
    __syncthreads();
    double off = 0.0;
    total = 0.0;
    for (int k = 0; k < PP_TB / 32; ++k) {
        if (k < wid) off = off + sd[k];
        total = total + sd[k];
    }
    __syncthreads();
    return off + (inc - x);
}

// dynamic shared memory of a block of bs items: item offsets (lights from
// the front, heavies from the back), weights, keys (+1 for DL(nl))
struct PPSmem {
    u32 *item;
    double *wt;
    double *key;
};
__device__ __forceinline__ PPSmem pp_smem(unsigned char *base, u32 bs)
{
    PPSmem S;
    S.wt = reinterpret_cast<double *>(base);
    S.key = S.wt + bs;
    S.item = reinterpret_cast<u32 *>(S.key + bs + 1);
    return S;
}

// lights: slots [0, nl); heavies: slot nl + j
template <typename T>
__global__ void __launch_bounds__(PP_TB) k_prepack_block(const T *__restrict__ w, u64 n, double avg,
                                                         u32 bs, u32 thr,
                                                         typename RowOf<T>::type *__restrict__ rows,
                                                         BlockInfo *__restrict__ info)
{
    typedef typename RowOf<T>::type RowT;
    typedef decltype(RowT::tw) TwT;
    typedef decltype(RowT::alias) AliasT;
    extern __shared__ __align__(16) unsigned char pp_raw[];
    PPSmem S = pp_smem(pp_raw, bs);
    __shared__ u64 s_written;
    const u64 b0 = (u64)blockIdx.x * bs;
    const u32 len = (u32)(b0 + bs <= n ? bs : n - b0);
    const u32 per = (len + PP_TB - 1) / PP_TB;
    const u32 i0 = threadIdx.x * per, i1 = i0 + per < len ? i0 + per : len;
    if (threadIdx.x == 0) s_written = 0;
    // classify; exactly-full items are final at once
    u32 cl = 0, ch = 0, cw = 0;
    for (u32 i = i0; i < i1; ++i) {
        const int c = item_class(w[b0 + i], avg);
        cl += c == 0;
        ch += c == 1;
        if (c == 2) {
            RowT row;
            row.tw = (TwT)w[b0 + i];
            row.alias = (AliasT)(b0 + i + 1);
            rows[b0 + i] = row;
            ++cw;
        }
    }
    u32 el, eh, nl, nh;
    block_scan2(cl, ch, el, eh, nl, nh);
    if (cw) atomicAdd((unsigned long long *)&s_written, (unsigned long long)cw);
    for (u32 i = i0; i < i1; ++i) {
        const T v = w[b0 + i];
        const int c = item_class(v, avg);
        if (c == 0) {
            S.item[el] = i;
            S.wt[el] = (double)v;
            ++el;
        } else if (c == 1) {
            S.item[nl + eh] = i;
            S.wt[nl + eh] = (double)v;
            ++eh;
        }
    }
    __syncthreads();
    const bool pair = nl >= thr && nh >= thr;
    u32 kend = 0, cur = 0;
    int jt = -1;
    double curw = 0.0;
    u64 nwritten = 0;
    if (pair) {
        // keys: DL exclusive over lights, DH inclusive over heavies
        {
            const u32 pl = (nl + PP_TB - 1) / PP_TB, a0 = threadIdx.x * pl;
            const u32 a1 = a0 + pl < nl ? a0 + pl : nl;
            double s = 0.0;
            for (u32 k = a0; k < a1; ++k) s = s + (avg - S.wt[k]);
            double tot;
            double x = block_scan_d(s, tot);
            for (u32 k = a0; k < a1; ++k) {
                S.key[k] = x;
                x = x + (avg - S.wt[k]);
            }
            (void)tot;
            if (a0 < a1 && a1 == nl) S.key[nl] = x;  // DL(nl): the block's whole deficit
        }
        __syncthreads();
        const double DLtot = S.key[nl];
        {
            const u32 ph = (nh + PP_TB - 1) / PP_TB, a0 = threadIdx.x * ph;
            const u32 a1 = a0 + ph < nh ? a0 + ph : nh;
            double s = 0.0;
            for (u32 j = a0; j < a1; ++j) s = s + (S.wt[nl + j] - avg);
            double tot;
            double x = block_scan_d(s, tot);
            for (u32 j = a0; j < a1; ++j) {
                x = x + (S.wt[nl + j] - avg);
                S.key[nl + 1 + j] = x;  // heavy keys after DL(nl)
            }
        }
        __syncthreads();
        const double *DL = S.key;           // [0, nl]
        const double *DH = S.key + nl + 1;  // [0, nh)
        // lights absorbed before the sweep stops: #lights with DL < DH(j)
        auto lights_below = [&](double x) {
            u32 a = 0, b = nl;  // first k with DL(k) >= x
            while (a < b) {
                const u32 m = (a + b) >> 1;
                if (DL[m] < x) a = m + 1;
                else b = m;
            }
            return a;
        };
        auto heavies_upto = [&](double x) {
            u32 a = 0, b = nh;  // first j with DH(j) > x
            while (a < b) {
                const u32 m = (a + b) >> 1;
                if (DH[m] <= x) a = m + 1;
                else b = m;
            }
            return a;
        };
        if (DH[nh - 1] <= DLtot) {
            jt = (int)nh - 1;
            kend = lights_below(DH[nh - 1]);
        } else {
            kend = nl;
            jt = (int)heavies_upto(DLtot);
        }
        const double wt_end = (DH[jt] - DL[kend]) + avg;
        cur = wt_end == avg ? 0u : 1u;
        curw = wt_end;
        if (fabs(wt_end - avg) <= 1e-9 * avg) {
            // The sweep ends at (or within rounding of) an exactly full
            // heavy: whether the reference closes it on itself depends on
            // the rounding of its own running residual, so replay its
            // sequential loop (partition.py:163-201) for this block.
            __shared__ u32 s_k, s_cur;
            __shared__ int s_j;
            __shared__ double s_w;
            if (threadIdx.x == 0) {
                u32 k = 0;
                int j = 0;
                double wc = S.wt[nl];
                while (true) {
                    if (wc > avg) {
                        if (k == nl) break;
                        const u64 it = b0 + S.item[k];
                        RowT row;
                        row.tw = (TwT)w[it];
                        row.alias = (AliasT)(b0 + S.item[nl + j] + 1);
                        rows[it] = row;
                        wc += S.wt[k] - avg;
                        ++k;
                    } else {
                        if ((u32)j + 1 >= nh) break;
                        RowT row;
                        row.tw = tw_store<T>(wc, avg);
                        row.alias = (AliasT)(b0 + S.item[nl + j + 1] + 1);
                        rows[b0 + S.item[nl + j]] = row;
                        wc += S.wt[nl + j + 1] - avg;
                        ++j;
                    }
                }
                const bool full = wc == avg;
                if (full) {
                    const u64 it = b0 + S.item[nl + j];
                    RowT row;
                    row.tw = tw_store<T>(wc, avg);
                    row.alias = (AliasT)(it + 1);
                    rows[it] = row;
                }
                s_k = k;
                s_j = j;
                s_cur = full ? 0u : 1u;
                s_w = wc;
            }
            __syncthreads();
            kend = s_k;
            jt = s_j;
            cur = s_cur;
            curw = s_w;
            nwritten = (u64)kend + (u64)jt + (cur ? 0 : 1);
        } else {
        // lights [0, kend): alias = first heavy with DH > DL(k)
        for (u32 k = threadIdx.x; k < kend; k += PP_TB) {
            const u32 j = heavies_upto(DL[k]);
            const u64 it = b0 + S.item[k];
            RowT row;
            row.tw = (TwT)w[it];
            row.alias = (AliasT)(b0 + S.item[nl + j] + 1);
            rows[it] = row;
        }
        // heavies [0, jt): close at DH(j) + avg - DL(#lights below DH(j))
        for (u32 j = threadIdx.x; j < (u32)jt; j += PP_TB) {
            const u32 k = lights_below(DH[j]);
            RowT row;
            row.tw = tw_store<T>((DH[j] - DL[k]) + avg, avg);
            row.alias = (AliasT)(b0 + S.item[nl + j + 1] + 1);
            rows[b0 + S.item[nl + j]] = row;
        }
        if (threadIdx.x == 0 && !cur) {
            const u64 it = b0 + S.item[nl + jt];
            RowT row;
            row.tw = tw_store<T>(wt_end, avg);
            row.alias = (AliasT)(it + 1);
            rows[it] = row;
        }
        nwritten = (u64)kend + (u64)jt + (cur ? 0 : 1);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        BlockInfo bi;
        bi.nl = nl;
        bi.nh = nh;
        bi.kend = kend;
        bi.jt = jt;
        bi.cur = pair ? cur : 0u;
        bi.curw = curw;
        bi.nres = (nl - kend) + (u32)((int)nh - (jt + 1)) + (pair ? cur : 0u);
        bi.nwritten = s_written + nwritten;
        info[blockIdx.x] = bi;
    }
}

// residual items of each block in item order at res_off[block] + ...
template <typename T>
__global__ void __launch_bounds__(PP_TB) k_prepack_emit(const T *__restrict__ w, u64 n, double avg,
                                                        u32 bs, const BlockInfo *__restrict__ info,
                                                        const i64 *__restrict__ res_off,
                                                        i64 *__restrict__ res_idx,
                                                        double *__restrict__ res_w)
{
    const BlockInfo bi = info[blockIdx.x];
    if (bi.nres == 0) return;
    const u64 b0 = (u64)blockIdx.x * bs;
    const u32 len = (u32)(b0 + bs <= n ? bs : n - b0);
    const u32 per = (len + PP_TB - 1) / PP_TB;
    const u32 i0 = threadIdx.x * per, i1 = i0 + per < len ? i0 + per : len;
    u32 cl = 0, ch = 0;
    for (u32 i = i0; i < i1; ++i) {
        const int c = item_class(w[b0 + i], avg);
        cl += c == 0;
        ch += c == 1;
    }
    u32 el, eh, tl, th;
    block_scan2(cl, ch, el, eh, tl, th);
    // forwarded flag per item, then a second scan for positions
    auto fwd = [&](int c, u32 lr, u32 hr) {
        if (c == 0) return lr >= bi.kend;
        if (c == 1) return (int)hr > bi.jt || ((int)hr == bi.jt && bi.cur);
        return false;
    };
    u32 cf = 0;
    {
        u32 lr = el, hr = eh;
        for (u32 i = i0; i < i1; ++i) {
            const int c = item_class(w[b0 + i], avg);
            cf += fwd(c, lr, hr);
            lr += c == 0;
            hr += c == 1;
        }
    }
    u32 ef, dummy, tf, td;
    block_scan2(cf, 0u, ef, dummy, tf, td);
    i64 pos = res_off[blockIdx.x] + ef;
    u32 lr = el, hr = eh;
    for (u32 i = i0; i < i1; ++i) {
        const T v = w[b0 + i];
        const int c = item_class(v, avg);
        if (fwd(c, lr, hr)) {
            res_idx[pos] = (i64)(b0 + i + 1);
            res_w[pos] = (c == 1 && (int)hr == bi.jt) ? bi.curw : (double)v;
            ++pos;
        }
        lr += c == 0;
        hr += c == 1;
    }
}

__global__ void k_info_to_counts(const BlockInfo *info, u64 nb, i64 *cnt, unsigned long long *nw)
{
    const u64 b = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    cnt[b] = info[b].nres;
    atomicAdd(nw, (unsigned long long)info[b].nwritten);
}

// exclusive scan of block counts (single CTA, sequential chunks)
__global__ void k_excl_scan_i64(const i64 *cnt, u64 nb, i64 *off, i64 *total)
{
    __shared__ i64 carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (u64 base = 0; base < nb; base += blockDim.x) {
        const u64 b = base + threadIdx.x;
        const i64 v = b < nb ? cnt[b] : 0;
        // warp + block inclusive scan
        __shared__ i64 ws[32];
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        i64 inc = v;
        for (int d = 1; d < 32; d <<= 1) {
            const i64 y = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += y;
        }
        if (lane == 31) ws[wid] = inc;
        __syncthreads();
        i64 wo = 0;
        for (int k = 0; k < wid; ++k) wo += ws[k];
        const i64 ex = carry + wo + inc - v;
        if (b < nb) off[b] = ex;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = ex + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

// residual table (f64 rows over residual positions) -> final rows
template <typename RowOut>
__global__ void k_residual_remap(const RowF64 *__restrict__ rt, const i64 *__restrict__ res_idx,
                                 u64 nres, double avg, RowOut *__restrict__ rows)
{
    typedef decltype(RowOut::tw) TwT;
    typedef decltype(RowOut::alias) AliasT;
    const u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nres) return;
    const RowF64 x = rt[r];
    RowOut o;
    o.tw = tw_store<TwT>(x.tw, avg);
    o.alias = (AliasT)res_idx[x.alias - 1];
    rows[res_idx[r] - 1] = o;
}

size_t pp_smem_bytes(u32 bs) { return (size_t)bs * 8 + (size_t)(bs + 1) * 8 + (size_t)bs * 4 + 16; }

inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

extern "C" int ak_build_psa_avg(const void *w, int dtype, uint64_t n, double avg, void *rows,
                                void *ws, size_t ws_bytes, void *stream);

extern "C" {

size_t ak_prepack_workspace_bytes(uint64_t n, uint32_t block_size)
{
    const u64 nb = block_size ? (n + block_size - 1) / block_size : 0;
    return al256(nb * sizeof(BlockInfo)) + 2 * al256((nb + 1) * 8) + 256 + 2 * al256(n * 8);
}

int ak_greedy_prepack(const void *w, int dtype, uint64_t n, double avg, uint32_t block_size,
                      uint32_t threshold, void *rows, int64_t *res_idx, double *res_w,
                      uint64_t *nres_out, uint64_t *nwritten_out, void *ws, size_t ws_bytes,
                      void *stream)
{
    if (n == 0) return AK_ERR_EMPTY_INPUT;
    if (block_size < 2 || threshold < 1) return AK_ERR_VALUE;
    const size_t smem = pp_smem_bytes(block_size);
    if (smem > 220 * 1024) return AK_ERR_VALUE;  // block does not fit in shared memory
    if (ws_bytes < ak_prepack_workspace_bytes(n, block_size)) return AK_ERR_WORKSPACE;
    cudaStream_t st = ak_stream(stream);
    const u64 nb = (n + block_size - 1) / block_size;
    char *p = (char *)ws;
    BlockInfo *info = (BlockInfo *)p;
    p += al256(nb * sizeof(BlockInfo));
    i64 *cnt = (i64 *)p;
    p += al256((nb + 1) * 8);
    i64 *off = (i64 *)p;
    p += al256((nb + 1) * 8);
    unsigned long long *nw = (unsigned long long *)p;
    i64 *tot = (i64 *)(p + 64);
    const size_t rb = dtype == AK_F32 ? 8 : 16;
    AK_CUDA_TRY(cudaMemsetAsync(rows, 0, n * rb, st));
    AK_CUDA_TRY(cudaMemsetAsync(nw, 0, 8, st));
    if (dtype == AK_F32) {
        AK_CUDA_TRY(cudaFuncSetAttribute(k_prepack_block<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_prepack_block<float><<<(unsigned)nb, PP_TB, smem, st>>>((const float *)w, n, avg, block_size,
                                                                 threshold, (RowF32 *)rows, info);
    } else if (dtype == AK_F64) {
        AK_CUDA_TRY(cudaFuncSetAttribute(k_prepack_block<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_prepack_block<double><<<(unsigned)nb, PP_TB, smem, st>>>((const double *)w, n, avg, block_size,
                                                                  threshold, (RowF64 *)rows, info);
    } else {
        return AK_ERR_VALUE;
    }
    AK_LAUNCH_CHECK("k_prepack_block");
    k_info_to_counts<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(info, nb, cnt, nw);
    AK_LAUNCH_CHECK("k_info_to_counts");
    k_excl_scan_i64<<<1, 1024, 0, st>>>(cnt, nb, off, tot);
    AK_LAUNCH_CHECK("k_excl_scan_i64");
    if (dtype == AK_F32)
        k_prepack_emit<float><<<(unsigned)nb, PP_TB, 0, st>>>((const float *)w, n, avg, block_size, info,
                                                             off, res_idx, res_w);
    else
        k_prepack_emit<double><<<(unsigned)nb, PP_TB, 0, st>>>((const double *)w, n, avg, block_size,
                                                              info, off, res_idx, res_w);
    AK_LAUNCH_CHECK("k_prepack_emit");
    i64 nres = 0;
    unsigned long long nwr = 0;
    AK_CUDA_TRY(cudaMemcpyAsync(&nres, tot, 8, cudaMemcpyDeviceToHost, st));
    AK_CUDA_TRY(cudaMemcpyAsync(&nwr, nw, 8, cudaMemcpyDeviceToHost, st));
    AK_CUDA_TRY(cudaStreamSynchronize(st));
    *nres_out = (u64)nres;
    *nwritten_out = (u64)nwr;
    return AK_OK;
}

int ak_residual_scatter(const void *res_rows, const int64_t *res_idx, uint64_t nres, double avg,
                        int dtype, void *rows, void *stream)
{
    if (nres == 0) return AK_OK;
    cudaStream_t st = ak_stream(stream);
    const unsigned g = (unsigned)((nres + 255) / 256);
    if (dtype == AK_F32)
        k_residual_remap<RowF32><<<g, 256, 0, st>>>((const RowF64 *)res_rows, res_idx, nres, avg,
                                                     (RowF32 *)rows);
    else if (dtype == AK_F64)
        k_residual_remap<RowF64><<<g, 256, 0, st>>>((const RowF64 *)res_rows, res_idx, nres, avg,
                                                     (RowF64 *)rows);
    else
        return AK_ERR_VALUE;
    AK_LAUNCH_CHECK("k_residual_remap");
    return AK_OK;
}

}  // extern "C"
