// ak_verify.cu — device verification and layout conversion.
//
//   ak_validate_table    validate_table (model.py:111-144): row invariants and
//                        per-item reconstructed mass.  Each donated row adds
//                        avg - tw to its alias with a compensated f64 atomic:
//                        the rounding error of every atomicAdd is recovered
//                        exactly from the returned old value (TwoSum) and
//                        accumulated separately, so heavy items receiving
//                        millions of contributions are still reconstructed to
//                        ~1 ulp.
//   ak_validate_table_range  the same for an item range (sharded validation)
//   ak_frequency_counts  frequency_counts (stats.py:25-32)
//   ak_chi2_partial      chi_square_test's sums over a bin range (stats.py:84-121)
//   ak_rows_to_soa / ak_soa_to_rows / ak_rows_to_alt1 / ak_count_unwritten
#include "ak_common.cuh"

namespace {

// Validation of the items [ilo, ihi) (the whole table: [0, n)).  Every row
// is read (its donation may land in the range); the row invariants are
// checked for the rows of the range only, so a sharded validation checks
// every row exactly once.  hi/lo are indexed relative to ilo.
template <typename RowT>
__global__ void k_donate(const RowT *__restrict__ rows, u64 n, u64 ilo, u64 ihi, double avg,
                         double row_tol, double *hi, double *lo, int *bad_rows)
{
    u64 stride = (u64)gridDim.x * blockDim.x;
    int bad = 0;
    for (u64 j = (u64)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        RowT r = rows[j];
        double tw = (double)r.tw;
        u64 a = (u64)r.alias;
        if (j >= ilo && j < ihi &&
            (!isfinite(tw) || !(tw >= 0.0) || !(tw <= avg * (1.0 + row_tol)) || a < 1 || a > n))
            bad = 1;
        if (a > ilo && a <= ihi && a != j + 1) {
            double c = avg - tw;
            double old = atomicAdd(&hi[a - 1 - ilo], c);
            double s, e;
            two_sum(old, c, s, e);
            if (e != 0.0) atomicAdd(&lo[a - 1 - ilo], e);
        }
    }
    if (bad) atomicOr(bad_rows, 1);
}

template <typename RowT, typename W>
__device__ __forceinline__ double item_rel_error(const RowT *rows, const W *w, u64 i,
                                                 const double *hi, const double *lo, u64 ilo)
{
    const double wi = (double)w[i];
    // received = tw + (hi + lo), evaluated in double-double
    dd rec = dd_add_d(dd_add_d(dd_make(hi[i - ilo]), lo[i - ilo]), (double)rows[i].tw);
    dd diff = dd_add_d(rec, -wi);
    double rel = fabs(diff.hi + diff.lo) / wi;
    return rel <= 1e300 ? rel : 1e300;  // NaN / inf -> huge
}

template <typename RowT, typename W>
__global__ void k_mass(const RowT *__restrict__ rows, const W *__restrict__ w, u64 ilo, u64 ihi,
                       const double *__restrict__ hi, const double *__restrict__ lo,
                       unsigned long long *worst_bits)
{
    u64 stride = (u64)gridDim.x * blockDim.x;
    double best = -1.0;
    for (u64 i = ilo + (u64)blockIdx.x * blockDim.x + threadIdx.x; i < ihi; i += stride)
        best = fmax(best, item_rel_error(rows, w, i, hi, lo, ilo));
    if (best >= 0.0) atomicMax(worst_bits, (unsigned long long)__double_as_longlong(best));
}

template <typename RowT, typename W>
__global__ void k_mass_argmax(const RowT *__restrict__ rows, const W *__restrict__ w, u64 ilo,
                              u64 ihi, const double *__restrict__ hi,
                              const double *__restrict__ lo, const unsigned long long *worst_bits,
                              unsigned long long *first)
{
    const double target = __longlong_as_double((long long)*worst_bits);
    u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = ilo + (u64)blockIdx.x * blockDim.x + threadIdx.x; i < ihi; i += stride)
        if (item_rel_error(rows, w, i, hi, lo, ilo) == target) atomicMin(first, (unsigned long long)i);
}

// chi-square pieces over bins [0, m) of counts (stats.py:84-121): expected
// e_i = M * w_i / W; bins with e_i >= 5 add (c_i - e_i)^2 / e_i, the others
// are pooled.  out[0] stat of kept bins, out[1] kept bins, out[2] pooled
// observed, out[3] pooled expected (block sums combined by f64 atomics).
template <typename W>
__global__ void k_chi2_partial(const i64 *__restrict__ counts, const W *__restrict__ w, u64 m,
                               double total_w, double draws, double *out)
{
    __shared__ double red[4][8];
    double st = 0.0, kept = 0.0, po = 0.0, pe = 0.0;
    u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        const double p = (double)w[i] / total_w;
        const double e = p * draws;
        const double o = (double)counts[i];
        if (e < 5.0) {
            po += o;
            pe += e;
        } else {
            const double d = o - e;
            st += d * d / e;
            kept += 1.0;
        }
    }
    double v[4] = {st, kept, po, pe};
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        if (lane == 0) red[k][wid] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double a = 0.0;
        for (int j = 0; j < (int)(blockDim.x >> 5); ++j) a += red[threadIdx.x][j];
        atomicAdd(&out[threadIdx.x], a);
    }
}

__global__ void k_freq(const i64 *__restrict__ s, u64 m, u64 n, unsigned long long *counts,
                       int *oor)
{
    u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        i64 v = s[i];
        if (v < 1 || (u64)v > n) {
            atomicOr(oor, 1);
            continue;
        }
        atomicAdd(&counts[v - 1], 1ull);
    }
}

template <typename RowT>
__global__ void k_to_soa(const RowT *__restrict__ rows, u64 n, double *tw, i64 *alias)
{
    u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        RowT r = rows[i];
        tw[i] = (double)r.tw;
        alias[i] = (i64)r.alias;
    }
}

// rows [first, first+count) as ALT1 file rows (f64 threshold, u64 alias)
template <typename RowT>
__global__ void k_to_alt1(const RowT *__restrict__ rows, u64 first, u64 count, double2 *out)
{
    u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const RowT r = rows[first + i];
        out[i] = make_double2((double)r.tw, __longlong_as_double((long long)(u64)r.alias));
    }
}

template <typename RowT>
__global__ void k_from_soa(const double *tw, const i64 *alias, u64 n, RowT *rows)
{
    typedef decltype(RowT::tw) TwT;
    typedef decltype(RowT::alias) AT;
    u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        RowT r;
        r.tw = (TwT)tw[i];
        r.alias = (AT)alias[i];
        rows[i] = r;
    }
}

template <typename RowT>
__global__ void k_unwritten(const RowT *__restrict__ rows, u64 n, unsigned long long *cnt)
{
    u64 stride = (u64)gridDim.x * blockDim.x;
    unsigned long long c = 0;
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        c += rows[i].alias == 0;
    if (c) atomicAdd(cnt, c);
}

int grid_of(u64 n)
{
    u64 g = (n + 255) / 256;
    u64 cap = (u64)ak_num_sms() * 8;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

template <typename RowT, typename W>
int run_validate(const void *rows, u64 n, u64 ilo, u64 ihi, const void *w, double avg,
                 double row_tol, int *rows_ok, double *worst_rel, int64_t *worst_item, void *ws,
                 cudaStream_t st)
{
    const u64 m = ihi - ilo;
    double *hi = (double *)ws;
    double *lo = hi + m;
    unsigned long long *misc = (unsigned long long *)(lo + m);  // [0] worst, [1] first
    int *bad = (int *)(misc + 2);
    AK_CUDA_TRY(cudaMemsetAsync(hi, 0, 2 * m * sizeof(double), st));
    {
        int rc0 = ak_fill_small(misc, 0, 2 * sizeof(unsigned long long) + 16, st);
        if (rc0 == AK_OK) rc0 = ak_fill_small(misc + 1, 0xff, sizeof(unsigned long long), st);
        if (rc0 != AK_OK) return rc0;
    }
    k_donate<RowT><<<grid_of(n), 256, 0, st>>>((const RowT *)rows, n, ilo, ihi, avg, row_tol, hi, lo, bad);
    if (m) {
        k_mass<RowT, W><<<grid_of(m), 256, 0, st>>>((const RowT *)rows, (const W *)w, ilo, ihi, hi, lo, misc);
        k_mass_argmax<RowT, W><<<grid_of(m), 256, 0, st>>>((const RowT *)rows, (const W *)w, ilo, ihi,
                                                          hi, lo, misc, misc + 1);
    }
    AK_LAUNCH_CHECK("k_validate");
    unsigned long long hm[2];
    int b = 0;
    {
        const int rc = ak_readback(st, hm, misc, sizeof(hm), &b, bad, sizeof(int));
        if (rc != AK_OK) return rc;
    }
    *rows_ok = !b;
    *worst_rel = m ? __builtin_bit_cast(double, hm[0]) : 0.0;
    *worst_item = m ? (int64_t)hm[1] + 1 : 0;
    return AK_OK;
}

int validate_dispatch(const void *rows, int dtype, uint64_t n, uint64_t ilo, uint64_t ihi,
                      const void *w, int w_dtype, double avg, double row_tol, int *rows_ok,
                      double *worst_rel, int64_t *worst_item, void *ws, cudaStream_t st)
{
    if (dtype == AK_F32 && w_dtype == AK_F32)
        return run_validate<RowF32, float>(rows, n, ilo, ihi, w, avg, row_tol, rows_ok, worst_rel, worst_item, ws, st);
    if (dtype == AK_F32 && w_dtype == AK_F64)
        return run_validate<RowF32, double>(rows, n, ilo, ihi, w, avg, row_tol, rows_ok, worst_rel, worst_item, ws, st);
    if (dtype == AK_F64 && w_dtype == AK_F32)
        return run_validate<RowF64, float>(rows, n, ilo, ihi, w, avg, row_tol, rows_ok, worst_rel, worst_item, ws, st);
    if (dtype == AK_F64 && w_dtype == AK_F64)
        return run_validate<RowF64, double>(rows, n, ilo, ihi, w, avg, row_tol, rows_ok, worst_rel, worst_item, ws, st);
    return AK_ERR_VALUE;
}

}  // namespace

extern "C" {

size_t ak_validate_workspace_bytes(uint64_t n) { return 2 * n * sizeof(double) + 256; }

int ak_validate_table(const void *rows, int dtype, uint64_t n, const void *w, int w_dtype,
                      double avg, double row_tol, int *rows_ok, double *worst_rel,
                      int64_t *worst_item, void *ws, size_t ws_bytes, void *stream)
{
    return ak_validate_table_range(rows, dtype, n, 0, n, w, w_dtype, avg, row_tol, rows_ok,
                                   worst_rel, worst_item, ws, ws_bytes, stream);
}

int ak_validate_table_range(const void *rows, int dtype, uint64_t n, uint64_t item_lo,
                            uint64_t item_hi, const void *w, int w_dtype, double avg,
                            double row_tol, int *rows_ok, double *worst_rel, int64_t *worst_item,
                            void *ws, size_t ws_bytes, void *stream)
{
    if (n == 0) return AK_ERR_EMPTY_INPUT;
    if (item_lo > item_hi || item_hi > n) return AK_ERR_VALUE;
    if (ws_bytes < ak_validate_workspace_bytes(item_hi - item_lo)) return AK_ERR_WORKSPACE;
    return validate_dispatch(rows, dtype, n, item_lo, item_hi, w, w_dtype, avg, row_tol, rows_ok,
                             worst_rel, worst_item, ws, ak_stream(stream));
}

int ak_chi2_partial(const int64_t *counts, const void *w, int w_dtype, uint64_t m,
                    double total_w, double draws, double *out4, void *stream)
{
    cudaStream_t st = ak_stream(stream);
    {
        const int rc0 = ak_fill_small(out4, 0, 4 * sizeof(double), st);
        if (rc0 != AK_OK) return rc0;
    }
    if (m == 0) return AK_OK;
    if (w_dtype == AK_F32)
        k_chi2_partial<float><<<grid_of(m), 256, 0, st>>>(counts, (const float *)w, m, total_w, draws, out4);
    else if (w_dtype == AK_F64)
        k_chi2_partial<double><<<grid_of(m), 256, 0, st>>>(counts, (const double *)w, m, total_w, draws, out4);
    else
        return AK_ERR_VALUE;
    AK_LAUNCH_CHECK("k_chi2_partial");
    return AK_OK;
}

int ak_frequency_counts(const int64_t *samples, uint64_t m, uint64_t n, int64_t *counts,
                        void *stream)
{
    cudaStream_t st = ak_stream(stream);
    if (n < 1) return AK_ERR_VALUE;
    int *oor = (int *)ak_stream_scratch(st);
    if (!oor) return AK_ERR_CUDA;
    {
        const int rc = ak_fill_small(oor, 0, 16, st);
        if (rc != AK_OK) return rc;
    }
    AK_CUDA_TRY(cudaMemsetAsync(counts, 0, n * sizeof(int64_t), st));
    if (m) k_freq<<<grid_of(m), 256, 0, st>>>(samples, m, n, (unsigned long long *)counts, oor);
    int f = 0;
    {
        const int rc = ak_readback(st, &f, oor, sizeof(int));
        if (rc != AK_OK) return rc;
    }
    AK_LAUNCH_CHECK("k_freq");
    return f ? AK_ERR_INDEX_OUT_OF_RANGE : AK_OK;
}

int ak_rows_to_soa(const void *rows, int dtype, uint64_t n, double *tw, int64_t *alias,
                   void *stream)
{
    if (n == 0) return AK_OK;
    cudaStream_t st = ak_stream(stream);
    if (dtype == AK_F32) k_to_soa<RowF32><<<grid_of(n), 256, 0, st>>>((const RowF32 *)rows, n, tw, alias);
    else if (dtype == AK_F64) k_to_soa<RowF64><<<grid_of(n), 256, 0, st>>>((const RowF64 *)rows, n, tw, alias);
    else return AK_ERR_VALUE;
    AK_LAUNCH_CHECK("k_to_soa");
    return AK_OK;
}

int ak_soa_to_rows(const double *tw, const int64_t *alias, uint64_t n, int dtype, void *rows,
                   void *stream)
{
    if (n == 0) return AK_OK;
    cudaStream_t st = ak_stream(stream);
    if (dtype == AK_F32) k_from_soa<RowF32><<<grid_of(n), 256, 0, st>>>(tw, alias, n, (RowF32 *)rows);
    else if (dtype == AK_F64) k_from_soa<RowF64><<<grid_of(n), 256, 0, st>>>(tw, alias, n, (RowF64 *)rows);
    else return AK_ERR_VALUE;
    AK_LAUNCH_CHECK("k_from_soa");
    return AK_OK;
}

int ak_rows_to_alt1(const void *rows, int dtype, uint64_t n, uint64_t first, uint64_t count,
                    void *out, void *stream)
{
    if (first > n || count > n - first) return AK_ERR_VALUE;
    if (count == 0) return AK_OK;
    cudaStream_t st = ak_stream(stream);
    if (dtype == AK_F32) k_to_alt1<RowF32><<<grid_of(count), 256, 0, st>>>((const RowF32 *)rows, first, count, (double2 *)out);
    else if (dtype == AK_F64) k_to_alt1<RowF64><<<grid_of(count), 256, 0, st>>>((const RowF64 *)rows, first, count, (double2 *)out);
    else return AK_ERR_VALUE;
    AK_LAUNCH_CHECK("k_to_alt1");
    return AK_OK;
}

int ak_count_unwritten(const void *rows, int dtype, uint64_t n, uint64_t *unwritten, void *stream)
{
    cudaStream_t st = ak_stream(stream);
    if (dtype != AK_F32 && dtype != AK_F64) return AK_ERR_VALUE;
    unsigned long long *c = (unsigned long long *)ak_stream_scratch(st);
    if (!c) return AK_ERR_CUDA;
    {
        const int rc = ak_fill_small(c, 0, 16, st);
        if (rc != AK_OK) return rc;
    }
    if (n) {
        if (dtype == AK_F32) k_unwritten<RowF32><<<grid_of(n), 256, 0, st>>>((const RowF32 *)rows, n, c);
        else k_unwritten<RowF64><<<grid_of(n), 256, 0, st>>>((const RowF64 *)rows, n, c);
    }
    unsigned long long h = 0;
    {
        const int rc = ak_readback(st, &h, c, sizeof(h));
        if (rc != AK_OK) return rc;
    }
    AK_LAUNCH_CHECK("k_unwritten");
    *unwritten = h;
    return AK_OK;
}

}  // extern "C"
