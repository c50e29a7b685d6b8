// ak_build.cu — fused PSA construction (psa_construct, pack.py:255-277).
//
// Formulation.  Let d_i = avg - w_i (light deficit) and e_i = w_i - avg (heavy
// excess).  The sequential construction (seqbuild.py:33-58) is a merge of two
// sorted key sequences: light k has key DL(k) = sum of the deficits of the
// lights before it, heavy j has key DH(j) = sum of the excess of the heavies
// up to and including it; heavy j closes before light k iff DH(j) <= DL(k).
// Hence
//   light k:  alias = first heavy (in item order) with DH > DL(k), else self;
//   heavy j:  tw = DH(j) - DL(first light with DL >= DH(j)) + avg,
//             alias = next heavy, or itself when it is the last;
// and the split predicate L[n-h] + H[h] <= n*avg of split.py:69-77 is exactly
// DH(h) <= DL(n-h).  Every row follows from prefix sums, in parallel.
//
// Keys.  Items are grouped in tiles of 2048 (8 chunks of 256, one warp each).
// A key is (tile base, double-double) + (local offset, double): the local part
// comes from a warp-level Kogge-Stone scan whose lane bases are clamped by a
// running max/min into the chunk's [base, bound] so keys never decrease and
// never pass the chunk bound; the chunk bases/bounds are a monotone scan of
// the chunk totals done once by pass 1 and stored.  Any warp can therefore
// rebuild the canonical keys of any chunk, bit-identically, without a block
// barrier.  Cross-tile comparisons are exact: a local key plus the double-
// double difference of two tile bases is formed as a normalised double-double
// and compared with a local key.
//
// Pipeline (three kernels):
//  1. k_build_scan   one pass over the weights (128-bit loads): classify, chunk
//                    scans, per-tile totals and chunk bounds; a single-pass
//                    decoupled look-back over super-tiles (32 tiles per CTA,
//                    so the inclusive frontier outruns DRAM) produces the
//                    exclusive tile bases DLb[t], DHb[t] (exact double-double
//                    sums) and light counts kL[t].
//  2. k_build_coarse merge of the two tile-boundary sequences: for each tile
//                    the first heavy tile covering its light keys (T1) and
//                    the first light tile covering its heavy keys (S1), and
//                    the first heavy after it (nextH).
//  3. k_build_pack   persistent warps stream through runs of chunks taken in
//                    order from a global queue, resolving each own chunk
//                    against two sliding windows of foreign keys (the heavies
//                    after its lights, the lights at or after its heavies),
//                    advanced chunk by chunk; rows staged in shared memory
//                    and stored once, coalesced.
//  DRAM traffic ~ read w twice + write the rows once = the algorithmic bytes.
#include "ak_common.cuh"

namespace {

constexpr int TB = 256;            // threads per CTA
constexpr int VV = 8;              // items per lane
constexpr int CH = 32 * VV;        // items per chunk (one warp)
constexpr int NW = TB / 32;        // chunks per tile
constexpr int TILE = TB * VV;      // items per tile
constexpr int SUPER = 32;          // tiles per pass-1 CTA (look-back granularity)
constexpr u64 NONE64 = ~0ull;
constexpr unsigned char NOFH = 0xFF;

// ---------------------------------------------------------------------------
// workspace layout
// ---------------------------------------------------------------------------
struct BuildWs {
    u64 nt, nst;  // tiles, super-tiles
    unsigned int *counter;
    u32 *status;            // [nst] 0 none, 1 aggregate, 2 inclusive
    dd *agg_D, *agg_H;      // [nst] super-tile aggregates (write once)
    u64 *agg_k;             // [nst]
    dd *inc_D, *inc_H;      // [nst] inclusive prefixes (write once)
    u64 *inc_k;             // [nst]
    dd *DLb, *DHb;          // [nt+1] exclusive tile bases
    u64 *kL;                // [nt+1] lights before tile
    u64 *firstH;            // [nt]
    double *mD, *mE;        // [nt*8] chunk bounds (monotone inclusive scans)
    unsigned char *mfh;     // [nt*8] first heavy offset in chunk, NOFH if none
    u32 *T1, *S1;           // [nt+1]
    u64 *nextH;             // [nt]
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

template <typename F> inline void layout(u64 n, F &&take)
{
    u64 nt = (n + TILE - 1) / TILE;
    u64 nst = (nt + SUPER - 1) / SUPER;
    size_t sizes[19] = {256,          nst * 4,      nst * 16,       nst * 16,       nst * 8,
                        nst * 16,     nst * 16,     nst * 8,        (nt + 1) * 16,  (nt + 1) * 16,
                        (nt + 1) * 8, nt * 8,       nt * NW * 8,    nt * NW * 8,    nt * NW,
                        (nt + 1) * 4, (nt + 1) * 4, nt * 8,         0};
    for (int i = 0; i < 18; ++i) take(i, sizes[i]);
}

inline BuildWs carve(void *ws, u64 n)
{
    BuildWs W;
    W.nt = (n + TILE - 1) / TILE;
    W.nst = (W.nt + SUPER - 1) / SUPER;
    char *base = (char *)ws;
    size_t off = 0;
    char *p[18];
    layout(n, [&](int i, size_t b) {
        p[i] = base + off;
        off += align256(b);
    });
    W.counter = (unsigned int *)p[0];
    W.status = (u32 *)p[1];
    W.agg_D = (dd *)p[2];
    W.agg_H = (dd *)p[3];
    W.agg_k = (u64 *)p[4];
    W.inc_D = (dd *)p[5];
    W.inc_H = (dd *)p[6];
    W.inc_k = (u64 *)p[7];
    W.DLb = (dd *)p[8];
    W.DHb = (dd *)p[9];
    W.kL = (u64 *)p[10];
    W.firstH = (u64 *)p[11];
    W.mD = (double *)p[12];
    W.mE = (double *)p[13];
    W.mfh = (unsigned char *)p[14];
    W.T1 = (u32 *)p[15];
    W.S1 = (u32 *)p[16];
    W.nextH = (u64 *)p[17];
    return W;
}

size_t ws_bytes_for(u64 n)
{
    size_t off = 0;
    layout(n, [&](int, size_t b) { off += align256(b); });
    return off + 256;
}

// ---------------------------------------------------------------------------
// loads and the canonical warp scan
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void load8(const T *__restrict__ w, u64 n, u64 i0, double v[VV])
{
    if (i0 + VV <= n) {
        if (sizeof(T) == 4) {
            const float4 *p = reinterpret_cast<const float4 *>(w + i0);
            float4 a = __ldg(p), b = __ldg(p + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
            const double2 *p = reinterpret_cast<const double2 *>(w + i0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double2 a = __ldg(p + q);
                v[2 * q] = a.x;
                v[2 * q + 1] = a.y;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < VV; ++k) v[k] = (i0 + k < n) ? (double)w[i0 + k] : -1.0;  // absent
    }
}

// inclusive Kogge-Stone scan followed by a running max: non-decreasing
__device__ __forceinline__ double warp_scan_mono(double x, int lane)
{
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        double y = shfl_up_d(x, d);
        if (lane >= d) x = x + y;
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        double y = shfl_up_d(x, d);
        if (lane >= d) x = fmax(x, y);
    }
    return x;
}

// Lane-level part of the canonical chunk scan for one class: per-item local
// prefixes (exclusive for lights, inclusive for heavies), the lane's
// exclusive base within the chunk and the chunk total.
template <bool LIGHT>
__device__ __forceinline__ void lane_class(const double v[VV], double avg, double loc[VV], u32 &mask,
                                           double &excl, double &total, int lane)
{
    double s = 0.0;
    u32 m = 0;
#pragma unroll
    for (int k = 0; k < VV; ++k) {
        const bool valid = v[k] >= 0.0;
        const bool in = LIGHT ? (valid && v[k] <= avg) : (valid && v[k] > avg);
        if (LIGHT) loc[k] = s;
        if (in) s = s + (LIGHT ? (avg - v[k]) : (v[k] - avg));
        if (!LIGHT) loc[k] = s;
        m |= (u32)in << k;
    }
    double inc = warp_scan_mono(s, lane);
    excl = shfl_up_d(inc, 1);
    if (lane == 0) excl = 0.0;
    total = inc;  // unused by callers that take bounds from pass 1
    mask = m;
}

// Lane sums of one class and the canonical chunk total: a butterfly (xor)
// tree sum, identical in every lane and every kernel.
template <bool LIGHT>
__device__ __forceinline__ double chunk_total(const double v[VV], double avg, u32 &mask)
{
    double s = 0.0;
    u32 m = 0;
#pragma unroll
    for (int k = 0; k < VV; ++k) {
        const bool valid = v[k] >= 0.0;
        const bool in = LIGHT ? (valid && v[k] <= avg) : (valid && v[k] > avg);
        if (in) s = s + (LIGHT ? (avg - v[k]) : (v[k] - avg));
        m |= (u32)in << k;
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) s = s + __shfl_xor_sync(0xffffffffu, s, d);
    mask = m;
    return s;
}

// Canonical keys of one class given the chunk's [base, bound].
__device__ __forceinline__ void class_keys(double loc[VV], double excl, double base, double bound,
                                           int lane)
{
    double B = fmin(base + excl, bound);
    double U = __shfl_down_sync(0xffffffffu, B, 1);
    if (lane == 31) U = bound;
#pragma unroll
    for (int k = 0; k < VV; ++k) loc[k] = fmin(B + loc[k], U);
}

// offset of the first set item in the chunk (lane-major), NOFH if none
__device__ __forceinline__ unsigned char first_item(u32 mask, int lane)
{
    unsigned b = __ballot_sync(0xffffffffu, mask != 0);
    if (!b) return NOFH;
    int fl = __ffs(b) - 1;
    u32 fm = __shfl_sync(0xffffffffu, mask, fl);
    return (unsigned char)(fl * VV + __ffs(fm) - 1);
}

// ---------------------------------------------------------------------------
// 1. scan + super-tile decoupled look-back
// ---------------------------------------------------------------------------
__device__ __forceinline__ dd shfl_xor_dd(dd x, int m)
{
    return dd_make(__shfl_xor_sync(0xffffffffu, x.hi, m), __shfl_xor_sync(0xffffffffu, x.lo, m));
}

template <typename T>
__global__ void __launch_bounds__(TB) k_build_scan(const T *__restrict__ w, u64 n, double avg,
                                                   BuildWs W)
{
    __shared__ double s_cD[NW], s_cE[NW];
    __shared__ u32 s_cL[NW];
    __shared__ unsigned char s_fh[NW];
    __shared__ double s_tD[SUPER], s_tE[SUPER];
    __shared__ u32 s_tL[SUPER];
    __shared__ u64 s_fH[SUPER];
    __shared__ unsigned int s_st;
    __shared__ dd s_exD, s_exH, s_agD, s_agH;
    __shared__ u64 s_exK, s_agK;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_st = atomicAdd(W.counter, 1u);
    __syncthreads();
    const u64 st = s_st;
    const u64 t0 = st * SUPER;
    const u64 tn = (t0 + SUPER <= W.nt) ? SUPER : W.nt - t0;

    double vnext[VV];
    load8(w, n, t0 * TILE + (u64)threadIdx.x * VV, vnext);
    for (u64 j = 0; j < tn; ++j) {
        const u64 t = t0 + j;
        double v[VV];
#pragma unroll
        for (int k = 0; k < VV; ++k) v[k] = vnext[k];
        if (j + 1 < tn) load8(w, n, (t + 1) * TILE + (u64)threadIdx.x * VV, vnext);
        u32 lm, hm;
        const double totD = chunk_total<true>(v, avg, lm);
        const double totE = chunk_total<false>(v, avg, hm);
        u32 nl = __popc(lm);
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) nl += __shfl_xor_sync(0xffffffffu, nl, d);
        const unsigned char fh = first_item(hm, lane);
        if (lane == 0) {
            s_cD[wid] = totD;
            s_cE[wid] = totE;
            s_cL[wid] = nl;
            s_fh[wid] = fh;
        }
        __syncthreads();
        if (wid == 0) {
            // monotone scan of the chunk totals -> chunk bounds
            double x = lane < NW ? s_cD[lane] : 0.0, y = lane < NW ? s_cE[lane] : 0.0;
#pragma unroll
            for (int d = 1; d < NW; d <<= 1) {
                double a = shfl_up_d(x, d), b = shfl_up_d(y, d);
                if (lane >= d) { x = x + a; y = y + b; }
            }
#pragma unroll
            for (int d = 1; d < NW; d <<= 1) {
                double a = shfl_up_d(x, d), b = shfl_up_d(y, d);
                if (lane >= d) { x = fmax(x, a); y = fmax(y, b); }
            }
            const unsigned char f = lane < NW ? s_fh[lane] : NOFH;
            if (lane < NW) {
                W.mD[t * NW + lane] = x;
                W.mE[t * NW + lane] = y;
                W.mfh[t * NW + lane] = f;
            }
            u32 cl = lane < NW ? s_cL[lane] : 0;
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) cl += __shfl_xor_sync(0xffffffffu, cl, d);
            unsigned fhm = __ballot_sync(0xffffffffu, lane < NW && f != NOFH);
            const int c = fhm ? __ffs(fhm) - 1 : 0;
            const unsigned char fc = (unsigned char)__shfl_sync(0xffffffffu, (int)f, c);
            if (lane == NW - 1) {
                s_tD[j] = x;
                s_tE[j] = y;
            }
            if (lane == 0) {
                s_tL[j] = cl;
                s_fH[j] = fhm ? t * TILE + (u64)c * CH + fc : NONE64;
            }
        }
        __syncthreads();
    }
    // super-tile aggregate: exact double-double sum of the tile totals
    if (threadIdx.x == 0) {
        dd aD = dd_make(0.0), aH = dd_make(0.0);
        u64 aK = 0;
        for (u64 j = 0; j < tn; ++j) {
            aD = dd_add_d(aD, s_tD[j]);
            aH = dd_add_d(aH, s_tE[j]);
            aK += s_tL[j];
        }
        s_agD = aD;
        s_agH = aH;
        s_agK = aK;
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
    __syncthreads();
    // look-back by warp 0
    if (threadIdx.x < 32) {
        dd aD = dd_make(0.0), aH = dd_make(0.0);
        u64 aK = 0;
        i64 pred = (i64)st - 1;
        while (pred >= 0) {
            const i64 p = pred - lane;
            u32 s = 2;
            if (p >= 0) {
                do { s = ld_acquire_u32(&W.status[p]); } while (s == 0);
            }
            const unsigned inc_mask = __ballot_sync(0xffffffffu, p >= 0 && s == 2);
            const int stop = inc_mask ? __ffs(inc_mask) - 1 : 32;
            dd cD = dd_make(0.0), cH = dd_make(0.0);
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
                cD = dd_add(cD, shfl_xor_dd(cD, m));
                cH = dd_add(cH, shfl_xor_dd(cH, m));
                cK += __shfl_xor_sync(0xffffffffu, cK, m);
            }
            aD = dd_add(aD, cD);
            aH = dd_add(aH, cH);
            aK += cK;
            if (stop < 32 || pred - 32 < 0) break;
            pred -= 32;
        }
        if (lane == 0) {
            if (st > 0) {
                W.inc_D[st] = dd_add(aD, s_agD);
                W.inc_H[st] = dd_add(aH, s_agH);
                W.inc_k[st] = aK + s_agK;
                __threadfence();
                st_release_u32(&W.status[st], 2u);
            }
            s_exD = aD;
            s_exH = aH;
            s_exK = aK;
        }
    }
    __syncthreads();
    // exclusive bases of the super-tile's tiles
    if (threadIdx.x == 0) {
        dd D = s_exD, H = s_exH;
        u64 K = s_exK;
        for (u64 j = 0; j < tn; ++j) {
            const u64 t = t0 + j;
            W.DLb[t] = D;
            W.DHb[t] = H;
            W.kL[t] = K;
            W.firstH[t] = s_fH[j];
            D = dd_add_d(D, s_tD[j]);
            H = dd_add_d(H, s_tE[j]);
            K += s_tL[j];
        }
        if (t0 + tn == W.nt) {
            W.DLb[W.nt] = D;
            W.DHb[W.nt] = H;
            W.kL[W.nt] = K;
        }
    }
}

// ---------------------------------------------------------------------------
// 2. coarse merge of the tile boundaries
// ---------------------------------------------------------------------------
__global__ void k_build_coarse(BuildWs W, u64 n)
{
    const u64 nt = W.nt;
    u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (u > nt) return;
    {  // T1[u] = max{t in [0, nt] : DHb[t] <= DLb[u]}
        const dd x = W.DLb[u];
        u64 lo = 0, hi = nt;
        while (lo < hi) {
            u64 mid = (lo + hi + 1) >> 1;
            if (dd_le(W.DHb[mid], x)) lo = mid;
            else hi = mid - 1;
        }
        W.T1[u] = (u32)lo;
    }
    {  // S1[u] = max{s in [0, nt] : DLb[s] < DHb[u]}, 0 if none
        const dd y = W.DHb[u];
        if (!dd_lt(W.DLb[0], y)) {
            W.S1[u] = 0;
        } else {
            u64 lo = 0, hi = nt;
            while (lo < hi) {
                u64 mid = (lo + hi + 1) >> 1;
                if (dd_lt(W.DLb[mid], y)) lo = mid;
                else hi = mid - 1;
            }
            W.S1[u] = (u32)lo;
        }
    }
    if (u < nt) {  // nextH[u]: first heavy item in tiles > u
        auto jH = [&](u64 t) -> u64 {
            u64 items = t * TILE < n ? t * TILE : n;
            return items - W.kL[t];
        };
        const u64 after = jH(u + 1);
        if (jH(nt) <= after) {
            W.nextH[u] = NONE64;
        } else {
            u64 lo = u + 1, hi = nt - 1;
            while (lo < hi) {
                u64 mid = (lo + hi) >> 1;
                if (jH(mid + 1) > after) hi = mid;
                else lo = mid + 1;
            }
            W.nextH[u] = W.firstH[lo];
        }
    }
}

// ---------------------------------------------------------------------------
// 3. warp-streaming pack
// ---------------------------------------------------------------------------
// Every warp takes runs of RUN consecutive chunks from a global queue (runs
// are handed out in order, so the runs in flight — and the foreign chunks
// they read — stay L2-resident) and streams through them.  It keeps two
// warp-private sliding windows of global double-double keys:
//   HW: the heavies following its current lights in key order,
//   LW: the lights at or after its current heavies in key order,
// each advanced monotonically by rebuilding the canonical keys of the next
// foreign chunk of that class (chunks whose key range lies entirely behind
// the request are skipped via the pass-1 chunk bounds).  An own chunk is
// resolved against the windows and its 256 rows are stored once, coalesced.
// No block barriers: warps are independent.
constexpr int RUN = 16;          // chunks per queue item
constexpr int WCAP = 512;        // window capacity (entries); a chunk adds <= 256
constexpr int PW = 4;            // warps per CTA

template <typename T> struct WarpSmem {
    dd OK[CH];                        // own global keys: lights [0,nl), heavies [nl,nl+nh)
    dd HK[WCAP];                      // heavy window keys (ring)
    dd LK[WCAP];                      // light window keys (ring)
    typename RowOf<T>::type RW[CH];   // staged rows
    u32 HI[WCAP];                     // heavy window items (0-based)
    unsigned char OP[CH];             // own item offsets
};

// d + x as a normalised double-double (exact for the key ranges in play)
__device__ __forceinline__ dd add_dd_d(dd d, double x)
{
    double s, e;
    two_sum(d.hi, x, s, e);
    e += d.lo;
    double h, l;
    fast_two_sum(s, e, h, l);
    return dd_make(h, l);
}

__device__ __forceinline__ dd chunk_base(const BuildWs &W, u64 g, bool light, bool upper)
{
    // global lower (upper) bound of the keys of one class in chunk g
    const u64 t = g / NW;
    const int c = (int)(g % NW);
    const double *mB = light ? W.mD : W.mE;
    const double loc = upper ? mB[g] : (c ? mB[g - 1] : 0.0);
    return add_dd_d(light ? W.DLb[t] : W.DHb[t], loc);
}

// Canonical global keys of one class of chunk g, appended to a window ring.
// Returns the number appended.
template <typename T, bool LIGHT>
__device__ __forceinline__ u32 append_chunk(const T *__restrict__ w, u64 n, double avg,
                                            const BuildWs &W, u64 g, dd *K, u32 *I, u32 tail,
                                            int lane)
{
    const u64 t = g / NW;
    const int c = (int)(g % NW);
    const double *mB = LIGHT ? W.mD : W.mE;
    const double base = c ? mB[g - 1] : 0.0, bound = mB[g];
    const dd B = LIGHT ? W.DLb[t] : W.DHb[t];
    double v[VV], k[VV], ex, tot;
    u32 m;
    load8(w, n, g * CH + (u64)lane * VV, v);
    lane_class<LIGHT>(v, avg, k, m, ex, tot, lane);
    class_keys(k, ex, base, bound, lane);
    const u32 cnt = __popc(m);
    u32 inc = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        u32 a = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += a;
    }
    const u32 total = __shfl_sync(0xffffffffu, inc, 31);
    u32 r = tail + inc - cnt;
#pragma unroll
    for (int q = 0; q < VV; ++q)
        if ((m >> q) & 1) {
            const u32 s = r & (WCAP - 1);
            K[s] = add_dd_d(B, k[q]);
            if (!LIGHT) I[s] = (u32)(g * CH + lane * VV + q);
            ++r;
        }
    __syncwarp();
    return total;
}

// first index i in [0, cnt) of the ring (from head) with pred(K[i]) false,
// pred monotone (true then false); warp-uniform
template <typename P>
__device__ __forceinline__ u32 ring_search(const dd *K, u32 head, u32 cnt, P pred)
{
    u32 a = 0, b = cnt;
    while (a < b) {
        const u32 mid = (a + b) >> 1;
        if (pred(K[(head + mid) & (WCAP - 1)])) a = mid + 1;
        else b = mid;
    }
    return a;
}

// seek: first chunk g >= from whose class bound passes key x
// (heavies: bound > x; lights: bound >= x), G if none
template <bool LIGHT>
__device__ u64 seek_chunk(const BuildWs &W, u64 from, u64 G, dd x)
{
    auto passes = [&](u64 g) {
        const dd b = chunk_base(W, g, LIGHT, true);
        return LIGHT ? !dd_lt(b, x) : dd_lt(x, b);
    };
    if (from >= G || passes(from)) return from;
    // gallop, then bisect
    u64 lo = from, step = 1;  // invariant: !passes(lo)
    while (lo + step < G && !passes(lo + step)) {
        lo += step;
        step <<= 1;
    }
    u64 hi = lo + step < G ? lo + step : G;  // passes(hi) or hi == G
    while (hi - lo > 1) {
        const u64 mid = (lo + hi) >> 1;
        if (passes(mid)) hi = mid;
        else lo = mid;
    }
    return hi;
}

template <typename T>
__global__ void __launch_bounds__(PW * 32) k_build_pack(const T *__restrict__ w, u64 n,
                                                        double avg, BuildWs W,
                                                        typename RowOf<T>::type *__restrict__ rows_out,
                                                        unsigned int *queue)
{
    typedef typename RowOf<T>::type RowT;
    typedef decltype(RowT::alias) AliasT;
    extern __shared__ __align__(16) unsigned char pack_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WarpSmem<T> &S = reinterpret_cast<WarpSmem<T> *>(pack_smem)[wid];
    const u64 G = (n + CH - 1) / CH;  // chunks
    const u64 nt = W.nt;
    const u64 nruns = (G + RUN - 1) / RUN;
    const dd Dtot = W.DLb[nt];
    for (;;) {
        u32 run = 0;
        if (lane == 0) run = atomicAdd(queue, 1u);
        run = __shfl_sync(0xffffffffu, run, 0);
        if (run >= nruns) break;
        const u64 g0 = (u64)run * RUN, g1 = g0 + RUN < G ? g0 + RUN : G;
        // windows start empty; cursors seek on first use
        u32 hh = 0, hc = 0, lh = 0, lc = 0;
        u64 gh = g0 / NW < nt ? (u64)W.T1[g0 / NW] * NW : G;  // first candidate heavy chunk
        u64 gl = (u64)W.S1[g0 / NW] * NW;                      // first candidate light chunk
        if (gh > G) gh = G;
        if (gl > G) gl = G;
        double vn[VV];
        load8(w, n, g0 * CH + (u64)lane * VV, vn);
        for (u64 g = g0; g < g1; ++g) {
            const u64 t = g / NW;
            const int c = (int)(g % NW);
            const u64 cb = g * CH;
            double v[VV];
#pragma unroll
            for (int k = 0; k < VV; ++k) v[k] = vn[k];
            if (g + 1 < g1) load8(w, n, (g + 1) * CH + (u64)lane * VV, vn);
            // ---- own chunk: global keys of both classes, compacted
            u32 lm, hm, nl, nh;
            {
                const double bD0 = c ? W.mD[g - 1] : 0.0, bD1 = W.mD[g];
                const double bE0 = c ? W.mE[g - 1] : 0.0, bE1 = W.mE[g];
                const dd DLu = W.DLb[t], DHu = W.DHb[t];
                double kD[VV], kE[VV], exD, exE, tD, tE;
                lane_class<true>(v, avg, kD, lm, exD, tD, lane);
                class_keys(kD, exD, bD0, bD1, lane);
                lane_class<false>(v, avg, kE, hm, exE, tE, lane);
                class_keys(kE, exE, bE0, bE1, lane);
                const u32 cl = __popc(lm), chh = __popc(hm);
                u32 il = cl, ih = chh;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    u32 a = __shfl_up_sync(0xffffffffu, il, d), b = __shfl_up_sync(0xffffffffu, ih, d);
                    if (lane >= d) { il += a; ih += b; }
                }
                nl = __shfl_sync(0xffffffffu, il, 31);
                nh = __shfl_sync(0xffffffffu, ih, 31);
                u32 rl = il - cl, rh = nl + ih - chh;
#pragma unroll
                for (int k = 0; k < VV; ++k) {
                    const u32 pos = lane * VV + k;
                    if ((lm >> k) & 1) {
                        S.OK[rl] = add_dd_d(DLu, kD[k]);
                        S.OP[rl] = (unsigned char)pos;
                        S.RW[pos].tw = (decltype(RowT::tw))v[k];
                        ++rl;
                    } else if ((hm >> k) & 1) {
                        S.OK[rh] = add_dd_d(DHu, kE[k]);
                        S.OP[rh] = (unsigned char)pos;
                        ++rh;
                    }
                }
            }
            __syncwarp();
            // heavy aliases: next heavy in the chunk, else after it
            if (nh) {
                const unsigned char fh = lane < NW ? W.mfh[t * NW + lane] : NOFH;
                unsigned m = __ballot_sync(0xffffffffu, lane < NW && lane > c && fh != NOFH);
                u64 after;
                if (m) {
                    const int cc = __ffs(m) - 1;
                    after = t * TILE + (u64)cc * CH + (unsigned char)__shfl_sync(0xffffffffu, (int)fh, cc);
                } else {
                    after = W.nextH[t];
                }
                for (u32 r = lane; r < nh; r += 32) {
                    const u32 pos = S.OP[nl + r];
                    u64 a;
                    if (r + 1 < nh) a = cb + S.OP[nl + r + 1] + 1;
                    else a = (after == NONE64) ? cb + pos + 1 : after + 1;
                    S.RW[pos].alias = (AliasT)a;
                }
            }
            // ---- lights: alias = first heavy key > light key
            for (u32 r0 = 0; r0 < nl;) {
                const dd x0 = S.OK[r0], xm = S.OK[nl - 1];
                // drop heavies with key <= x0
                const u32 d = ring_search(S.HK, hh, hc, [&](dd k) { return dd_le(k, x0); });
                hh = (hh + d) & (WCAP - 1);
                hc -= d;
                // fill until a heavy key > xm is present
                while ((hc == 0 || dd_le(S.HK[(hh + hc - 1) & (WCAP - 1)], xm)) && gh < G &&
                       hc + CH <= WCAP) {
                    if (hc == 0) gh = seek_chunk<false>(W, gh, G, x0);
                    if (gh >= G) break;
                    hc += append_chunk<T, false>(w, n, avg, W, gh, S.HK, S.HI, hh + hc, lane);
                    ++gh;
                }
                u32 r1;
                if (hc == 0) {
                    r1 = nl;  // no heavy key past these lights: own rows
                    for (u32 r = r0 + lane; r < r1; r += 32) {
                        const u32 pos = S.OP[r];
                        S.RW[pos].alias = (AliasT)(cb + pos + 1);
                    }
                } else {
                    const dd last = S.HK[(hh + hc - 1) & (WCAP - 1)];
                    r1 = nl;
                    if (!dd_lt(xm, last)) {  // window ends inside this chunk's lights
                        u32 a = r0, b = nl;
                        while (a < b) {
                            const u32 mid = (a + b) >> 1;
                            if (dd_lt(S.OK[mid], last)) a = mid + 1;
                            else b = mid;
                        }
                        r1 = a;
                        if (gh >= G) r1 = nl;  // nothing left to append: the rest have no heavy past them
                    }
                    for (u32 r = r0 + lane; r < r1; r += 32) {
                        const dd x = S.OK[r];
                        const u32 i = ring_search(S.HK, hh, hc, [&](dd k) { return dd_le(k, x); });
                        const u32 pos = S.OP[r];
                        const u64 al = i < hc ? (u64)S.HI[(hh + i) & (WCAP - 1)] + 1 : cb + pos + 1;
                        S.RW[pos].alias = (AliasT)al;
                    }
                }
                __syncwarp();
                r0 = r1;
            }
            // ---- heavies: tw = key - (first light key >= heavy key) + avg
            for (u32 r0 = 0; r0 < nh;) {
                const dd y0 = S.OK[nl + r0], ym = S.OK[nl + nh - 1];
                const u32 d = ring_search(S.LK, lh, lc, [&](dd k) { return dd_lt(k, y0); });
                lh = (lh + d) & (WCAP - 1);
                lc -= d;
                while ((lc == 0 || dd_lt(S.LK[(lh + lc - 1) & (WCAP - 1)], ym)) && gl < G &&
                       lc + CH <= WCAP) {
                    if (lc == 0) gl = seek_chunk<true>(W, gl, G, y0);
                    if (gl >= G) break;
                    lc += append_chunk<T, true>(w, n, avg, W, gl, S.LK, nullptr, lh + lc, lane);
                    ++gl;
                }
                u32 r1 = nh;
                if (lc > 0) {
                    const dd last = S.LK[(lh + lc - 1) & (WCAP - 1)];
                    if (dd_lt(last, ym) && gl < G) {  // window ends inside: resolve y <= last
                        u32 a = r0, b = nh;
                        while (a < b) {
                            const u32 mid = (a + b) >> 1;
                            if (dd_le(S.OK[nl + mid], last)) a = mid + 1;
                            else b = mid;
                        }
                        r1 = a;
                    }
                }
                for (u32 r = r0 + lane; r < r1; r += 32) {
                    const dd y = S.OK[nl + r];
                    const u32 i = ring_search(S.LK, lh, lc, [&](dd k) { return dd_lt(k, y); });
                    const dd DL = i < lc ? S.LK[(lh + i) & (WCAP - 1)] : Dtot;
                    const dd tw = dd_add_d(dd_sub(y, DL), avg);
                    S.RW[S.OP[nl + r]].tw = tw_store<T>(tw.hi + tw.lo, avg);
                }
                __syncwarp();
                r0 = r1;
            }
            __syncwarp();
            // ---- store the chunk's rows (each lane its 8 consecutive rows)
            const u64 i0 = cb + (u64)lane * VV;
            if (i0 + VV <= n) {
                const uint4 *src = reinterpret_cast<const uint4 *>(&S.RW[lane * VV]);
                uint4 *dst = reinterpret_cast<uint4 *>(rows_out + i0);
#pragma unroll
                for (int q = 0; q < (int)(VV * sizeof(RowT) / 16); ++q) dst[q] = src[q];
            } else {
                for (int k = 0; k < VV; ++k)
                    if (i0 + k < n) rows_out[i0 + k] = S.RW[lane * VV + k];
            }
            __syncwarp();
        }
    }
}

template <typename T>
int run_build(const void *wv, u64 n, double total, void *rows, void *ws, cudaStream_t st)
{
    const T *w = (const T *)wv;
    BuildWs W = carve(ws, n);
    const double avg = total / (double)n;
    AK_CUDA_TRY(cudaMemsetAsync(W.counter, 0, 256, st));
    AK_CUDA_TRY(cudaMemsetAsync(W.status, 0, W.nst * 4, st));
    k_build_scan<T><<<(unsigned)W.nst, TB, 0, st>>>(w, n, avg, W);
    AK_LAUNCH_CHECK("k_build_scan");
    k_build_coarse<<<(unsigned)((W.nt + 1 + 255) / 256), 256, 0, st>>>(W, n);
    AK_LAUNCH_CHECK("k_build_coarse");
    const size_t smem = sizeof(WarpSmem<T>) * PW;
    AK_CUDA_TRY(cudaFuncSetAttribute(k_build_pack<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    int per_sm = 0;
    AK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_build_pack<T>, PW * 32, smem));
    if (per_sm < 1) per_sm = 1;
    const u64 G = (n + CH - 1) / CH, nruns = (G + RUN - 1) / RUN;
    u64 grid = (u64)ak_num_sms() * per_sm;
    if (grid * PW > nruns) grid = (nruns + PW - 1) / PW;
    k_build_pack<T><<<(unsigned)grid, PW * 32, smem, st>>>(w, n, avg, W, (typename RowOf<T>::type *)rows,
                                                          W.counter + 1);
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
    if (n == 0) return AK_ERR_EMPTY_INPUT;
    if (ws_bytes < ws_bytes_for(n)) return AK_ERR_WORKSPACE;
    if (((uintptr_t)w & 15) != 0 || ((uintptr_t)rows & 15) != 0) return AK_ERR_VALUE;
    cudaStream_t st = ak_stream(stream);
    if (dtype == AK_F32) {
        if (n >= 0xFFFFFFFFull) return AK_ERR_VALUE;  // u32 aliases
        return run_build<float>(w, n, total, rows, ws, st);
    }
    if (dtype == AK_F64) {
        if (n >= 0xFFFFFFFFull) return AK_ERR_VALUE;  // u32 item ids in the pack windows
        return run_build<double>(w, n, total, rows, ws, st);
    }
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
