// ak_build.cu — fused PSA construction (psa_construct, pack.py:255-277).
//
// Formulation.  Let d_i = avg - w_i (light deficit) and e_i = w_i - avg (heavy
// excess).  The sequential construction (seqbuild.py:33-58) is a merge of two
// sorted key sequences: light k has key DL(k) = sum of deficits of the lights
// before it, heavy j has key DH(j) = sum of excess of heavies up to and
// including it; heavy j closes before light k iff DH(j) <= DL(k).  Hence
//   light k:  alias = first heavy (in item order) with DH > DL(k), else self;
//   heavy j:  tw = DH(j) - DL(first light with DL >= DH(j)) + avg,
//             alias = next heavy, or itself when it is the last;
// and the split predicate L[n-h] + H[h] <= n*avg of split.py:69-77 is exactly
// DH(h) <= DL(n-h).  Every row follows from prefix sums, in parallel.
//
// Pipeline (three kernels, TILE = 2048 items):
//  1. k_build_scan   read the weights once (128-bit loads); classify; block
//                    scan of deficits / excess / light counts per tile; a
//                    single-pass decoupled look-back chains the tile totals
//                    into exclusive tile bases DLb[t], DHb[t] (double-double,
//                    exact sums) and light counts kL[t].
//  2. k_build_coarse merge of the two boundary sequences: for each tile the
//                    range of heavy tiles whose keys cover its lights
//                    (T1) and of light tiles covering its heavies (S1), and
//                    the first heavy after it (nextH).
//  3. k_build_pack   tile-owner pack: a CTA owns the rows of one item tile,
//                    rescans it, resolves its lights against the covering
//                    heavy tiles and its heavies against the covering light
//                    tiles (usually one or two each, L2-resident because
//                    neighbouring CTAs own them), and writes its rows once,
//                    coalesced.  DRAM traffic ~ read w twice + write rows.
//
// Keys inside a tile come from one deterministic "monotone" block scan (lane
// and warp bases clamped by max/min so keys never decrease and never exceed
// the tile total), so every CTA that rescans a tile sees bit-identical keys
// and tile totals.  Cross-tile comparisons are exact: (a - b) of two local
// f64 keys is formed as an exact double-double and compared with the
// double-double difference of the tile bases.
#include "ak_common.cuh"

namespace {

constexpr int TB = 256;           // threads per CTA
constexpr int VV = 8;             // items per thread
constexpr int TILE = TB * VV;     // items per tile
constexpr int NWARP = TB / 32;
constexpr u64 NONE64 = ~0ull;

// ---------------------------------------------------------------------------
// workspace layout
// ---------------------------------------------------------------------------
struct BuildWs {
    u64 nt;  // tiles
    unsigned int *counter;
    u32 *status;
    double *agg_d, *agg_e;
    u32 *agg_n;
    dd *inc_D, *inc_H;
    u64 *inc_k;
    dd *DLb, *DHb;   // [nt+1]
    u64 *kL;         // [nt+1]
    u64 *firstH;     // [nt]
    u32 *T1, *S1;    // [nt+1]
    u64 *nextH;      // [nt]
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

__host__ __device__ inline BuildWs carve(void *ws, u64 n)
{
    BuildWs W;
    u64 nt = (n + TILE - 1) / TILE;
    W.nt = nt;
    char *p = (char *)ws;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char *r = p + off;
        off += align256(bytes);
        return r;
    };
    W.counter = (unsigned int *)take(256);
    W.status = (u32 *)take(nt * 4);
    W.agg_d = (double *)take(nt * 8);
    W.agg_e = (double *)take(nt * 8);
    W.agg_n = (u32 *)take(nt * 4);
    W.inc_D = (dd *)take(nt * 16);
    W.inc_H = (dd *)take(nt * 16);
    W.inc_k = (u64 *)take(nt * 8);
    W.DLb = (dd *)take((nt + 1) * 16);
    W.DHb = (dd *)take((nt + 1) * 16);
    W.kL = (u64 *)take((nt + 1) * 8);
    W.firstH = (u64 *)take(nt * 8);
    W.T1 = (u32 *)take((nt + 1) * 4);
    W.S1 = (u32 *)take((nt + 1) * 4);
    W.nextH = (u64 *)take(nt * 8);
    return W;
}

size_t ws_bytes_for(u64 n)
{
    u64 nt = (n + TILE - 1) / TILE;
    size_t off = 0;
    auto take = [&](size_t b) { off += align256(b); };
    take(256);
    take(nt * 4);
    take(nt * 8);
    take(nt * 8);
    take(nt * 4);
    take(nt * 16);
    take(nt * 16);
    take(nt * 8);
    take((nt + 1) * 16);
    take((nt + 1) * 16);
    take((nt + 1) * 8);
    take(nt * 8);
    take((nt + 1) * 4);
    take((nt + 1) * 4);
    take(nt * 8);
    return off + 256;
}

// ---------------------------------------------------------------------------
// the monotone tile scan
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void load_items(const T *__restrict__ w, u64 n, u64 base, double v[VV])
{
    const u64 i0 = base + (u64)threadIdx.x * VV;
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
        for (int k = 0; k < VV; ++k) v[k] = (i0 + k < n) ? (double)w[i0 + k] : -1.0;  // -1: absent
    }
}

struct ScanOut {
    double key[VV];    // light: exclusive deficit prefix; heavy: inclusive excess prefix
    u32 lmask, hmask;  // class bits per item
    u32 lrank0, hrank0;  // exclusive ranks of this thread's first light/heavy in the tile
    u32 nl, nh;        // tile counts
    double totD, totE; // tile totals (upper bounds of all keys)
};

struct ScanSmem {
    double wD[NWARP], wE[NWARP];
    u32 wL[NWARP], wH[NWARP];
};

// Inclusive warp scan (Kogge-Stone) followed by a running max so the result
// is non-decreasing whatever the rounding.
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

__device__ __forceinline__ void tile_scan(const double v[VV], double avg, ScanOut &o, ScanSmem &S)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double ld[VV], le[VV];
    double sd = 0.0, se = 0.0;
    u32 lm = 0, hm = 0;
#pragma unroll
    for (int k = 0; k < VV; ++k) {
        const bool valid = v[k] >= 0.0;
        const bool light = valid && v[k] <= avg;
        const bool heavy = valid && v[k] > avg;
        ld[k] = sd;                    // exclusive
        if (light) sd = sd + (avg - v[k]);
        if (heavy) se = se + (v[k] - avg);
        le[k] = se;                    // inclusive
        lm |= (u32)light << k;
        hm |= (u32)heavy << k;
    }
    const u32 nlt = __popc(lm), nht = __popc(hm);
    // lane level
    double iD = warp_scan_mono(sd, lane), iE = warp_scan_mono(se, lane);
    double eD = shfl_up_d(iD, 1), eE = shfl_up_d(iE, 1);
    if (lane == 0) { eD = 0.0; eE = 0.0; }
    u32 iL = nlt, iH = nht;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        u32 a = __shfl_up_sync(0xffffffffu, iL, d), b = __shfl_up_sync(0xffffffffu, iH, d);
        if (lane >= d) { iL += a; iH += b; }
    }
    if (lane == 31) { S.wD[wid] = iD; S.wE[wid] = iE; S.wL[wid] = iL; S.wH[wid] = iH; }
    __syncthreads();
    // warp level (every warp recomputes the 8-entry scan: no second barrier)
    double bD = 0.0, bE = 0.0, nD = 0.0, nE = 0.0;
    u32 bL = 0, bH = 0, tL = 0, tH = 0;
    {
        double xD = lane < NWARP ? S.wD[lane] : 0.0, xE = lane < NWARP ? S.wE[lane] : 0.0;
        double sD = warp_scan_mono(xD, lane), sE = warp_scan_mono(xE, lane);
        // tile totals: the last warp-inclusive value
        o.totD = shfl_idx_d(sD, NWARP - 1);
        o.totE = shfl_idx_d(sE, NWARP - 1);
        bD = wid ? shfl_idx_d(sD, wid - 1) : 0.0;
        bE = wid ? shfl_idx_d(sE, wid - 1) : 0.0;
        nD = shfl_idx_d(sD, wid);  // upper bound for this warp's keys
        nE = shfl_idx_d(sE, wid);
        u32 xL = lane < NWARP ? S.wL[lane] : 0, xH = lane < NWARP ? S.wH[lane] : 0;
#pragma unroll
        for (int d = 1; d < NWARP; d <<= 1) {
            u32 a = __shfl_up_sync(0xffffffffu, xL, d), b = __shfl_up_sync(0xffffffffu, xH, d);
            if (lane >= d) { xL += a; xH += b; }
        }
        tL = __shfl_sync(0xffffffffu, xL, NWARP - 1);
        tH = __shfl_sync(0xffffffffu, xH, NWARP - 1);
        bL = wid ? __shfl_sync(0xffffffffu, xL, wid - 1) : 0;
        bH = wid ? __shfl_sync(0xffffffffu, xH, wid - 1) : 0;
    }
    // lane bases, clamped into the warp's range; next lane's base = upper bound
    double BD = fmin(bD + eD, nD), BE = fmin(bE + eE, nE);
    double UD = __shfl_down_sync(0xffffffffu, BD, 1), UE = __shfl_down_sync(0xffffffffu, BE, 1);
    if (lane == 31) { UD = nD; UE = nE; }
#pragma unroll
    for (int k = 0; k < VV; ++k) {
        if ((lm >> k) & 1) o.key[k] = fmin(BD + ld[k], UD);
        else if ((hm >> k) & 1) o.key[k] = fmin(BE + le[k], UE);
        else o.key[k] = 0.0;
    }
    o.lmask = lm;
    o.hmask = hm;
    o.lrank0 = bL + iL - nlt;
    o.hrank0 = bH + iH - nht;
    o.nl = tL;
    o.nh = tH;
    __syncthreads();  // S reusable
}

// ---------------------------------------------------------------------------
// 1. scan + decoupled look-back
// ---------------------------------------------------------------------------
__device__ __forceinline__ dd shfl_xor_dd(dd x, int m)
{
    return dd_make(__shfl_xor_sync(0xffffffffu, x.hi, m), __shfl_xor_sync(0xffffffffu, x.lo, m));
}

template <typename T>
__global__ void __launch_bounds__(TB) k_build_scan(const T *__restrict__ w, u64 n, double avg,
                                                   BuildWs W)
{
    __shared__ ScanSmem S;
    __shared__ unsigned int s_tile;
    __shared__ unsigned long long s_firstH;
    __shared__ dd s_exD, s_exH;
    __shared__ u64 s_exK;
    if (threadIdx.x == 0) {
        s_tile = atomicAdd(W.counter, 1u);
        s_firstH = NONE64;
    }
    __syncthreads();
    const u64 t = s_tile;
    const u64 base = t * TILE;
    double v[VV];
    load_items(w, n, base, v);
    ScanOut o;
    tile_scan(v, avg, o, S);
    if (o.hmask) {
        u64 fi = base + (u64)threadIdx.x * VV + (__ffs(o.hmask) - 1);
        atomicMin(&s_firstH, (unsigned long long)fi);
    }
    // publish the aggregate
    if (threadIdx.x == 0) {
        W.agg_d[t] = o.totD;
        W.agg_e[t] = o.totE;
        W.agg_n[t] = o.nl;
        __threadfence();
        st_release_u32(&W.status[t], t == 0 ? 2u : 1u);
        if (t == 0) {  // tile 0 is its own inclusive prefix
            W.inc_D[0] = dd_make(o.totD);
            W.inc_H[0] = dd_make(o.totE);
            W.inc_k[0] = o.nl;
            __threadfence();
            st_release_u32(&W.status[0], 2u);
        }
    }
    // warp 0 looks back
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        dd aD = dd_make(0.0), aH = dd_make(0.0);
        u64 aK = 0;
        i64 pred = (i64)t - 1;
        while (pred >= 0) {
            i64 p = pred - lane;
            u32 st = 2;
            if (p >= 0) {
                do { st = ld_acquire_u32(&W.status[p]); } while (st == 0);
            }
            unsigned inc_mask = __ballot_sync(0xffffffffu, p >= 0 && st == 2);
            int stop = inc_mask ? __ffs(inc_mask) - 1 : 32;  // first lane with an inclusive
            dd cD = dd_make(0.0), cH = dd_make(0.0);
            u64 cK = 0;
            if (p >= 0 && lane < stop) {
                cD = dd_make(W.agg_d[p]);
                cH = dd_make(W.agg_e[p]);
                cK = W.agg_n[p];
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
            if (t > 0) {
                W.inc_D[t] = dd_add_d(aD, o.totD);
                W.inc_H[t] = dd_add_d(aH, o.totE);
                W.inc_k[t] = aK + o.nl;
                __threadfence();
                st_release_u32(&W.status[t], 2u);
            }
            s_exD = aD;
            s_exH = aH;
            s_exK = aK;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        W.DLb[t] = s_exD;
        W.DHb[t] = s_exH;
        W.kL[t] = s_exK;
        W.firstH[t] = s_firstH;
        if (t == W.nt - 1) {
            W.DLb[W.nt] = dd_add_d(s_exD, o.totD);
            W.DHb[W.nt] = dd_add_d(s_exH, o.totE);
            W.kL[W.nt] = s_exK + o.nl;
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
    // T1[u] = max{t in [0, nt] : DHb[t] <= DLb[u]}
    {
        const dd x = W.DLb[u];
        u64 lo = 0, hi = nt;  // DHb[0] = 0 <= x always
        while (lo < hi) {
            u64 mid = (lo + hi + 1) >> 1;
            if (dd_le(W.DHb[mid], x)) lo = mid;
            else hi = mid - 1;
        }
        W.T1[u] = (u32)lo;
    }
    // S1[u] = max{s in [0, nt] : DLb[s] < DHb[u]}, 0 if none
    {
        const dd y = W.DHb[u];
        u64 lo = 0, hi = nt;
        if (!dd_lt(W.DLb[0], y)) {
            W.S1[u] = 0;
        } else {
            while (lo < hi) {
                u64 mid = (lo + hi + 1) >> 1;
                if (dd_lt(W.DLb[mid], y)) lo = mid;
                else hi = mid - 1;
            }
            W.S1[u] = (u32)lo;
        }
    }
    // nextH[u]: first heavy item in tiles > u
    if (u < nt) {
        auto jH = [&](u64 t) -> u64 {  // heavies before tile t
            u64 items = t * TILE < n ? t * TILE : n;
            return items - W.kL[t];
        };
        const u64 after = jH(u + 1);
        if (jH(nt) <= after) {
            W.nextH[u] = NONE64;
        } else {
            u64 lo = u + 1, hi = nt - 1;  // smallest t with jH(t+1) > after
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
// 3. tile-owner pack
// ---------------------------------------------------------------------------
template <typename T> struct PackSmem {
    double ownLk[TILE];
    double ownHk[TILE];
    double fk[TILE];
    u32 fidx[TILE];
    unsigned short ownLp[TILE];
    unsigned short ownHp[TILE];
    typename RowOf<T>::type rows[TILE];
    ScanSmem S;
    u32 nLo, nHo, nF;
    u32 r_next;
    u64 tile_sel;
};

// compact one class of tile t into (fk, fidx); lights if want_light
template <typename T>
__device__ void load_foreign(const T *__restrict__ w, u64 n, double avg, u64 t, bool want_light,
                             PackSmem<T> &P)
{
    double v[VV];
    load_items(w, n, t * TILE, v);
    ScanOut o;
    tile_scan(v, avg, o, P.S);
    u32 m = want_light ? o.lmask : o.hmask;
    u32 r = want_light ? o.lrank0 : o.hrank0;
#pragma unroll
    for (int k = 0; k < VV; ++k) {
        if ((m >> k) & 1) {
            P.fk[r] = o.key[k];
            P.fidx[r] = (u32)(threadIdx.x * VV + k);
            ++r;
        }
    }
    if (threadIdx.x == 0) P.nF = want_light ? o.nl : o.nh;
    __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(TB) k_build_pack(const T *__restrict__ w, u64 n, double avg,
                                                   BuildWs W,
                                                   typename RowOf<T>::type *__restrict__ rows_out)
{
    extern __shared__ __align__(16) unsigned char pack_smem[];
    PackSmem<T> &P = *reinterpret_cast<PackSmem<T> *>(pack_smem);
    typedef typename RowOf<T>::type RowT;
    typedef decltype(RowT::alias) AliasT;
    const u64 u = blockIdx.x;
    const u64 nt = W.nt;
    const u64 base = u * TILE;
    const u32 items = (u32)((n - base) < (u64)TILE ? (n - base) : (u64)TILE);

    // --- own tile: keys, compaction, light thresholds, heavy aliases
    double v[VV];
    load_items(w, n, base, v);
    ScanOut o;
    tile_scan(v, avg, o, P.S);
    {
        u32 rl = o.lrank0, rh = o.hrank0;
#pragma unroll
        for (int k = 0; k < VV; ++k) {
            const u32 pos = threadIdx.x * VV + k;
            if ((o.lmask >> k) & 1) {
                P.ownLk[rl] = o.key[k];
                P.ownLp[rl] = (unsigned short)pos;
                P.rows[pos].tw = (T)v[k];
                ++rl;
            } else if ((o.hmask >> k) & 1) {
                P.ownHk[rh] = o.key[k];
                P.ownHp[rh] = (unsigned short)pos;
                ++rh;
            }
        }
        if (threadIdx.x == 0) {
            P.nLo = o.nl;
            P.nHo = o.nh;
        }
    }
    __syncthreads();
    const u32 nLo = P.nLo, nHo = P.nHo;
    const dd DLu = W.DLb[u], DHu = W.DHb[u];
    // heavy aliases: next heavy in the tile, or the first heavy after it
    {
        const u64 nxt = W.nextH[u];
        for (u32 r = threadIdx.x; r < nHo; r += TB) {
            const u32 pos = P.ownHp[r];
            u64 a;
            if (r + 1 < nHo) a = base + P.ownHp[r + 1] + 1;
            else a = (nxt == NONE64) ? base + pos + 1 : nxt + 1;
            P.rows[pos].alias = (AliasT)a;
        }
    }

    // --- lights: alias = first heavy with key > light key
    {
        u64 cur = W.T1[u];  // DHb[cur] <= DLu <= every own light key
        u32 r0 = 0;
        while (r0 < nLo) {
            // t = max{t >= cur : DHb[t] <= DLu + lk[r0]}  (gallop, then bisect)
            if (threadIdx.x == 0) {
                const dd x = dd_make(P.ownLk[r0]);
                u64 lo = cur, step = 1;
                while (lo + step <= nt && dd_le(dd_sub(W.DHb[lo + step], DLu), x)) {
                    lo += step;
                    step <<= 1;
                }
                u64 hi = lo + step - 1 < nt ? lo + step - 1 : nt;
                while (lo < hi) {
                    u64 mid = (lo + hi + 1) >> 1;
                    if (dd_le(dd_sub(W.DHb[mid], DLu), x)) lo = mid;
                    else hi = mid - 1;
                }
                P.tile_sel = lo;
            }
            __syncthreads();
            const u64 t = P.tile_sel;
            if (t >= nt) {
                // no heavy key above: the remaining lights keep their own rows
                for (u32 r = r0 + threadIdx.x; r < nLo; r += TB) {
                    const u32 pos = P.ownLp[r];
                    P.rows[pos].alias = (AliasT)(base + pos + 1);
                }
                __syncthreads();
                break;
            }
            const double *hk;
            const u32 *hpos = nullptr;
            u32 nF;
            const u64 tbase = t * TILE;
            if (t == u) {
                hk = P.ownHk;
                nF = nHo;
            } else {
                load_foreign(w, n, avg, t, false, P);
                hk = P.fk;
                nF = P.nF;
                hpos = P.fidx;
            }
            const u64 after_t = W.nextH[t];
            const dd lim = dd_sub(W.DHb[t + 1], DLu);  // resolved here: lk < lim
            const dd Dlt = dd_sub(DLu, W.DHb[t]);      // heavy m <= light  <=>  hk - lk <= Dlt
            if (threadIdx.x == 0) {
                u32 lo = r0 + 1, hi = nLo;  // r0 itself is resolved here
                while (lo < hi) {
                    u32 mid = (lo + hi) >> 1;
                    if (dd_lt(dd_make(P.ownLk[mid]), lim)) lo = mid + 1;
                    else hi = mid;
                }
                P.r_next = lo;
            }
            __syncthreads();
            const u32 r1 = P.r_next;
            for (u32 r = r0 + threadIdx.x; r < r1; r += TB) {
                const double lk = P.ownLk[r];
                u32 lo = 0, hi = nF;  // first heavy m with key > light key
                while (lo < hi) {
                    u32 mid = (lo + hi) >> 1;
                    if (diff_le(hk[mid], lk, Dlt)) lo = mid + 1;
                    else hi = mid;
                }
                const u32 pos = P.ownLp[r];
                u64 a;
                if (lo < nF) a = tbase + (hpos ? hpos[lo] : P.ownHp[lo]) + 1;
                else a = (after_t == NONE64) ? base + pos + 1 : after_t + 1;
                P.rows[pos].alias = (AliasT)a;
            }
            __syncthreads();
            r0 = r1;
            cur = t + 1;
        }
    }

    // --- heavies: tw = key - DL(first light with key >= heavy key) + avg
    {
        u64 cur = W.S1[u];  // DLb[cur] < every own heavy key (or cur = 0)
        u32 r0 = 0;
        while (r0 < nHo) {
            // s = max{s >= cur : DLb[s] < DHu + hk[r0]}
            if (threadIdx.x == 0) {
                const dd y = dd_make(P.ownHk[r0]);
                u64 lo = cur, step = 1;
                while (lo + step <= nt && dd_lt(dd_sub(W.DLb[lo + step], DHu), y)) {
                    lo += step;
                    step <<= 1;
                }
                u64 hi = lo + step - 1 < nt ? lo + step - 1 : nt;
                while (lo < hi) {
                    u64 mid = (lo + hi + 1) >> 1;
                    if (dd_lt(dd_sub(W.DLb[mid], DHu), y)) lo = mid;
                    else hi = mid - 1;
                }
                P.tile_sel = lo;
            }
            __syncthreads();
            const u64 s = P.tile_sel;
            if (s >= nt) {
                // no light key >= heavy key: DL = total deficit
                const dd A = dd_sub(DHu, W.DLb[nt]);
                for (u32 r = r0 + threadIdx.x; r < nHo; r += TB) {
                    dd tw = dd_add_d(dd_add_d(A, P.ownHk[r]), avg);
                    P.rows[P.ownHp[r]].tw = tw_store<T>(tw.hi + tw.lo, avg);
                }
                __syncthreads();
                break;
            }
            const double *lk;
            u32 nF;
            if (s == u) {
                lk = P.ownLk;
                nF = nLo;
            } else {
                load_foreign(w, n, avg, s, true, P);
                lk = P.fk;
                nF = P.nF;
            }
            const dd lim = dd_sub(W.DLb[s + 1], DHu);  // resolved here: hk <= lim
            const dd Dhs = dd_sub(DHu, W.DLb[s]);      // light m < heavy  <=>  lk - hk < Dhs
            const dd Aend = dd_sub(DHu, W.DLb[s + 1]);
            if (threadIdx.x == 0) {
                u32 lo = r0 + 1, hi = nHo;
                while (lo < hi) {
                    u32 mid = (lo + hi) >> 1;
                    if (dd_le(dd_make(P.ownHk[mid]), lim)) lo = mid + 1;
                    else hi = mid;
                }
                P.r_next = lo;
            }
            __syncthreads();
            const u32 r1 = P.r_next;
            for (u32 r = r0 + threadIdx.x; r < r1; r += TB) {
                const double hk = P.ownHk[r];
                u32 lo = 0, hi = nF;  // first light m with key >= heavy key
                while (lo < hi) {
                    u32 mid = (lo + hi) >> 1;
                    if (dd_lt(two_diff_dd(lk[mid], hk), Dhs)) lo = mid + 1;
                    else hi = mid;
                }
                dd tw = (lo < nF) ? dd_add(Dhs, two_diff_dd(hk, lk[lo])) : dd_add_d(Aend, hk);
                tw = dd_add_d(tw, avg);
                P.rows[P.ownHp[r]].tw = tw_store<T>(tw.hi + tw.lo, avg);
            }
            __syncthreads();
            r0 = r1;
            cur = s + 1;
        }
    }
    __syncthreads();
    RowT *dst = rows_out + base;
    for (u32 i = threadIdx.x; i < items; i += TB) dst[i] = P.rows[i];
}

template <typename T>
int run_build(const void *wv, u64 n, double total, void *rows, void *ws, cudaStream_t st)
{
    const T *w = (const T *)wv;
    BuildWs W = carve(ws, n);
    const double avg = total / (double)n;
    AK_CUDA_TRY(cudaMemsetAsync(W.counter, 0, 256, st));
    AK_CUDA_TRY(cudaMemsetAsync(W.status, 0, W.nt * 4, st));
    k_build_scan<T><<<(unsigned)W.nt, TB, 0, st>>>(w, n, avg, W);
    AK_LAUNCH_CHECK("k_build_scan");
    k_build_coarse<<<(unsigned)((W.nt + 1 + 255) / 256), 256, 0, st>>>(W, n);
    AK_LAUNCH_CHECK("k_build_coarse");
    size_t smem = sizeof(PackSmem<T>);
    AK_CUDA_TRY(cudaFuncSetAttribute(k_build_pack<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    k_build_pack<T><<<(unsigned)W.nt, TB, smem, st>>>(w, n, avg, W,
                                                      (typename RowOf<T>::type *)rows);
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
    if (((uintptr_t)w & 15) != 0) return AK_ERR_VALUE;
    cudaStream_t st = ak_stream(stream);
    if (dtype == AK_F32) {
        if (n >= 0xFFFFFFFFull) return AK_ERR_VALUE;  // u32 aliases
        return run_build<float>(w, n, total, rows, ws, st);
    }
    if (dtype == AK_F64) return run_build<double>(w, n, total, rows, ws, st);
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
