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
//   k_prepack_block   classify (thread = P consecutive items, branch-free),
//                     CTA scan, compacted keys, the pairing decision (a
//                     warp-cooperative 32-ary search), merge, handled rows,
//                     per-block residual summary; warms L2 for the block one
//                     resident grid ahead
//   k_pp_partials / k_excl_scan_i64 / k_pp_offsets
//                     the blocks' residual offsets (chunk sums, their scan,
//                     chunk rescans)
//   k_prepack_emit    residual items (index, weight) in global item order,
//                     a warp per block
//   k_residual_remap  a residual table scattered into the final table
//                     (ak_residual_scatter; psa_plus_construct builds the
//                     residual straight into the table instead,
//                     ak_build_psa_residual in ak_build.cu)
#include "ak_common.cuh"

namespace {

struct BlockInfo {
    u32 nl, nh;     // lights / heavies of the block
    u32 kend;       // lights [0, kend) handled
    int jt;         // terminal heavy (-1: no pairing); heavies (jt, nh) forwarded
    u32 cur;        // 1: heavy jt forwarded with residual curw
    u32 nres;       // forwarded items
    u32 pL, pH;     // block offsets of the first forwarded light / heavy (len: none)
    u32 pT;         // block offset of the forwarded terminal heavy (~0: none)
    double curw;
    u64 nwritten;   // rows written by the block
};

// a T at a shared-space address
template <typename T> __device__ __forceinline__ T lds_at(u32 a);
template <> __device__ __forceinline__ float lds_at<float>(u32 a)
{
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
template <> __device__ __forceinline__ double lds_at<double>(u32 a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

template <typename T> __device__ __forceinline__ int item_class(T v, double avg)
{
    const double d = (double)v;
    return d == avg ? 2 : (d < avg ? 0 : 1);  // 0 light, 1 heavy, 2 exactly full
}

// item_class in the weight type: for floats, (double)v < avg <=> v < ru(avg)
// (no float lies strictly between rd(avg) and ru(avg)) and v == avg only
// when avg is itself a float
template <typename T> struct ClassCut {
    T a;
    bool exact;
    __device__ explicit ClassCut(double avg) : a(T(0)), exact(true)
    {
#ifdef __CUDA_ARCH__
        if constexpr (sizeof(T) == 4) {
            a = __double2float_ru(avg);
            exact = (double)a == avg;
        } else {
            a = avg;
        }
#endif
    }
    __device__ __forceinline__ int operator()(T v) const { return v < a ? 0 : (exact && v == a ? 2 : 1); }
};

// Dynamic shared memory of a block of bs items: the raw weights (staged
// once), the class-compacted keys (logical index: lights [0, nl] with DL(nl)
// at nl, heavies from nl + 1; stored at pk(x) = x + x/8 to spread the
// merge's key loads over the banks) and block offsets (lights [0, nl),
// heavies from nl).
__host__ __device__ __forceinline__ u32 pk(u32 x) { return x + (x >> 3); }
template <typename T> struct PPSmem {
    T *sw;
    double *key;
    unsigned short *item;
};
template <typename T> __device__ __forceinline__ PPSmem<T> pp_smem(unsigned char *base, u32 bs)
{
    PPSmem<T> S;
    S.sw = reinterpret_cast<T *>(base);
    S.key = reinterpret_cast<double *>(base + (((size_t)bs * sizeof(T) + 15) & ~(size_t)15));
    S.item = reinterpret_cast<unsigned short *>(S.key + pk(bs + 2) + 1);
    return S;
}

// Per block: stage the weights (bulk async copy); one classification pass in
// which each thread owns P consecutive items (16-byte shared loads) and sums
// its lights' deficits and heavies' excess; a CTA scan of those sums and
// counts (running max in the warp, warp bases summed sequentially, keys
// clamped to the next thread's base, so keys are non-decreasing); one pass
// that writes the class-compacted keys and items; then one merge path over
// the two key sequences writes every handled row (heavy first on ties:
// DH <= DL).  Round 1's count pass + strided compaction + two in-place key
// prefixes took 54% of the kernel; this front half took it from 9.4 to
// 7.6 ms at N=1e9 f32 (6.8 ms with the later changes listed above).
// threads per prepack block: each owns P consecutive items read as 16-byte
// vectors; 512 threads for f64 keep P = 8 (64 B per thread, the f32 pattern)
// minb: CTAs per SM the register budget must allow.  Shared memory holds
// f32 blocks to 3 CTAs/SM (61 KB each) and f64 blocks to 2 (77 KB); f32 at
// minb 1 gets 77 registers (3 x 256 threads still fit), f64 at minb 2 gets
// 64 (at minb 1 it took 88 and ran 1 CTA/SM: 15.9 ms against 11.0).
template <typename T> struct PPTB {
    static constexpr int v = sizeof(T) == 4 ? 256 : 512;
    static constexpr int minb = sizeof(T) == 4 ? 1 : 2;
};
template <typename T>
__global__ void __launch_bounds__(PPTB<T>::v, PPTB<T>::minb) k_prepack_block(const T *__restrict__ w, u64 n, double avg,
                                                         u32 bs, u32 thr, u32 pf_ahead,
                                                         typename RowOf<T>::type *__restrict__ rows,
                                                         BlockInfo *__restrict__ info)
{
    constexpr int TBT = PPTB<T>::v;
    typedef typename RowOf<T>::type RowT;
    typedef decltype(RowT::tw) TwT;
    typedef decltype(RowT::alias) AliasT;
    extern __shared__ __align__(16) unsigned char pp_raw[];
    const PPSmem<T> S = pp_smem<T>(pp_raw, bs);
    __shared__ u64 s_written;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u64 b0 = (u64)blockIdx.x * bs;
    const u32 len = (u32)(b0 + bs <= n ? bs : n - b0);
    // stage the block's weights: one bulk async copy (TMA) when aligned
    __shared__ __align__(8) u64 bar;
    const T *src = w + b0;
    const u32 bytes = len * (u32)sizeof(T);
    const bool bulk = ((((uintptr_t)src) | bytes) & 15) == 0;
    if (threadIdx.x == 0) {
        s_written = 0;
        if (bulk) {
            mbar_init(&bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_expect_tx(&bar, bytes);
            bulk_g2s(S.sw, src, bytes, &bar);
        }
        // warm L2 with the weights of the block that starts about one
        // resident grid later, so its own bulk copy hits L2
        const u64 pb = (u64)blockIdx.x + pf_ahead;
        if (pf_ahead && (pb + 1) * bs <= n) {
            const T *pf = w + pb * bs;
            if ((((uintptr_t)pf) & 15) == 0 && ((bs * (u32)sizeof(T)) & 15) == 0)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"(bs * (u32)sizeof(T)) : "memory");
        }
    }
    if (bulk) {
        __syncthreads();  // the barrier is initialised before anyone waits on it
        mbar_wait(&bar, 0);
    } else {
        for (u32 i = threadIdx.x; i < len; i += TBT) S.sw[i] = src[i];
        __syncthreads();
    }
    // One classification pass: thread t owns the P consecutive items
    // [t P, t P + P) (P a multiple of 4, so its values are 16-byte loads from
    // the staged block).  Exactly-full items are final at once; lights and
    // heavies are counted and their deficit / excess summed in item order.
    const ClassCut<T> cls(avg);
    const u32 P = ((len + TBT - 1) / TBT + 3) & ~3u;
    const u32 i0 = threadIdx.x * P;
    u64 lmask = 0, hmask = 0;
    u32 cw = 0, tl = 0, th = 0;
    double sl = 0.0, sh = 0.0;
    for (u32 q = 0; q < P; q += 4) {
        T v4[4];
        const u32 i = i0 + q;
        if (i + 4 <= len) {
            if (sizeof(T) == 4) {
                const float4 f = *reinterpret_cast<const float4 *>(S.sw + i);
                v4[0] = (T)f.x; v4[1] = (T)f.y; v4[2] = (T)f.z; v4[3] = (T)f.w;
            } else {
                const double2 d0 = *reinterpret_cast<const double2 *>(S.sw + i);
                const double2 d1 = *reinterpret_cast<const double2 *>(S.sw + i + 2);
                v4[0] = (T)d0.x; v4[1] = (T)d0.y; v4[2] = (T)d1.x; v4[3] = (T)d1.y;
            }
        } else {
#pragma unroll
            for (int z = 0; z < 4; ++z) v4[z] = i + z < len ? S.sw[i + z] : (T)0;
        }
        // branch-free (classes are random per lane): adding an exact 0.0
        // leaves a sum unchanged, so the sums equal the per-class chains
        u32 l4 = 0, h4 = 0;
#pragma unroll
        for (int z = 0; z < 4; ++z) {
            const bool in = i + z < len;
            const int c = cls(v4[z]);
            const bool L = in && c == 0, H = in && c == 1;
            const double x = (double)v4[z] - avg;
            sl = sl - (L ? x : 0.0);  // avg - w == -(w - avg) exactly
            sh = sh + (H ? x : 0.0);
            l4 |= (u32)L << z;
            h4 |= (u32)H << z;
            if (in && c == 2) {  // exactly full: final at once (rare)
                RowT row;
                row.tw = (TwT)v4[z];
                row.alias = (AliasT)(b0 + i + z + 1);
                rows[b0 + i + z] = row;
                ++cw;
            }
        }
        lmask |= (u64)l4 << q;
        hmask |= (u64)h4 << q;
    }
    tl = __popcll(lmask);
    th = __popcll(hmask);
    if (cw) atomicAdd((unsigned long long *)&s_written, (unsigned long long)cw);
    // CTA scan of (sl, sh, tl, th): warp Kogge-Stone with a running max on the
    // sums (non-decreasing lane bases), warp bases summed sequentially, so a
    // thread's last key never passes the next thread's base: keys are
    // non-decreasing in item order (the merge needs sorted keys)
    __shared__ double s_wl[TBT / 32 + 1], s_wh[TBT / 32 + 1];
    __shared__ u32 s_cl[TBT / 32 + 1], s_ch[TBT / 32 + 1];
    double il = sl, ih = sh;
    u32 cl = tl, ch = th;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double yl = __shfl_up_sync(0xffffffffu, il, d), yh = __shfl_up_sync(0xffffffffu, ih, d);
        const u32 zl = __shfl_up_sync(0xffffffffu, cl, d), zh = __shfl_up_sync(0xffffffffu, ch, d);
        if (lane >= d) {
            il = il + yl;
            ih = ih + yh;
            cl += zl;
            ch += zh;
        }
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double yl = __shfl_up_sync(0xffffffffu, il, d), yh = __shfl_up_sync(0xffffffffu, ih, d);
        if (lane >= d) {
            il = il > yl ? il : yl;
            ih = ih > yh ? ih : yh;
        }
    }
    if (lane == 31) {
        s_wl[wid] = il;
        s_wh[wid] = ih;
        s_cl[wid] = cl;
        s_ch[wid] = ch;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // sequential warp bases (exclusive), totals at [NW]
        double al = 0.0, ah = 0.0;
        u32 bl = 0, bh = 0;
        for (int k = 0; k < TBT / 32; ++k) {
            const double xl = s_wl[k], xh = s_wh[k];
            const u32 yl = s_cl[k], yh = s_ch[k];
            s_wl[k] = al;
            s_wh[k] = ah;
            s_cl[k] = bl;
            s_ch[k] = bh;
            al = al + xl;
            ah = ah + xh;
            bl += yl;
            bh += yh;
        }
        s_wl[TBT / 32] = al;
        s_wh[TBT / 32] = ah;
        s_cl[TBT / 32] = bl;
        s_ch[TBT / 32] = bh;
    }
    __syncthreads();
    const u32 nl = s_cl[TBT / 32], nh = s_ch[TBT / 32];
    const double DLtot = s_wl[TBT / 32];
    {
        const double el = __shfl_up_sync(0xffffffffu, il, 1), eh = __shfl_up_sync(0xffffffffu, ih, 1);
        const double Wl = s_wl[wid], Wh = s_wh[wid];
        // this thread's bases and the next thread's (the clamp)
        const double BL = Wl + (lane ? el : 0.0), BH = Wh + (lane ? eh : 0.0);
        const double nBL = lane < 31 ? Wl + il : s_wl[wid + 1];
        const double nBH = lane < 31 ? Wh + ih : s_wh[wid + 1];
        u32 rl = s_cl[wid] + cl - tl, rh = s_ch[wid] + ch - th;
        double pl = 0.0, ph = 0.0;
        for (u32 q = 0; q < P; q += 4) {
            if (!(((lmask | hmask) >> q) & 0xFull)) continue;
            const u32 i = i0 + q;
            T v4[4];
            if (i + 4 <= len) {
                if (sizeof(T) == 4) {
                    const float4 f = *reinterpret_cast<const float4 *>(S.sw + i);
                    v4[0] = (T)f.x; v4[1] = (T)f.y; v4[2] = (T)f.z; v4[3] = (T)f.w;
                } else {
                    const double2 d0 = *reinterpret_cast<const double2 *>(S.sw + i);
                    const double2 d1 = *reinterpret_cast<const double2 *>(S.sw + i + 2);
                    v4[0] = (T)d0.x; v4[1] = (T)d0.y; v4[2] = (T)d1.x; v4[3] = (T)d1.y;
                }
            } else {
#pragma unroll
                for (int z = 0; z < 4; ++z) v4[z] = i + z < len ? S.sw[i + z] : (T)0;
            }
            const u32 l4 = (u32)(lmask >> q) & 0xFu, h4 = (u32)(hmask >> q) & 0xFu;
#pragma unroll
            for (int z = 0; z < 4; ++z) {
                // branch-free, as the classification pass
                const bool isl = (l4 >> z) & 1, ish = (h4 >> z) & 1;
                const double x = (double)v4[z] - avg;
                ph = ph + (ish ? x : 0.0);
                const double k = isl ? BL + pl : BH + ph;
                const double cap = isl ? nBL : nBH;
                if (isl || ish) {
                    S.key[pk(isl ? rl : nl + 1 + rh)] = k < cap ? k : cap;
                    S.item[isl ? rl : nl + rh] = (unsigned short)(i + z);
                }
                pl = pl - (isl ? x : 0.0);
                rl += isl;
                rh += ish;
            }
        }
    }
    if (threadIdx.x == 0) S.key[pk(nl)] = DLtot;
    __syncthreads();
    const bool pair = nl >= thr && nh >= thr;
    u32 kend = 0, cur = 0;
    int jt = -1;
    double curw = 0.0;
    u64 nwritten = 0;
    if (pair) {
        // keys: DL exclusive over lights (DL(nl) = the whole deficit), DH inclusive
        const double *key = S.key;
        auto DL = [&](u32 k) { return key[pk(k)]; };           // [0, nl]
        auto DH = [&](u32 j) { return key[pk(nl + 1 + j)]; };  // [0, nh)
        // lights absorbed before the sweep stops: #lights with DL < DH(j)
        // first index in [0, cnt) satisfying a monotone (false .. true)
        // predicate, cnt if none: a warp-cooperative 32-ary search (32 probes
        // and a ballot per step, 3 steps for a 4096-item block), run by every
        // warp on the same keys -- the binary search's answer without its 12
        // dependent shared loads per thread
        auto warp_first = [&](u32 cnt, auto pred) {
            u32 lo = 0, hi = cnt;  // answer in [lo, hi]
            while (hi - lo >= 32) {  // the last step's 32 probes then cover [lo, hi]
                const u32 step = (hi - lo + 31) / 32;
                const u32 q = lo + (lane + 1) * step - 1;
                const unsigned m = __ballot_sync(0xffffffffu, q >= hi || pred(q));
                if (!m) { lo = hi; break; }
                const u32 f = (u32)__ffs(m) - 1;
                const u32 qf = lo + (f + 1) * step - 1;
                lo += f * step;
                hi = qf < hi ? qf : hi;
            }
            const u32 q = lo + lane;
            const unsigned m = __ballot_sync(0xffffffffu, q >= hi || pred(q));
            return lo + (u32)__ffs(m) - 1;
        };
        auto lights_below = [&](double x) {  // first k with DL(k) >= x
            return warp_first(nl, [&](u32 k) { return DL(k) >= x; });
        };
        auto heavies_upto = [&](double x) {  // first j with DH(j) > x
            return warp_first(nh, [&](u32 j) { return DH(j) > x; });
        };
        if (DH(nh - 1) <= DLtot) {
            jt = (int)nh - 1;
            kend = lights_below(DH(nh - 1));
        } else {
            kend = nl;
            jt = (int)heavies_upto(DLtot);
        }
        const double wt_end = (DH(jt) - DL(kend)) + avg;
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
                auto wl = [&](u32 k) { return (double)S.sw[S.item[k]]; };
                auto wh = [&](u32 j) { return (double)S.sw[S.item[nl + j]]; };
                u32 k = 0;
                int j = 0;
                double wc = wh(0);
                while (true) {
                    if (wc > avg) {
                        if (k == nl) break;
                        const u64 it = b0 + S.item[k];
                        RowT row;
                        row.tw = (TwT)S.sw[S.item[k]];
                        row.alias = (AliasT)(b0 + S.item[nl + j] + 1);
                        rows[it] = row;
                        wc += wl(k) - avg;
                        ++k;
                    } else {
                        if ((u32)j + 1 >= nh) break;
                        RowT row;
                        row.tw = tw_store<T>(wc, avg);
                        row.alias = (AliasT)(b0 + S.item[nl + j + 1] + 1);
                        rows[b0 + S.item[nl + j]] = row;
                        wc += wh(j + 1) - avg;
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
        } else {
            // merge path over lights [0, nl) and heavies [0, nh): thread t
            // takes merged positions [t per, (t + 1) per); a taken light k
            // (k < kend) aliases the next heavy, a taken heavy j (j < jt)
            // closes against the lights taken before it
            const u32 total = nl + nh;
            const u32 per = (total + TBT - 1) / TBT;
            const u32 d0 = threadIdx.x * per;
            if (d0 < total) {
                const u32 lo0 = d0 > nh ? d0 - nh : 0, hi0 = d0 < nl ? d0 : nl;
                u32 lo = lo0, hi = hi0;  // greatest i with light i-1 before heavy d0-i
                while (lo < hi) {
                    const u32 m = (lo + hi + 1) >> 1;
                    if (d0 - m >= nh || DL(m - 1) < DH(d0 - m)) lo = m;
                    else hi = m - 1;
                }
                u32 k = lo, j = d0 - lo;
                const u32 steps = d0 + per < total ? per : total - d0;
                // loop invariants kept in registers: the staged weights'
                // shared-space address (opaque to the compiler, which would
                // otherwise re-derive the dynamic shared base every step) and
                // the block's first row
                u32 sw_sa = (u32)__cvta_generic_to_shared(S.sw);
                asm("" : "+r"(sw_sa));
                RowT *const rb = rows + b0;
                // one row per step on a single (branch-free) path: a taken
                // heavy j closes against DL(k), a taken light k aliases heavy j
                double dh = j < nh ? DH(j) : 0.0, dl = DL(k < nl ? k : nl);
                for (u32 d = 0; d < steps; ++d) {
                    const bool take_h = j < nh && (k >= nl || dh <= dl);
                    const u32 self = take_h ? nl + j : k;
                    const u32 it = S.item[self < nl + nh ? self : 0];
                    const u32 al = S.item[take_h ? (nl + j + 1 < nl + nh ? nl + j + 1 : nl + j) : nl + (j < nh ? j : 0)];
                    const bool wr = take_h ? j < (u32)jt : k < kend;
                    // only a closing heavy's value is <= avg (+ rounding); any other
                    // step passes avg, as tw_store walks values above avg down
                    const TwT hv = tw_store<T>(take_h && wr ? (dh - dl) + avg : avg, avg);
                    RowT row;
                    row.tw = take_h ? hv : (TwT)lds_at<T>(sw_sa + it * (u32)sizeof(T));
                    row.alias = (AliasT)(b0 + al + 1);
                    if (wr) rb[it] = row;
                    if (take_h) {
                        ++j;
                        dh = j < nh ? DH(j) : 0.0;
                    } else {
                        ++k;
                        dl = DL(k < nl ? k : nl);
                    }
                }
            }
            if (threadIdx.x == 0 && !cur) {
                const u64 it = b0 + S.item[nl + jt];
                RowT row;
                row.tw = tw_store<T>(wt_end, avg);
                row.alias = (AliasT)(it + 1);
                rows[it] = row;
            }
        }
        nwritten = (u64)kend + (u64)jt + (cur ? 0 : 1);
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
        // forwarded items: the lights from rank kend and the heavies from
        // rank jt + 1 (jt itself when it carries a residual), in item order
        const u32 hf = (u32)(jt + 1) - (pair && cur ? 1u : 0u);
        bi.pL = kend < nl ? S.item[kend] : len;
        bi.pH = hf < nh ? S.item[nl + hf] : len;
        bi.pT = pair && cur ? S.item[nl + jt] : 0xFFFFFFFFu;
        info[blockIdx.x] = bi;
    }
}

// Residual items of each block in item order at res_off[block] + ...: the
// lights at block offsets >= pL and the heavies at offsets >= pH (the
// terminal heavy at pT with its residual weight), i.e. only the block's tail
// from min(pL, pH) is visited.  One warp per block (PE_WARPS blocks per CTA)
// with 128 items in flight per step: the pass is latency-bound (info ->
// offset -> tail loads), and a CTA per block with barriers between 256-item
// steps left most of that latency exposed.
constexpr int PE_WARPS = 8;
template <typename T>
__global__ void __launch_bounds__(PE_WARPS * 32) k_prepack_emit(const T *__restrict__ w, u64 n, double avg,
                                                             u32 bs, u64 nb,
                                                             const BlockInfo *__restrict__ info,
                                                             const i64 *__restrict__ res_off,
                                                             i64 *__restrict__ res_idx,
                                                             double *__restrict__ res_w)
{
    const int lane = threadIdx.x & 31;
    const u64 b = (u64)blockIdx.x * PE_WARPS + (threadIdx.x >> 5);
    if (b >= nb) return;
    const BlockInfo bi = info[b];
    if (bi.nres == 0) return;
    const u64 b0 = b * bs;
    const u32 len = (u32)(b0 + bs <= n ? bs : n - b0);
    const u32 lt = (1u << lane) - 1u;
    i64 pos = res_off[b];
    for (u32 base = bi.pL < bi.pH ? bi.pL : bi.pH; base < len; base += 128) {
        T v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const u32 i = base + u * 32 + lane;
            v[u] = i < len ? w[b0 + i] : T(0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const u32 i = base + u * 32 + lane;
            bool f = false;
            if (i < len) {
                const int c = item_class(v[u], avg);
                f = (c == 0 && i >= bi.pL) || (c == 1 && i >= bi.pH);
            }
            const unsigned fb = __ballot_sync(0xffffffffu, f);
            if (f) {
                const i64 q = pos + __popc(fb & lt);
                res_idx[q] = (i64)(b0 + i + 1);
                res_w[q] = i == bi.pT ? bi.curw : (double)v[u];
            }
            pos += __popc(fb);
        }
    }
}

// Block-count scan, multi-CTA: each CTA of PPS_T threads owns PPS_CHUNK
// consecutive blocks.  k_pp_partials sums a chunk's residual counts (and adds
// its written pairs into *nw, one atomic per CTA); k_excl_scan_i64 scans the
// chunk sums; k_pp_offsets rescans each chunk from its base.
constexpr int PPS_T = 256, PPS_PER = 8, PPS_CHUNK = PPS_T * PPS_PER;

__device__ __forceinline__ i64 pps_block_sum(i64 v, i64 *ws)
{
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    i64 t = 0;
#pragma unroll
    for (int k = 0; k < PPS_T / 32; ++k) t += ws[k];
    return t;
}

__global__ void __launch_bounds__(PPS_T) k_pp_partials(const BlockInfo *__restrict__ info, u64 nb,
                                                       i64 *__restrict__ part,
                                                       unsigned long long *nw)
{
    __shared__ i64 ws0[PPS_T / 32], ws1[PPS_T / 32];
    const u64 c0 = (u64)blockIdx.x * PPS_CHUNK;
    i64 r = 0, w = 0;
#pragma unroll
    for (int k = 0; k < PPS_PER; ++k) {
        const u64 b = c0 + (u64)k * PPS_T + threadIdx.x;
        if (b < nb) {
            r += info[b].nres;
            w += info[b].nwritten;
        }
    }
    r = pps_block_sum(r, ws0);
    w = pps_block_sum(w, ws1);
    if (threadIdx.x == 0) {
        part[blockIdx.x] = r;
        if (w) atomicAdd(nw, (unsigned long long)w);
    }
}

__global__ void __launch_bounds__(PPS_T) k_pp_offsets(const BlockInfo *__restrict__ info, u64 nb,
                                                      const i64 *__restrict__ part_off,
                                                      i64 *__restrict__ off)
{
    __shared__ i64 ws[PPS_T / 32];
    const u64 b0 = (u64)blockIdx.x * PPS_CHUNK + (u64)threadIdx.x * PPS_PER;
    i64 v[PPS_PER], s = 0;
#pragma unroll
    for (int k = 0; k < PPS_PER; ++k) {
        v[k] = b0 + k < nb ? info[b0 + k].nres : 0;
        s += v[k];
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    i64 inc = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const i64 y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
    }
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    i64 ex = part_off[blockIdx.x] + inc - s;
    for (int k = 0; k < wid; ++k) ex += ws[k];
#pragma unroll
    for (int k = 0; k < PPS_PER; ++k) {
        if (b0 + k < nb) off[b0 + k] = ex;
        ex += v[k];
    }
}

// exclusive scan of chunk sums (single CTA, sequential chunks; a few hundred
// values for N=1e9)
__global__ void k_excl_scan_i64(const i64 *cnt, u64 nb, i64 *off, i64 *total)
{
    __shared__ i64 carry;
    __shared__ i64 ws[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (u64 base = 0; base < nb; base += blockDim.x) {
        const u64 b = base + threadIdx.x;
        const i64 v = b < nb ? cnt[b] : 0;
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

// residual table (f64 rows over residual positions) -> final rows; with
// `written` non-null, also counts the rows it writes with a nonzero alias
// (a written bucket) — the residual half of PSA+'s every-bucket-written check
template <typename RowOut>
__global__ void k_residual_remap(const RowF64 *__restrict__ rt, const i64 *__restrict__ res_idx,
                                 u64 nres, double avg, RowOut *__restrict__ rows,
                                 unsigned long long *written)
{
    typedef decltype(RowOut::tw) TwT;
    typedef decltype(RowOut::alias) AliasT;
    const u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = false;
    if (r < nres) {
        const RowF64 x = rt[r];
        RowOut o;
        o.tw = tw_store<TwT>(x.tw, avg);
        o.alias = x.alias ? (AliasT)res_idx[x.alias - 1] : (AliasT)0;
        ok = o.alias != 0;
        rows[res_idx[r] - 1] = o;
    }
    if (written) {  // one atomic per block (every thread reaches the count)
        const int c = __syncthreads_count(ok);
        if (threadIdx.x == 0 && c) atomicAdd(written, (unsigned long long)c);
    }
}

size_t pp_smem_bytes(u32 bs, size_t wb) { return (((size_t)bs * wb + 15) & ~(size_t)15) + (size_t)(pk(bs + 2) + 1) * 8 + (size_t)bs * 2 + 16; }

inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

// blocks resident at once (SMs x CTAs per SM): how far ahead a block warms
// L2 for its successor on the same SM slot (queried once, ak_host.cpp)
u32 pp_prefetch_distance(const void *kern, int threads, size_t smem)
{
    return ak_resident_ctas(kern, threads, smem);
}

}  // namespace

extern "C" int ak_build_psa_avg(const void *w, int dtype, uint64_t n, double avg, void *rows,
                                void *ws, size_t ws_bytes, void *stream);

extern "C" {

size_t ak_prepack_workspace_bytes(uint64_t n, uint32_t block_size)
{
    const u64 nb = block_size ? (n + block_size - 1) / block_size : 0;
    return al256(nb * sizeof(BlockInfo)) + 2 * al256((nb + 1) * 8) + 256;
}

int ak_greedy_prepack(const void *w, int dtype, uint64_t n, double avg, uint32_t block_size,
                      uint32_t threshold, void *rows, int64_t *res_idx, double *res_w,
                      uint64_t *nres_out, uint64_t *nwritten_out, void *ws, size_t ws_bytes,
                      void *stream)
{
    return ak_greedy_prepack_ex(w, dtype, n, avg, block_size, threshold, 1, rows, res_idx, res_w,
                                nres_out, nwritten_out, ws, ws_bytes, stream);
}

int ak_greedy_prepack_ex(const void *w, int dtype, uint64_t n, double avg, uint32_t block_size,
                         uint32_t threshold, int clear_rows, void *rows, int64_t *res_idx,
                         double *res_w, uint64_t *nres_out, uint64_t *nwritten_out, void *ws,
                         size_t ws_bytes, void *stream)
{
    if (n == 0) return AK_ERR_EMPTY_INPUT;
    if (block_size < 2 || threshold < 1) return AK_ERR_VALUE;
    const size_t smem = pp_smem_bytes(block_size, dtype == AK_F32 ? 4 : 8);
    if (smem > 220 * 1024 || block_size > 11000) return AK_ERR_VALUE;  // block does not fit
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
    if (clear_rows) AK_CUDA_TRY(cudaMemsetAsync(rows, 0, n * rb, st));
    {
        const int rc0 = ak_fill_small(nw, 0, 8, st);
        if (rc0 != AK_OK) return rc0;
    }
    if (dtype == AK_F32) {
        AK_SMEM_ATTR(k_prepack_block<float>, (int)smem);
        k_prepack_block<float><<<(unsigned)nb, PPTB<float>::v, smem, st>>>(
            (const float *)w, n, avg, block_size, threshold,
            pp_prefetch_distance((const void *)k_prepack_block<float>, PPTB<float>::v, smem), (RowF32 *)rows, info);
    } else if (dtype == AK_F64) {
        AK_SMEM_ATTR(k_prepack_block<double>, (int)smem);
        k_prepack_block<double><<<(unsigned)nb, PPTB<double>::v, smem, st>>>(
            (const double *)w, n, avg, block_size, threshold,
            pp_prefetch_distance((const void *)k_prepack_block<double>, PPTB<double>::v, smem), (RowF64 *)rows, info);
    } else {
        return AK_ERR_VALUE;
    }
    AK_LAUNCH_CHECK("k_prepack_block");
    {
        // chunk sums in cnt[0, G), their exclusive scan in cnt[G, 2G)
        // (2G <= nb + 1 slots for every nb >= 1)
        const u64 G = (nb + PPS_CHUNK - 1) / PPS_CHUNK;
        k_pp_partials<<<(unsigned)G, PPS_T, 0, st>>>(info, nb, cnt, nw);
        AK_LAUNCH_CHECK("k_pp_partials");
        k_excl_scan_i64<<<1, 1024, 0, st>>>(cnt, G, cnt + G, tot);
        AK_LAUNCH_CHECK("k_excl_scan_i64");
        k_pp_offsets<<<(unsigned)G, PPS_T, 0, st>>>(info, nb, cnt + G, off);
        AK_LAUNCH_CHECK("k_pp_offsets");
    }
    {
        const unsigned g = (unsigned)((nb + PE_WARPS - 1) / PE_WARPS);
        if (dtype == AK_F32)
            k_prepack_emit<float><<<g, PE_WARPS * 32, 0, st>>>((const float *)w, n, avg, block_size, nb,
                                                              info, off, res_idx, res_w);
        else
            k_prepack_emit<double><<<g, PE_WARPS * 32, 0, st>>>((const double *)w, n, avg, block_size, nb,
                                                               info, off, res_idx, res_w);
    }
    AK_LAUNCH_CHECK("k_prepack_emit");
    i64 nres = 0;
    unsigned long long nwr = 0;
    {
        const int rc = ak_readback(st, &nres, tot, 8, &nwr, nw, 8);
        if (rc != AK_OK) return rc;
    }
    *nres_out = (u64)nres;
    *nwritten_out = (u64)nwr;
    return AK_OK;
}

static int residual_scatter(const void *res_rows, const int64_t *res_idx, uint64_t nres, double avg,
                            int dtype, void *rows, unsigned long long *written, cudaStream_t st)
{
    const unsigned g = (unsigned)((nres + 255) / 256);
    if (dtype == AK_F32)
        k_residual_remap<RowF32><<<g, 256, 0, st>>>((const RowF64 *)res_rows, res_idx, nres, avg,
                                                     (RowF32 *)rows, written);
    else if (dtype == AK_F64)
        k_residual_remap<RowF64><<<g, 256, 0, st>>>((const RowF64 *)res_rows, res_idx, nres, avg,
                                                     (RowF64 *)rows, written);
    else
        return AK_ERR_VALUE;
    AK_LAUNCH_CHECK("k_residual_remap");
    return AK_OK;
}

int ak_residual_scatter(const void *res_rows, const int64_t *res_idx, uint64_t nres, double avg,
                        int dtype, void *rows, void *stream)
{
    if (nres == 0) return AK_OK;
    return residual_scatter(res_rows, res_idx, nres, avg, dtype, rows, nullptr, ak_stream(stream));
}

int ak_residual_scatter_count(const void *res_rows, const int64_t *res_idx, uint64_t nres,
                              double avg, int dtype, void *rows, uint64_t *written, void *stream)
{
    *written = 0;
    if (nres == 0) return AK_OK;
    cudaStream_t st = ak_stream(stream);
    unsigned long long *c = (unsigned long long *)ak_stream_scratch(st);
    if (!c) return AK_ERR_CUDA;
    int rc = ak_fill_small(c, 0, 8, st);
    if (rc == AK_OK) rc = residual_scatter(res_rows, res_idx, nres, avg, dtype, rows, c, st);
    unsigned long long h = 0;
    if (rc == AK_OK) rc = ak_readback(st, &h, c, sizeof(h));
    *written = h;
    return rc;
}

}  // extern "C"
