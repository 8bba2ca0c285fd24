// Row-stripe machinery shared by the batch and wavefront kernels.
//
// Layout (device memory), the reference's PreparedSeries (core.py:177-234):
//   V   (rows, D) row-major, row 0 of each series the zero vector   [type R]
//                 -- +inf in the DP kernels' copy (see COL0_BY_INF)
//   Tm  (rows)    timestamps, row 0 = 0                              [type R]
//   Del (rows)    deletion costs, row 0 = +inf                        [type Z]
// Series lists are packed back to back; series k occupies prepared rows
// [poff[k], poff[k+1]) with poff[k] = off[k] + k.
//
// Precision modes: fp64  R = Z = double   (bit-identical to the reference)
//                  fp32  R = float, Z = float  (short series: batch)
//                  fp32  R = float, Z = double (long pairs: fp64 accumulator)
//
// Execution model. A warp owns 32*K consecutive DP rows of series A: lane t
// holds rows r0..r0+K-1 in registers. The warp streams the columns of the B
// side (one or many prepared series back to back, each with its virtual column
// 0) with a one-step skew per lane: at step s lane t computes column j = s - t
// for its K rows, top to bottom. The cell above its first row comes from lane
// t-1 by warp shuffle (computed one step earlier); lane 0 gets it from the
// row-0 boundary, the previous warp (shared-memory ring) or the previous CTA
// (flag-synchronised global buffer). Per row the lane keeps z(r, j-1),
// d(r, j-1) and t_a(r) - t_b(j-1), so interior_cost's d_prev and second
// t_gap term (_kernels.py:70-71) are reused bit-identically instead of being
// recomputed. Column data is staged per warp into a 128-column shared-memory
// ring by cp.async, two 32-column blocks ahead of use.
#pragma once

#include "twb_device.cuh"

namespace twb {

template <typename R, typename Z>
struct PreparedT {
    const R* v;    // (rows, D)
    const R* t;    // (rows)
    const Z* del;  // (rows)
    // D == 0 (runtime dimension): the same values dim-major, element k of
    // prepared row r at vt[k * ldt + r] (read column-wise by the DP kernels)
    const R* vt = nullptr;
    int64_t ldt = 0;
};

constexpr int RING_COLS = 128;  // per-warp column staging ring (4 blocks of 32)

// Per-warp column staging ring of NC columns (power of 2, multiple of 32).
// D == 0 (runtime dimension): values are not staged (read from the dim-major
// copy), only times and deletion costs.
template <int D, typename R, typename Z, int NC = RING_COLS>
struct ColRing {
    static constexpr int N = NC;
    R v[D > 0 ? NC * D : 1];
    R t[NC];
    Z del[NC];
};

template <typename X>
__device__ __forceinline__ void cp_async_elem(X* smem, const X* gmem, bool valid) {
    if constexpr (sizeof(X) == 8) cp_async8(smem, gmem, valid);
    else cp_async4(smem, gmem, valid);
}

// Stage 32-column block `blk` (stream columns 32*blk .. 32*blk+31, i.e. global
// prepared rows c0 + ...) into its ring slot. Columns >= ncols are zero-filled.
template <int D, typename R, typename Z, int NC>
__device__ __forceinline__ void stage_block(ColRing<D, R, Z, NC>& ring, const PreparedT<R, Z>& B,
                                            int64_t c0, int64_t ncols, int64_t blk, int lane) {
    const int64_t j = blk * 32 + lane;
    const bool ok = j < ncols;
    const int64_t g = c0 + (ok ? j : 0);
    const int slot = (int)(j & (NC - 1));
    if constexpr (D > 0) {
        const int base = (int)((blk * 32) & (NC - 1)) * D;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const int e = lane + 32 * k;  // element of the block's 32*D words
            const int64_t gj = blk * 32 + e / D;
            const bool okk = gj < ncols;
            cp_async_elem(&ring.v[base + e], B.v + (c0 + (okk ? gj : 0)) * D + (e % D), okk);
        }
    }
    cp_async_elem(&ring.t[slot], B.t + g, ok);
    cp_async_elem(&ring.del[slot], B.del + g, ok);
    cp_async_commit();
}

// fp32 lp distance (fp32 mode only; tolerance, not bit parity).
template <int D, int P>
__device__ __forceinline__ float lp_dist_f(const float (&x)[D], const float (&y)[D], int p) {
    if constexpr (D == 1) {
        return fabsf(x[0] - y[0]);
    } else {
        const int pp = P ? P : p;
        if (pp == 1) {
            float acc = fabsf(x[0] - y[0]);
#pragma unroll
            for (int k = 1; k < D; ++k) acc += fabsf(x[k] - y[k]);
            return acc;
        }
        if (pp == 2) {
            float d0 = x[0] - y[0];
            float acc = d0 * d0;
#pragma unroll
            for (int k = 1; k < D; ++k) {
                float dk = x[k] - y[k];
                acc = acc + dk * dk;
            }
            float r;
            asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(acc));
            return r;
        }
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < D; ++k) acc += __powf(fabsf(x[k] - y[k]), (float)pp);
        return __powf(acc, 1.0f / (float)pp);
    }
}

template <int D, int P, typename R>
__device__ __forceinline__ R dist(const R (&x)[D], const R (&y)[D], int p) {
    if constexpr (sizeof(R) == 8) return lp_dist<D, P>(x, y, p);
    else return lp_dist_f<D, P>(x, y, p);
}

template <typename Z>
__device__ __forceinline__ Z zinf() {
    if constexpr (sizeof(Z) == 8) return dinf();
    else return __int_as_float(0x7f800000);
}

// Sum of squared differences, the p == 2 accumulator of lp_dist
// (_kernels.py:39-44: acc = 0.0; acc += diff*diff, sequentially).
template <int D>
__device__ __forceinline__ double sumsq(const double (&x)[D], const double (&y)[D]) {
    double d0 = x[0] - y[0];
    double acc = __dmul_rn(d0, d0);
#pragma unroll
    for (int k = 1; k < D; ++k) {
        double dk = x[k] - y[k];
        acc = __dadd_rn(acc, __dmul_rn(dk, dk));
    }
    return acc;
}

// fp32 square root: sqrt.approx (MUFU.SQRT). FTZ on the proven-safe path
// (the host flags nonzero |x| < 2^-30 as unsafe, so a nonzero sum of squares
// is never denormal there); the exact-NaN path keeps denormal handling.
template <bool FTZ>
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    if constexpr (FTZ) asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    else asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Per-lane DP state for K rows.
//
// fp64 (bit-exact): per row the lane keeps d(r, j-1) and t_a(r) - t_b(j-1),
// the d_prev and second t-gap term of interior_cost for (r+1, j), and sums in
// the reference's association.
// fp32 modes (tolerance 1e-5): per row it keeps the edge cost
// c(r, j-1) = d(r, j-1) + nu*|t_a(r) - t_b(j-1)|, so the match candidate is
// z_diag + (c(r, j) + c(r-1, j-1)) -- the same terms regrouped, 3 adds per cell
// instead of 5, and sums of squares use FMA.
//
// d_prev (fp64) / c (fp32) of the lane's first row is the value the lane above
// computed for its last row two steps earlier; it arrives by shuffle (or
// through the warp/CTA boundary rings) instead of being recomputed. Same value,
// same bits.
// SPLIT_SQRT (fp64, d >= 2, degree 2): the K square roots of a column run as
// straight-line sqrt_fast (interleavable), with one rare fix-up branch per
// column for out-of-range arguments (twb_device.cuh).
// COL0_BY_INF (every proven-safe mode): the DP kernels' prepared virtual row 0
// holds +inf values (prepare_kernel), so at a virtual column all three
// candidates are already +inf and no per-cell select is needed; the caller
// feeds zup = +inf above row 1 and zupp_next = 0 after the virtual column
// (z(0, 0) = 0 is the diagonal of cell (1, 1)). The d / c values computed
// against the virtual column (+inf, or NaN for infinite inputs) only ever meet
// z_diag = z(r, 0) = +inf, whose match candidate is never selected.
//
// The work of one column is split in two so kernels can software-pipeline it:
// dists() (the K local distances, independent of the wavefront) and chain()
// (the K-row min recurrence that carries z down the lane's rows).
// SA (shared-memory rows): the lane's K rows of A (values and times) live in
// shared memory instead of registers, [row][16-byte chunk][32 lanes] so every
// warp-wide LDS.128 is one contiguous 512-byte access; frees (D+1)*K*2
// registers per thread for the scheduler. sa = this lane's first chunk.
template <int D, typename R>
struct RowChunks {
    static constexpr int EPC = 16 / sizeof(R);                // elements per chunk
    static constexpr int NCH = (D + 1 + EPC - 1) / EPC;       // chunks per row
    static constexpr int BYTES_PER_LANE_ROW = NCH * 16;
};

// D == 0: runtime dimension `dd` (any d >= 1). The lane's K rows of A live at
// sa[(q * dd + k) * 32] -- the warp's block [row][component][32 lanes] in
// shared memory, or in a per-warp global scratch block when it does not fit
// (the same addressing through a generic pointer); times stay in registers.
// Column values come from the dim-major copy (PreparedT::vt): element k of
// the lane's column at bcol[k * ldt], so a warp's 32 consecutive columns are
// one coalesced load per component, reused for the K rows.
#ifndef TWB_DYN_PREFETCH
#define TWB_DYN_PREFETCH 0
#endif
// unrolling of the runtime-d component loop (loads of later components in
// flight while earlier ones are summed)
#ifndef TWB_DYN_UNROLL
#define TWB_DYN_UNROLL 4
#endif
constexpr int DYN_UNROLL = TWB_DYN_UNROLL;
template <int D, int K, int P, bool EXACT_NAN, bool NU1, typename R, typename Z, bool SA = false>
struct LaneRows {
    static constexpr bool F32 = sizeof(R) == 4;
    static constexpr bool DYN = D == 0;
    static constexpr int DV = DYN ? 1 : D;  // static extent of value arrays
    static constexpr bool SPLIT_SQRT = !F32 && (D >= 2 || DYN) && P == 2;
    static constexpr bool COL0_BY_INF = !EXACT_NAN;
    static_assert(!(DYN && SA), "runtime-d rows have their own layout");
    using RC = RowChunks<DV, R>;
    R a[(SA || DYN) ? 1 : K][DV];
    R ta[SA ? 1 : K];
    R* sa = nullptr;  // SA: element (lane * EPC) of the warp's row block; DYN: see above
    int dd = DV;      // DYN: components per sample

    // values and time of row slot q
    __device__ __forceinline__ void row(int q, R (&v)[DV], R& t) const {
        if constexpr (SA) {
            R e[RC::NCH * RC::EPC];
#pragma unroll
            for (int c = 0; c < RC::NCH; ++c) {
                const R* src = sa + (q * RC::NCH + c) * 32 * RC::EPC;
                if constexpr (sizeof(R) == 8) {
                    const double2 w = *reinterpret_cast<const double2*>(src);
                    e[2 * c] = w.x;
                    e[2 * c + 1] = w.y;
                } else {
                    const float4 w = *reinterpret_cast<const float4*>(src);
                    e[4 * c] = w.x;
                    e[4 * c + 1] = w.y;
                    e[4 * c + 2] = w.z;
                    e[4 * c + 3] = w.w;
                }
            }
#pragma unroll
            for (int k = 0; k < D; ++k) v[k] = e[k];
            t = e[D];
        } else {
#pragma unroll
            for (int k = 0; k < D; ++k) v[k] = a[q][k];
            t = ta[q];
        }
    }
    __device__ __forceinline__ R row_t(int q) const {
        if constexpr (DYN) {
            return ta[q];
        } else {
            R v[D], t;
            row(q, v, t);
            return t;
        }
    }
    Z da[K];
    Z zl[K];  // z(r, j-1)
    R mr[K];  // fp64: d(r, j-1); fp32: c(r, j-1)
    R gr[K];  // fp64: t_a(r) - t_b(j-1) (signed, |.| at use)
    Z zupp;   // z(r0-1, j-1)
    R mupp;   // d(r0-1, j-1) / c(r0-1, j-1)
    R tup;    // t_a(r0-1)
    R tbp;    // t_b(j-1)

    // Rows [r0, r0+K) of the prepared series at `base`; rows > n are zero
    // (computed, never read back).
    __device__ __forceinline__ void load(const PreparedT<R, Z>& A, int64_t base, int64_t r0,
                                         int64_t n) {
#pragma unroll
        for (int q = 0; q < K; ++q) {
            const int64_t r = r0 + q;
            const bool ok = r <= n;
            const int64_t g = base + (ok ? r : 0);
            if constexpr (DYN) {
                for (int k = 0; k < dd; ++k) sa[(q * dd + k) * 32] = ok ? A.v[g * dd + k] : R(0);
                ta[q] = ok ? A.t[g] : R(0);
            } else if constexpr (SA) {
                R e[RC::NCH * RC::EPC];
#pragma unroll
                for (int k = 0; k < RC::NCH * RC::EPC; ++k) e[k] = R(0);
#pragma unroll
                for (int k = 0; k < D; ++k) e[k] = ok ? A.v[g * D + k] : R(0);
                e[D] = ok ? A.t[g] : R(0);
#pragma unroll
                for (int c = 0; c < RC::NCH; ++c)
#pragma unroll
                    for (int k = 0; k < RC::EPC; ++k)
                        sa[(q * RC::NCH + c) * 32 * RC::EPC + k] = e[c * RC::EPC + k];
            } else {
#pragma unroll
                for (int k = 0; k < D; ++k) a[q][k] = ok ? A.v[g * D + k] : R(0);
                ta[q] = ok ? A.t[g] : R(0);
            }
            da[q] = ok ? A.del[g] : Z(0);
        }
        const int64_t ru = r0 - 1;
        tup = ru <= n ? A.t[base + ru] : R(0);
        tbp = R(0);
        zupp = zinf<Z>();
        mupp = R(0);
#pragma unroll
        for (int q = 0; q < K; ++q) {
            zl[q] = zinf<Z>();
            mr[q] = R(0);
            gr[q] = R(0);
        }
    }

    // d(r, j) for the lane's K rows.
    __device__ __forceinline__ void dists(const R (&vb)[DV], int p, R (&mn)[K]) const {
        if constexpr (SPLIT_SQRT) {
            bool ok = true;
#pragma unroll
            for (int q = 0; q < K; ++q) {
                R av[D], t;
                row(q, av, t);
                const double acc = sumsq<D>(av, vb);
                ok &= sqrt_fast_ok(acc);
                mn[q] = sqrt_fast(acc);
            }
            if (!ok) {
#pragma unroll
                for (int q = 0; q < K; ++q) {
                    R av[D], t;
                    row(q, av, t);
                    const double acc = sumsq<D>(av, vb);
                    if (!sqrt_fast_ok(acc)) mn[q] = __dsqrt_rn(acc);
                }
            }
        } else if constexpr (F32 && D >= 2 && P == 2) {
#pragma unroll
            for (int q = 0; q < K; ++q) {
                R av[D], t;
                row(q, av, t);
                const float d0 = av[0] - vb[0];
                float acc = d0 * d0;
#pragma unroll
                for (int k = 1; k < D; ++k) {
                    const float dk = av[k] - vb[k];
                    acc = __fmaf_rn(dk, dk, acc);
                }
                mn[q] = sqrt_approx<!EXACT_NAN>(acc);
            }
        } else {
#pragma unroll
            for (int q = 0; q < K; ++q) {
                R av[D], t;
                row(q, av, t);
                mn[q] = dist<D, P, R>(av, vb, p);
            }
        }
    }

    // DYN: d(r, j) for the lane's K rows, lp_dist (_kernels.py:24-48) with a
    // runtime dimension: d == 1 -> |x0 - y0|; p == 1 -> sequential sum of
    // |diff|; p == 2 -> sqrt of the sequential sum of diff*diff (fp64: same
    // association, correctly rounded root; fp32 mode: FMA sums, approximate
    // root, as the static-d fp32 kernels); else binary-exponentiation powers
    // and pow for the root. bcol = element 0 of column j in the dim-major copy.
    __device__ __forceinline__ void dists_dyn(const R* __restrict__ bcol, int64_t ldt, int p,
                                              R (&mn)[K]) const {
        static_assert(DYN, "runtime-d rows only");
        const int d = dd;
#if TWB_DYN_PREFETCH > 0
        // the column TWB_DYN_PREFETCH steps ahead into L1 (the warp's 32
        // lanes cover consecutive columns: one or two lines per component)
        for (int k = 0; k < d; ++k)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(bcol + TWB_DYN_PREFETCH + k * ldt));
#endif
        const R* ar[K];
#pragma unroll
        for (int q = 0; q < K; ++q) ar[q] = sa + (size_t)q * d * 32;
        const int pp = P ? P : p;
        if (d == 1) {
            const R b = __ldg(bcol);
#pragma unroll
            for (int q = 0; q < K; ++q) mn[q] = F32 ? (R)fabsf((float)(ar[q][0] - b)) : (R)fabs((double)(ar[q][0] - b));
            return;
        }
        if (pp == 1 || pp == 2) {
            R acc[K];
            {
                const R b = __ldg(bcol);
#pragma unroll
                for (int q = 0; q < K; ++q) {
                    const R df = ar[q][0] - b;
                    if constexpr (F32) acc[q] = pp == 1 ? fabsf(df) : df * df;
                    else acc[q] = pp == 1 ? fabs(df) : __dmul_rn(df, df);
                }
            }
            // the component loop is latency-bound (the column values come
            // from L1/L2): long vectors unroll deeper, so more loads are in
            // flight (B200, pair n = 100k: d = 28 12.1 -> 16.7 GCUPS with 8;
            // d = 8 best at 4)
            auto term = [&](int k) {
                const R b = __ldg(bcol + k * ldt);
#pragma unroll
                for (int q = 0; q < K; ++q) {
                    const R df = ar[q][k * 32] - b;
                    if constexpr (F32) acc[q] = pp == 1 ? acc[q] + fabsf(df) : __fmaf_rn(df, df, acc[q]);
                    else acc[q] = pp == 1 ? __dadd_rn(acc[q], fabs(df)) : __dadd_rn(acc[q], __dmul_rn(df, df));
                }
            };
            if (d >= 16) {
#pragma unroll 8
                for (int k = 1; k < d; ++k) term(k);
            } else {
#pragma unroll DYN_UNROLL
                for (int k = 1; k < d; ++k) term(k);
            }
            if (pp == 1) {
#pragma unroll
                for (int q = 0; q < K; ++q) mn[q] = acc[q];
            } else if constexpr (F32) {
#pragma unroll
                for (int q = 0; q < K; ++q) mn[q] = sqrt_approx<!EXACT_NAN>(acc[q]);
            } else if constexpr (!EXACT_NAN) {
                sqrt_fast0_k<K>(acc, mn);
            } else {
#pragma unroll
                for (int q = 0; q < K; ++q) mn[q] = __dsqrt_rn(acc[q]);
            }
            return;
        }
        if constexpr (P == 0) {  // degree >= 3 (runtime degree, NaN-exact kernels only)
            R acc[K];
#pragma unroll
            for (int q = 0; q < K; ++q) acc[q] = R(0);
            for (int k = 0; k < d; ++k) {
                const R b = __ldg(bcol + k * ldt);
#pragma unroll
                for (int q = 0; q < K; ++q) {
                    const R df = ar[q][k * 32] - b;
                    if constexpr (F32) acc[q] += __powf(fabsf(df), (float)pp);
                    else acc[q] = __dadd_rn(acc[q], int_power(fabs(df), pp));
                }
            }
#pragma unroll
            for (int q = 0; q < K; ++q) {
                if constexpr (F32) mn[q] = __powf(acc[q], 1.0f / (float)pp);
                else mn[q] = pow(acc[q], 1.0 / (double)pp);
            }
        }
    }

    // The K-row recurrence of column j (interior_cost, _kernels.py:61-80, per
    // row) given mn = dists(column j). zup = z(r0-1, j); mup = d / c of row
    // r0-1 at j (kept for the next column); col0: j is a virtual column 0.
    // Returns z(r0+K-1, j); mbot = d / c of row r0+K-1 at j.
    __device__ __forceinline__ Z chain(const R (&mn)[K], R tb, Z delb, Z zup, R mup, bool col0,
                                       double nu, R& mbot, Z zupp_next) {
        const Z INF = zinf<Z>();
        Z zu = zup;
        Z zd = zupp;
        if constexpr (F32) {
            const float nuf = (float)nu;
            R c_up = mupp;
#pragma unroll
            for (int q = 0; q < K; ++q) {
                const float g = row_t(q) - tb;
                const float c = NU1 ? mn[q] + fabsf(g) : __fmaf_rn(nuf, fabsf(g), mn[q]);
                const float w = c + c_up;
                Z match;
                if constexpr (sizeof(Z) == 4) match = zd + w;
                else match = zd + (double)w;  // fp32 local cost, fp64 accumulator
                const Z del_b = zl[q] + delb;
                const Z del_a = zu + da[q];
                Z z = cell_min<EXACT_NAN>(del_a, del_b, match);
                if constexpr (!COL0_BY_INF) z = col0 ? INF : z;
                zd = zl[q];
                zl[q] = z;
                zu = z;
                c_up = mr[q];
                mr[q] = c;
            }
        } else {
            R m_up = mupp;
            R g_up = tup - tbp;
#pragma unroll
            for (int q = 0; q < K; ++q) {
                const R m = mn[q];
                const R g = row_t(q) - tb;
                // ((z_diag + d_now) + d_prev) + nu * (|g_now| + |g_prev|)
                const double gs = __dadd_rn(fabs(g), fabs(g_up));
                const double tt = NU1 ? gs : __dmul_rn(nu, gs);
                const Z match = __dadd_rn(__dadd_rn(__dadd_rn(zd, m), m_up), tt);
                const Z del_b = zl[q] + delb;
                const Z del_a = zu + da[q];
                Z z = cell_min<EXACT_NAN>(del_a, del_b, match);
                if constexpr (!COL0_BY_INF) z = col0 ? INF : z;
                zd = zl[q];
                zl[q] = z;
                zu = z;
                m_up = mr[q];
                g_up = gr[q];
                mr[q] = m;
                gr[q] = g;
            }
        }
        zupp = zupp_next;
        mupp = mup;
        tbp = tb;
        mbot = mr[K - 1];
        return zu;
    }

    // ---- split form of the proven-safe recurrence (software pipelining) ----
    // In safe mode min is order-free, so cell (r, j) = min(del_a, pre) with
    // pre = min(match, del_b) computable before z(r-1, j) is known:
    //   prep(j) needs column j's distances and the column j-1 state
    //   (z, d, t-gap of rows r0-1 .. r0+K-1), chain2(j) needs pre and z(r0-1, j).
    // The kernels run chain2(j) and dists(j+1) + prep(j+1) in the same basic
    // block so the K-row recurrence overlaps the next column's arithmetic.

    // Straight-line distances (fp64 safe mode: sqrt_fast0, no branch; the
    // +inf virtual column gives NaN distances there, which only ever meet
    // z_diag = +inf and lose every min: pre = del_b, as with +inf).
    __device__ __forceinline__ void dists_safe(const R (&vb)[DV], int p, R (&mn)[K]) const {
        if constexpr (SPLIT_SQRT) {
            double acc[K];
#pragma unroll
            for (int q = 0; q < K; ++q) {
                R av[D], t;
                row(q, av, t);
                acc[q] = sumsq<D>(av, vb);
            }
            sqrt_fast0_k<K>(acc, mn);
        } else {
            dists(vb, p, mn);
        }
    }

    // pre[q] = min(match(r, j), del_b(r, j)) for the K rows; z of column j-1
    // in zl, zd0 = z(r0-1, j-1), m0 = d / c(r0-1, j-1), tbprev = t_b(j-1).
    // Updates mr / gr to column j.
    __device__ __forceinline__ void prep(const R (&mn)[K], R tb, Z delb, Z zd0, R m0, R tbprev,
                                         double nu, Z (&pre)[K]) {
        if constexpr (F32) {
            const float nuf = (float)nu;
#pragma unroll
            for (int q = K - 1; q >= 0; --q) {
                const float g = row_t(q) - tb;
                const float c = NU1 ? mn[q] + fabsf(g) : __fmaf_rn(nuf, fabsf(g), mn[q]);
                const float c_up = q > 0 ? mr[q - 1] : m0;
                const Z zd = q > 0 ? zl[q - 1] : zd0;
                const float w = c + c_up;
                Z match;
                if constexpr (sizeof(Z) == 4) match = zd + w;
                else match = zd + (double)w;
                const Z del_b = zl[q] + delb;
                pre[q] = sizeof(Z) == 4 ? (Z)fminf((float)match, (float)del_b)
                                        : safe_min(match, del_b);
                mr[q] = c;
            }
        } else {
#pragma unroll
            for (int q = K - 1; q >= 0; --q) {
                const R g = row_t(q) - tb;
                const R g_up = q > 0 ? gr[q - 1] : tup - tbprev;
                const R m_up = q > 0 ? mr[q - 1] : m0;
                const Z zd = q > 0 ? zl[q - 1] : zd0;
                const double gs = __dadd_rn(fabs(g), fabs(g_up));
                const double tt = NU1 ? gs : __dmul_rn(nu, gs);
                const Z match = __dadd_rn(__dadd_rn(__dadd_rn(zd, mn[q]), m_up), tt);
                const Z del_b = zl[q] + delb;
                pre[q] = safe_min(match, del_b);
                mr[q] = mn[q];
                gr[q] = g;
            }
        }
    }

    // The K-row recurrence z(r, j) = min(z(r-1, j) + del_a(r), pre[r]).
    __device__ __forceinline__ Z chain2(const Z (&pre)[K], Z zup) {
        Z zu = zup;
#pragma unroll
        for (int q = 0; q < K; ++q) {
            const Z del_a = zu + da[q];
            Z z;
            if constexpr (sizeof(Z) == 4) z = fminf(pre[q], del_a);
            else z = chain_min<D >= 2 && !F32>(pre[q], del_a);
            zl[q] = z;
            zu = z;
        }
        return zu;
    }

    __device__ __forceinline__ Z step(const R (&vb)[DV], R tb, Z delb, Z zup, R mup, bool col0,
                                      double nu, int p, R& mbot, Z zupp_next) {
        R mn[K];
        dists(vb, p, mn);
        return chain(mn, tb, delb, zup, mup, col0, nu, mbot, zupp_next);
    }

    // z of row slot q (runtime index) without local-memory indexing.
    __device__ __forceinline__ Z z_at(int q) const {
        Z r = zl[0];
#pragma unroll
        for (int k = 1; k < K; ++k) r = (q == k) ? zl[k] : r;
        return r;
    }
};

}  // namespace twb
