// Kernels of the B200 TWED library (sm_100a).
//
//   prepare_kernel  : per-series precompute (core.py:218-234): zero-prefixed
//                     values/times and deletion costs, HBM-bound, fused with
//                     the input check (twb_prepare.cuh).
//   batch_kernel    : all-pairs matrix (engine.py:183-226). One warp per task
//                     (A series i, a run of B series); the warp keeps A's
//                     rows in registers and streams the task's B series back
//                     to back, so the 31-step lane skew is paid once per task,
//                     not once per pair.
//   wave_kernel     : one long pair (engine.py:101-121, the band of
//                     _kernels.py:127-174). Persistent grid of row stripes;
//                     warps of a CTA are chained through shared-memory rings,
//                     CTAs through flag-synchronised global boundary rows
//                     (st.release.gpu / ld.acquire.gpu progress counters), so
//                     the anti-diagonal wavefront sweeps without a launch or a
//                     grid barrier per diagonal. The ring of CTAs may span
//                     several kernels (one per device: system-scope links to
//                     the next kernel's inbox in peer memory).
//   (lcs_kernel, the bit-parallel LCS sweep, lives in twb_lcs.cu.)
#pragma once

#include "twb_prepare.cuh"
#include "twb_stripe.cuh"

namespace twb {

// ---------------------------------------------------------------------------
// Batch: all-pairs matrix.
// ---------------------------------------------------------------------------
constexpr int MAX_CHUNK = 64;  // B series per task
#ifndef TWB_BATCH_ALLEND  // 1: every lane runs the series-end bookkeeping (A/B only)
#define TWB_BATCH_ALLEND 0
#endif

template <int D, typename R, typename Z>
__host__ __device__ constexpr size_t batch_smem(int warps) {
    return (sizeof(ColRing<D, R, Z>) * warps + sizeof(int) * MAX_CHUNK * warps + 15) / 16 * 16;
}

template <typename R, typename Z>
struct BatchArgs {
    PreparedT<R, Z> A, B;
    const int64_t* a_poff;  // prepared offsets of the A series (nAA+1)
    const int64_t* b_poff;  // prepared offsets of the B series (nBB+1)
    int64_t nBB;
    int64_t row_begin;           // first A series of this shard
    int64_t nrows;               // A series in this shard
    const int64_t* task_prefix;  // (ngroups+1) tasks before local row group
    int64_t ngroups;             // row groups of 32/LW consecutive local rows
    int64_t ntasks;
    int chunk;   // B series per task (<= MAX_CHUNK)
    int tri;     // only j >= i (engine.py:200-201)
    int mirror;  // also write (j, i) (engine.py:223-225); only when all rows are local
    Z* out;
    int64_t ld;
    double nu;
    int p;
    unsigned long long* counter;
    int dd;    // components per sample (D == 0 kernels)
    R* arows;  // D == 0: per-warp global blocks for the A rows (null: shared memory)
};

// Lanes per A series: 16 when every row-side series has <= 128 samples (two
// series per warp share one staged B stream), else 32.
// TWB_BATCH_LW8: series of <= 32 samples get 8 lanes x 4 rows (four series per
// warp) instead of 16 x 2: twice the rows per lane (more independent work per
// loaded column value) and half the lane skew.
#ifndef TWB_BATCH_LW8
#define TWB_BATCH_LW8 1
#endif
__host__ __device__ constexpr int batch_lanes(int64_t max_rows) {
    return (TWB_BATCH_LW8 && max_rows <= 32) ? 8 : max_rows <= 128 ? 16 : 32;
}

// One warp per task = (row group, run of `chunk` B series). A row group is
// 32/LW consecutive A series (LW lanes each, K rows per lane, rows in
// registers); all of them stream the same B series back to back through one
// cp.async-staged shared-memory ring, each B series with its virtual column 0,
// so the (LW-1)-step lane skew is paid once per task, not once per pair.
template <int D, int K, int LW, int P, bool EXACT_NAN, bool NU1, int WARPS, typename R, typename Z>
__global__ void __launch_bounds__(WARPS * 32) batch_kernel(const BatchArgs<R, Z> args) {
    using Lane = LaneRows<D, K, P, EXACT_NAN, NU1, R, Z>;
    constexpr int GROUPS = 32 / LW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto* rings = reinterpret_cast<ColRing<D, R, Z>*>(smem_raw);
    auto* slen = reinterpret_cast<int(*)[MAX_CHUNK]>(smem_raw + sizeof(ColRing<D, R, Z>) * WARPS);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int grp = lane / LW;
    const int hl = lane % LW;  // lane within the series' lane group
    ColRing<D, R, Z>& ring = rings[warp];
    const Z INF = zinf<Z>();
    Lane L;
    if constexpr (D == 0) {  // the warp's rows block: shared memory after the rings, or global
        R* srows = reinterpret_cast<R*>(smem_raw + batch_smem<D, R, Z>(WARPS));
        const size_t blk = (size_t)K * args.dd * 32;
        L.dd = args.dd;
        L.sa = (args.arows ? args.arows + ((size_t)blockIdx.x * WARPS + warp) * blk
                           : srows + (size_t)warp * blk) + lane;
    }
    // d(r, j) of the K rows at column j of the task's column stream
    auto col_dists = [&](int64_t c0, int j, R (&mn)[K], bool safe) {
        if constexpr (D == 0) {
            L.dists_dyn(args.B.vt + c0 + j, args.B.ldt, args.p, mn);
        } else {
            const int slot = j & (RING_COLS - 1);
            R vb[D];
#pragma unroll
            for (int k = 0; k < D; ++k) vb[k] = ring.v[slot * D + k];
            if (safe) L.dists_safe(vb, args.p, mn);
            else L.dists(vb, args.p, mn);
        }
    };

    while (true) {
        unsigned long long task = 0;
        if (lane == 0) task = atomicAdd(args.counter, 1ull);
        task = __shfl_sync(FULL, task, 0);
        if ((int64_t)task >= args.ntasks) return;
        // row group: last gi with task_prefix[gi] <= task
        int64_t lo = 0, hi = args.ngroups;
        while (hi - lo > 1) {
            int64_t mid = (lo + hi) >> 1;
            if (args.task_prefix[mid] <= (int64_t)task) lo = mid; else hi = mid;
        }
        const int64_t li0 = lo * GROUPS;             // first local row of the group
        const int64_t i0 = args.row_begin + li0;
        const int64_t jfirst = args.tri ? i0 : 0;
        const int64_t j0 = jfirst + ((int64_t)task - args.task_prefix[lo]) * args.chunk;
        const int64_t j1 = min(j0 + (int64_t)args.chunk, args.nBB);
        const int nser = (int)(j1 - j0);

        const int64_t li = li0 + grp;  // this lane group's local row
        const bool row_ok = li < args.nrows;
        const int64_t i = args.row_begin + (row_ok ? li : li0);
        const int64_t abase = args.a_poff[i];
        const int64_t nA = args.a_poff[i + 1] - abase - 1;
        L.load(args.A, abase, 1 + (int64_t)hl * K, nA);
        for (int k = lane; k < nser; k += 32)
            slen[warp][k] = (int)(args.b_poff[j0 + k + 1] - args.b_poff[j0 + k]);
        const int64_t c0 = args.b_poff[j0];
        const int ncols = (int)(args.b_poff[j1] - c0);
        stage_block<D>(ring, args.B, c0, ncols, 0, lane);
        stage_block<D>(ring, args.B, c0, ncols, 1, lane);
        __syncwarp();

        const int own_lane = (int)((nA - 1) / K);
        const int own_q = (int)((nA - 1) % K);
        const bool writer = row_ok && hl == own_lane;
        Z* orow = args.out + li * args.ld;
        int sidx = 0, pos = 0;
        int curlen = slen[warp][0];
        Z zbot = INF;
        R mbot = R(0);
        const int nsteps = ncols + LW - 1;
        auto stage = [&](int s) {  // s % 32 == 0
            cp_async_wait<0>();  // the pipelined body reads one column ahead
            __syncwarp();
            stage_block<D>(ring, args.B, c0, ncols, (s >> 5) + 2, lane);
        };
        // end of a B series at this lane's column j: write the result, advance
        auto series_end = [&](int j) {
            const int64_t jj = j0 + sidx;
            if (writer && (!args.tri || jj >= i)) {
                const Z v = L.z_at(own_q);
                orow[jj] = v;
                if (args.mirror && jj != i) args.out[(jj - args.row_begin) * args.ld + i] = v;
            }
            ++sidx;
            pos = 0;
            curlen = sidx < nser ? slen[warp][sidx] : 0;
        };
        // Generic step (fill / drain, NaN-exact mode): lanes outside [0, ncols) idle.
        auto generic = [&](int s) {
            if ((s & 31) == 0) stage(s);
            Z zup = __shfl_up_sync(FULL, zbot, 1, LW);
            R mup = __shfl_up_sync(FULL, mbot, 1, LW);
            const int j = s - hl;
            if (j >= 0 && j < ncols) {
                const int slot = j & (RING_COLS - 1);
                const R tb = ring.t[slot];
                const Z delb = ring.del[slot];
                const bool col0 = pos == 0;
                Z zpn = zup;
                if (hl == 0) {  // row 0: z(0,0)=0, z(0,j)=inf; d(0,j) only meets z=inf
                    if constexpr (Lane::COL0_BY_INF) {
                        zup = INF;
                        zpn = col0 ? Z(0) : INF;
                    } else {
                        zup = col0 ? Z(0) : INF;
                        zpn = zup;
                    }
                    mup = R(0);
                }
                R mn[K];
                col_dists(c0, j, mn, false);
                zbot = L.chain(mn, tb, delb, zup, mup, col0, args.nu, mbot, zpn);
                if (++pos == curlen) series_end(j);
            }
        };
        int s = 0;
        if constexpr (EXACT_NAN) {
            for (; s < nsteps; ++s) generic(s);
        } else {
            // Safe modes: after the LW-step fill, groups of 16 steps in which
            // every lane is busy run a software-pipelined body (chain2 of
            // column j with the distances + prep of column j+1, as in
            // wave_kernel) with predicated series bookkeeping; the drain runs
            // the same body lane-predicated.
            // (at least 16 steps: the 16-step groups below must start at a
            // multiple of 16 for the every-32-steps column staging)
            for (; s < min(LW > 16 ? LW : 16, nsteps); ++s) generic(s);
            if (s < nsteps) {
                Z pre[K];
                R tbj;
                {
                    const int j = s - hl;
                    const int slot = j & (RING_COLS - 1);
                    R mn[K];
                    col_dists(c0, j, mn, true);
                    tbj = ring.t[slot];
                    L.prep(mn, tbj, ring.del[slot], L.zupp, L.mupp, L.tbp, args.nu, pre);
                }
                auto body = [&](int t, bool check) {
                    Z zup = __shfl_up_sync(FULL, zbot, 1, LW);
                    R mup = __shfl_up_sync(FULL, mbot, 1, LW);
                    const int j = t - hl;
                    if (!check || j < ncols) {
                        const bool col0 = pos == 0;
                        // row 0 above the lane group: z(0, j) = +inf; z(0, 0) = 0
                        // enters as the diagonal of the next column
                        Z zpn = zup;
                        zup = hl == 0 ? INF : zup;
                        zpn = hl == 0 ? (col0 ? Z(0) : INF) : zpn;
                        mup = hl == 0 ? R(0) : mup;
                        zbot = L.chain2(pre, zup);
                        mbot = L.mr[K - 1];
                        const int slot = (j + 1) & (RING_COLS - 1);
                        R mn[K];
                        col_dists(c0, j + 1, mn, true);
                        const R tbn = ring.t[slot];
                        L.prep(mn, tbn, ring.del[slot], zpn, mup, tbj, args.nu, pre);
                        tbj = tbn;
                        // only lane 0 (col0 of the next series) and the writer (the result) need
                        // the series bookkeeping: other lanes skip it, so a series end is a
                        // divergent step for two lanes instead of all 32
                        if (++pos == curlen && (TWB_BATCH_ALLEND || hl == 0 || writer)) series_end(j);
                    }
                };
                while (s + 16 <= ncols) {  // lanes' columns s - hl .. s + 15 - hl all valid
                    if ((s & 31) == 0) stage(s);
#pragma unroll 1
                    for (int u = 0; u < 16; ++u) body(s + u, false);
                    s += 16;
                }
                for (; s < nsteps; ++s) {
                    if ((s & 31) == 0) stage(s);
                    body(s, true);
                }
            }
        }
        cp_async_wait<0>();
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Wavefront: one long pair.
// ---------------------------------------------------------------------------
// A waiting warp backs off so that it does not take issue slots from the warps
// it shares a sub-partition with (which include the one it waits for). B200,
// n = 1M: d = 1 1008 vs 988 GCUPS with 128 ns, d = 3 486 vs 485; 300k d = 3
// 385 vs 382 (profiles/r01g_session_ab.log).
#ifndef TWB_SPIN_NS
#define TWB_SPIN_NS 128
#endif
__device__ __forceinline__ void spin_pause() {
    if constexpr (TWB_SPIN_NS > 0) __nanosleep(TWB_SPIN_NS);
}

// Steady-state steps per loop iteration: unrolling lets the scheduler overlap
// one step's latency-bound z chain with the next step's distance arithmetic.
// 2 where the rows sit in shared memory (fp64 d >= 2: n = 1M d = 3 490 vs
// 483 GCUPS at 4), 8 where they sit in registers (vs 2: n = 100k d = 1 401 vs
// 364, 300k d = 1 845 vs 795, 1M d = 1 +1.6 %, fp32 mode +1.4 %; 16 is slower;
// profiles/r02_wave_ab.log).
#ifndef TWB_WAVE_UNROLL
#define TWB_WAVE_UNROLL 2
#endif
#ifndef TWB_WAVE_UNROLL_REG
#define TWB_WAVE_UNROLL_REG 8
#endif
// Timing experiments only (results are wrong): 1 = CTAs do not wait for the
// previous stripe's boundary row, 2 = warps do not wait for each other either.
#ifndef TWB_DBG_NOSYNC
#define TWB_DBG_NOSYNC 0
#endif
#ifndef TWB_ZRS
#define TWB_ZRS 256
#endif
constexpr int ZRS = TWB_ZRS;  // shared-memory ring between consecutive warps (columns; power of 2)
#ifndef TWB_CHS
#define TWB_CHS 32
#endif
// 32 since the 8-step unroll (r02AM: +0.3 % at the headline, +1.2 % at cfg2)
constexpr int CHS = TWB_CHS;  // warp-to-warp publish granularity (columns); divides 32
constexpr int CHG = 32;   // CTA-to-CTA read granularity (columns; publish = args.chg)
constexpr int CHG_RAMP = 4096;  // publish every group for the first columns of a stripe

template <int D, typename R, typename Z, int C>
using WaveRing = ColRing<D, R, Z, RING_COLS * C>;

template <int D, typename R, typename Z, int C>
__host__ __device__ constexpr size_t wave_smem_rings(int warps) {
    return (sizeof(WaveRing<D, R, Z, C>) * warps + 15) / 16 * 16;
}
// rings | zring[W][ZRS] | mring[W][ZRS] | gstage z[ZRS] | gstage m[ZRS] | prog[W] | cons[W]
// TWB_WAVE_SA: the lanes' rows of A in shared memory (LaneRows SA) instead
// of registers.
// -1 (default): fp64 with d >= 2, where the 3*K registers of row values
// crowd the scheduler (B200, n = 1M, d = 3: 468 vs 438 GCUPS); with d = 1 the
// extra LDS cost more than they free (944 vs 1015).
#ifndef TWB_WAVE_SA
#define TWB_WAVE_SA -1
#endif
template <int D, typename R, int K = 6>
__host__ __device__ constexpr bool wave_sa() {
    return TWB_WAVE_SA < 0 ? (D >= 2 && sizeof(R) == 8) : TWB_WAVE_SA != 0;
}
// Warp-ring size: 512 columns where the rows sit in registers (d = 1, fp32
// mode: shared memory to spare; more slack between neighbouring warps, n = 100k
// d = 1 364 vs 357 GCUPS), 256 where the rows take the shared memory.
#ifndef TWB_ZRS_REG
#define TWB_ZRS_REG 512
#endif
template <int D, typename R>
__host__ __device__ constexpr int wave_zrs() {
    return (D >= 1 && !wave_sa<D, R>()) ? TWB_ZRS_REG : TWB_ZRS;
}
template <int D, typename R, int K>
__host__ __device__ constexpr size_t wave_smem_rows(int warps) {
    return wave_sa<D, R, K>() ? (size_t)warps * 32 * K * RowChunks<D, R>::BYTES_PER_LANE_ROW : 0;
}
template <int D, typename R, typename Z, int C>
__host__ __device__ constexpr size_t wave_smem_base(int warps) {  // 16-aligned
    constexpr size_t zrs = wave_zrs<D, R>();
    return (wave_smem_rings<D, R, Z, C>(warps) + sizeof(Z) * (zrs * warps + zrs) +
            sizeof(R) * (zrs * warps + zrs) + sizeof(int) * 2 * warps + 15) / 16 * 16;
}
template <int D, typename R, typename Z, int C, int K>
__host__ __device__ constexpr size_t wave_smem(int warps) {
    return wave_smem_base<D, R, Z, C>(warps) + wave_smem_rows<D, R, K>(warps);
}

template <typename R, typename Z>
struct WaveArgs {
    PreparedT<R, Z> A, B;  // single prepared series each (row 0 virtual)
    int64_t nA, nB;
    int64_t S;  // stripes
    int64_t H;  // rows per stripe
    // Inboxes: slot b holds the bottom row (z, d / c) of the stripe above the
    // one CTA b is sweeping, written by the CTA before it in the ring, and
    // that producer's progress counter (stripe*(nB+1) + columns published).
    Z* gbuf;            // gridDim.x x (nB+1)
    R* gmbuf;           // gridDim.x x (nB+1)
    long long* gprog;   // gridDim.x
    // The ring of CTAs may span several kernels (one per device, or several
    // on one device): this kernel's CTAs are ring positions cta0 .. cta0+G-1
    // of GT; stripe s belongs to ring position s % GT. The last CTA feeds the
    // next kernel's CTA 0 through next_* (a peer pointer across devices; for a
    // single kernel next_* = slot 0 of the own inboxes).
    int64_t cta0, GT;
    Z* next_z;
    R* next_m;
    long long* next_prog;
    int sys;            // publish / poll the cross-kernel links at system scope
    int* abort;         // multi-kernel rings: set on a wait timeout (null: no timeout)
    long long timeout_ns;
    int chg;            // publish granularity of the bottom row (power of 2, >= 32)
    double nu;
    int p;
    double* out;
    long long* dbg;  // diagnostics (TWB_DBG_TIMES): per stripe start / input ready / end (ns)
    const int* gate;  // run only if (*gate & 1) == gate_want (device-side variant choice)
    int gate_want;
    int dd;    // components per sample (D == 0 kernels)
    R* arows;  // D == 0: per-warp global blocks for the A rows (null: shared memory)
};

__device__ __forceinline__ long long globaltimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Stripe sweep. C = columns per lane step: lane t at step s handles columns
// C*(s - t) + c, c < C, so one step carries C*K cells per lane and the
// steady-state body holds C chain2/prep pairs -- more independent work per
// step for the same per-step latency of the warp-to-warp wavefront.
template <int D, int K, int C, int P, bool EXACT_NAN, bool NU1, int WARPS, int MINB, typename R,
          typename Z>
__global__ void __launch_bounds__(WARPS * 32, MINB) wave_kernel(const WaveArgs<R, Z> args) {
    using Lane = LaneRows<D, K, P, EXACT_NAN, NU1, R, Z, wave_sa<D, R, K>()>;
    using Ring = WaveRing<D, R, Z, C>;
    constexpr int NC = Ring::N;
    constexpr int GCOLS = C * CHS;  // columns per group of CHS steps
    constexpr int ZRS = wave_zrs<D, R>();  // this configuration's warp-ring size
    constexpr int UNROLL = (D >= 1 && !wave_sa<D, R>()) ? TWB_WAVE_UNROLL_REG : TWB_WAVE_UNROLL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto* rings = reinterpret_cast<Ring*>(smem_raw);
    unsigned char* p0 = smem_raw + wave_smem_rings<D, R, Z, C>(WARPS);
    auto* zring = reinterpret_cast<Z(*)[ZRS]>(p0);
    p0 += sizeof(Z) * ZRS * WARPS;
    auto* mring = reinterpret_cast<R(*)[ZRS]>(p0);
    p0 += sizeof(R) * ZRS * WARPS;
    Z* gstage = reinterpret_cast<Z*>(p0);  // warp 0's row-above ring (global input / row 0)
    p0 += sizeof(Z) * ZRS;
    R* gmstage = reinterpret_cast<R*>(p0);
    p0 += sizeof(R) * ZRS;
    int* prog = reinterpret_cast<int*>(p0);
    int* cons = prog + WARPS;
    R* srows = reinterpret_cast<R*>(smem_raw + wave_smem_base<D, R, Z, C>(WARPS));  // SA rows (16-aligned)
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (args.gate && ((__ldcg(args.gate) & 1) != args.gate_want)) return;  // the other variant runs
    const int G = gridDim.x;
    const int b = blockIdx.x;
    const int64_t gb = args.cta0 + b;  // ring position
    __shared__ int s_abort;
    if (threadIdx.x == 0) s_abort = 0;
    auto s_abort_seen = [&]() { return args.abort != nullptr && *(volatile int*)&s_abort != 0; };
    // cross-kernel links: CTA 0 polls a producer in another kernel, the last
    // CTA publishes to one
    const bool sys_in = args.sys && b == 0;
    const bool sys_out = args.sys && b == G - 1;
    Ring& ring = rings[warp];
    const Z INF = zinf<Z>();
    const int ncols = (int)(args.nB + 1);
    const int nsteps = (ncols + C - 1) / C + 31;
    Lane L;
    if constexpr (D == 0) {
        const size_t blk = (size_t)K * args.dd * 32;
        L.dd = args.dd;
        L.sa = (args.arows ? args.arows + ((size_t)b * WARPS + warp) * blk : srows + (size_t)warp * blk) +
               lane;
    } else if constexpr (wave_sa<D, R, K>()) {
        L.sa = srows + ((size_t)warp * K * Lane::RC::NCH * 32 + lane) * Lane::RC::EPC;
    }

    const int64_t s_last = (args.nA - 1) / args.H;
    const int64_t loc_last = (args.nA - 1) - s_last * args.H;
    const int own_warp = (int)(loc_last / (32 * K));
    const int own_lane = (int)((loc_last / K) % 32);
    const int own_q = (int)(loc_last % K);

    for (int64_t s = gb; s < args.S; s += args.GT) {
        __syncthreads();
        if (threadIdx.x < WARPS) {
            prog[threadIdx.x] = 0;
            cons[threadIdx.x] = 0;
        }
        __syncthreads();
        const int64_t first_row = 1 + s * args.H;
        const int64_t rows = min(args.H, args.nA - s * args.H);
        const int wact = (int)((rows + 32 * K - 1) / (32 * K));
        if (warp >= wact) continue;

        if (args.dbg && lane == 0) {
            if (warp == 0) args.dbg[s * 4] = globaltimer();
            args.dbg[args.S * (4 + WARPS) + s * WARPS + warp] = globaltimer();
        }
        L.load(args.A, 0, first_row + (int64_t)(warp * 32 + lane) * K, args.nA);
        // columns [0, 64C): the first 64 steps
#pragma unroll
        for (int k = 0; k < 2 * C; ++k) stage_block<D>(ring, args.B, 0, ncols, k, lane);
        __syncwarp();

        const bool top_boundary = s == 0;                    // row 0 above warp 0
        const bool to_ring = warp < wact - 1;                // feed warp+1
        const bool to_global = !to_ring && s + 1 < args.S;   // feed the next stripe
        const bool owner = s == s_last && warp == own_warp && lane == own_lane;
        const long long gbase_in = (long long)(s - 1) * ncols;
        const long long gbase_out = (long long)s * ncols;
        // own inbox in, the next ring position's inbox out
        const Z* grow_in = args.gbuf + (int64_t)b * ncols;
        const R* gmrow_in = args.gmbuf + (int64_t)b * ncols;
        Z* grow_out = b + 1 < G ? args.gbuf + (int64_t)(b + 1) * ncols : args.next_z;
        R* gmrow_out = b + 1 < G ? args.gmbuf + (int64_t)(b + 1) * ncols : args.next_m;
        long long* prog_out = b + 1 < G ? args.gprog + b + 1 : args.next_prog;

        // Previous stripe's bottom row (warp 0 of a non-top stripe): the 32C
        // columns of the next 32 steps are loaded into registers one block
        // ahead (latency hidden behind 32 steps) and parked in the gstage ring.
        const bool from_global = warp == 0 && !top_boundary;
        Z pz[C];
        R pm[C];
        auto fetch = [&](int c0) {  // columns [c0, c0 + 32C) -> registers
            const long long need = gbase_in + min(c0 + 32 * C, ncols);
            if (TWB_DBG_NOSYNC < 1) {
                if (args.abort) {  // multi-kernel ring: bounded wait
                    if (!gwait_bounded(args.gprog + b, need, sys_in, args.abort, args.timeout_ns))
                        s_abort = 1;
                } else {
                    gwait(args.gprog + b, need);
                }
            }
#pragma unroll
            for (int k = 0; k < C; ++k) {
                const int c = c0 + 32 * k + lane;
                pz[k] = c < ncols ? __ldcg(grow_in + c) : Z(0);
                pm[k] = c < ncols ? __ldcg(gmrow_in + c) : R(0);
            }
        };
        if (from_global) fetch(0);
        if (args.dbg && warp == 0 && lane == 0) args.dbg[s * 4 + 1] = globaltimer();

        // Warp-uniform per-step bookkeeping: column staging, boundary-row
        // fetch, ring flow control with the neighbouring warps.
        auto preamble = [&](int st) {
            if ((st & 31) == 0) {
                // every staged block has landed; the pipelined body reads up to
                // 2C columns past its own
                cp_async_wait<0>();
                __syncwarp();
#pragma unroll
                for (int k = 0; k < C; ++k)
                    stage_block<D>(ring, args.B, 0, ncols, (C * (st + 64)) / 32 + k, lane);
                if (from_global && C * st < ncols) {
#pragma unroll
                    for (int k = 0; k < C; ++k) {
                        const int c = C * st + 32 * k + lane;
                        gstage[c % ZRS] = pz[k];
                        gmstage[c % ZRS] = pm[k];
                    }
                    if (C * (st + 32) < ncols) fetch(C * (st + 32));
                    __syncwarp();
                }
            }
            if (warp > 0 && (st % CHS) == 0 && C * st < ncols) {
                if (lane == 0) st_release_cta(&cons[warp], C * st);
                const int need = min(C * (st + CHS), ncols);
                while (TWB_DBG_NOSYNC < 2 && ld_acquire_cta(&prog[warp]) < need && !s_abort_seen())
                    spin_pause();
            }
            const int j31 = C * (st - 31);  // lane 31's first column this step
            if (to_ring && j31 >= 0 && j31 < ncols && (j31 % GCOLS) == 0) {
                const int need = j31 + GCOLS - ZRS;
                while (TWB_DBG_NOSYNC < 2 && ld_acquire_cta(&cons[warp + 1]) < need &&
                       !s_abort_seen())
                    spin_pause();
            }
        };
        // The row above lane 0 at column C*st + c, read by every lane from a
        // warp-uniform address, selected for lane 0.
        auto top_input = [&](int st, int c, Z& zup, R& mup, Z& zpn) {
            const int col = C * st + c;
            Z zt;
            R mt;
            Z pn;
            if (warp > 0) {
                zt = zring[warp][col % ZRS];
                mt = mring[warp][col % ZRS];
                pn = zt;
            } else if (top_boundary) {  // row 0; d(0, j) only meets z = inf
                const bool c0 = col == 0;
                if constexpr (Lane::COL0_BY_INF) {
                    zt = INF;
                    pn = c0 ? Z(0) : INF;
                } else {
                    zt = c0 ? Z(0) : INF;
                    pn = zt;
                }
                mt = R(0);
            } else {
                zt = gstage[col % ZRS];
                mt = gmstage[col % ZRS];
                pn = zt;
            }
            if (lane == 0) {
                zup = zt;
                mup = mt;
                zpn = pn;
            }
        };
        // publish after lane 31 finished column j (generic / drain steps)
        auto publish = [&](int j) {
            if (to_ring) {
                if (((j + 1) % GCOLS) == 0 || j == ncols - 1)
                    if (lane == 31) st_release_cta(&prog[warp + 1], j + 1);
            } else if (to_global) {
                if (((j + 1) & (args.chg - 1)) == 0 || j == ncols - 1)
                    if (lane == 31) publish_gpu(prog_out, gbase_out + j + 1, sys_out);
            }
        };
        // Lane 31's bottom row at column j -> next warp / next stripe.
        auto bottom_output = [&](int j, Z zb, R mb) {
            if (to_ring) {
                if (lane == 31) {
                    zring[warp + 1][j % ZRS] = zb;
                    mring[warp + 1][j % ZRS] = mb;
                }
            } else if (to_global) {
                if (lane == 31) {
                    grow_out[j] = zb;
                    gmrow_out[j] = mb;
                }
            }
            publish(j);
        };
        // d(r, j) of the lane's K rows (staged column, or the dim-major copy)
        auto col_dists = [&](int j, R (&mn)[K], bool safe) {
            if constexpr (D == 0) {
                L.dists_dyn(args.B.vt + j, args.B.ldt, args.p, mn);
            } else {
                const int slot = j & (NC - 1);
                R vb[D];
#pragma unroll
                for (int k = 0; k < D; ++k) vb[k] = ring.v[slot * D + k];
                if (safe) L.dists_safe(vb, args.p, mn);
                else L.dists(vb, args.p, mn);
            }
        };

        Z zbot[C];
        R mbot[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            zbot[c] = INF;
            mbot[c] = R(0);
        }
        // Generic step (NaN-exact mode, and the fill / drain of rows too short
        // for the pipelined body): lanes' columns outside [0, ncols) idle.
        auto generic = [&](int st) {
            preamble(st);
            Z zin[C];
            R min_[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                zin[c] = __shfl_up_sync(FULL, zbot[c], 1);
                min_[c] = __shfl_up_sync(FULL, mbot[c], 1);
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int j = C * (st - lane) + c;
                Z zup = zin[c];
                R mup = min_[c];
                Z zpn = zup;
                if (C * st + c < ncols) top_input(st, c, zup, mup, zpn);
                if (j >= 0 && j < ncols) {
                    const int slot = j & (NC - 1);
                    R mn[K];
                    col_dists(j, mn, false);
                    zbot[c] = L.chain(mn, ring.t[slot], ring.del[slot], zup, mup, j == 0, args.nu,
                                      mbot[c], zpn);
                    if (owner && j == ncols - 1) args.out[0] = L.z_at(own_q);
                }
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int j = C * (st - 31) + c;
                if (j >= 0 && j < ncols) bottom_output(j, zbot[c], mbot[c]);
            }
        };

        int st = 0;
        // Pipeline fill (the first 32 steps, lanes t > st idle): the pipelined
        // body below, lane-predicated. The fill is on the critical path of the
        // whole sweep (each warp's lane 31 feeds the next warp, each CTA the
        // next CTA), and the generic step runs ~2.4x slower than the pipelined
        // one (B200, n = 1M: 51 vs 21 us per warp). Tiny rows keep the generic
        // path.
#ifndef TWB_PFILL
#define TWB_PFILL 1
#endif
        const bool pfill = TWB_PFILL && !EXACT_NAN && ncols > C * (32 + 2 * CHS) + 64;
        if (!pfill)
            for (; st < min(32, nsteps); ++st) generic(st);
        // Steady state (safe modes), software-pipelined: chain2 of a column and
        // the distances + prep of the next column form one basic block, C times
        // per step. Groups of CHS steps in which every lane's every column is
        // valid run a branch-free body with flow control once per group; the
        // drain runs the same body lane-predicated.
        if (args.dbg && lane == 0) args.dbg[args.S * 4 + s * WARPS + warp] = globaltimer();
        if (!EXACT_NAN && st < nsteps) {
            if (warp == 0 && top_boundary) {  // row 0 for columns >= 32C: z = +inf, d = 0
                for (int c = lane; c < ZRS; c += 32) {
                    gstage[c] = INF;
                    gmstage[c] = R(0);
                }
                __syncwarp();
            }
            const Z* tz = warp > 0 ? zring[warp] : gstage;
            const R* tm = warp > 0 ? mring[warp] : gmstage;
            // lane 31's output: next warp's ring, the global boundary row, or
            // a dummy slot (last stripe's last warp); generic pointers
            Z* oz = to_ring ? zring[warp + 1] : (to_global ? grow_out : gstage);
            R* om = to_ring ? mring[warp + 1] : (to_global ? gmrow_out : gmstage);
            const int omask = to_ring ? ZRS - 1 : (to_global ? 0x7fffffff : 0);
            const bool ow = lane == 31 && (to_ring || to_global);
            Z pre[K];
#pragma unroll
            for (int q = 0; q < K; ++q) pre[q] = INF;
            R tbj = L.tbp;
            // the column staging of [0, 64C) was only issued: without this
            // wait the pipelined fill's first prep (lane 0, column 0) can read
            // the slot's previous stripe (nondeterministic +2432 at d = 3)
            cp_async_wait<0>();
            __syncwarp();
            if (C * (st - lane) >= 0) {
                const int j = C * (st - lane);
                const int slot = j & (NC - 1);
                R mn[K];
                col_dists(j, mn, true);
                tbj = ring.t[slot];
                L.prep(mn, tbj, ring.del[slot], L.zupp, L.mupp, L.tbp, args.nu, pre);
            }
            // check = false: every column < ncols; fill: columns may be < 0
            // (the lane has not started: no chain, prep only from column 0 on)
            auto body = [&](int t, bool check, bool fill) {
                Z zin[C];
                R min_[C];
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    zin[c] = __shfl_up_sync(FULL, zbot[c], 1);
                    min_[c] = __shfl_up_sync(FULL, mbot[c], 1);
                    const Z zt = tz[(C * t + c) % ZRS];
                    const R mt = tm[(C * t + c) % ZRS];
                    zin[c] = lane == 0 ? zt : zin[c];
                    min_[c] = lane == 0 ? mt : min_[c];
                }
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const int j = C * (t - lane) + c;  // column j + 1 next
                    if (fill) {
                        if (j >= 0) {
                            zbot[c] = L.chain2(pre, zin[c]);
                            mbot[c] = L.mr[K - 1];
                        }
                        if (j + 1 >= 0) {
                            // z(0, 0) = 0 is the diagonal of cell (1, 1); the
                            // row-0 ring holds +inf (the row above column 0)
                            const Z zd0 = (top_boundary && lane == 0 && j == 0) ? Z(0) : zin[c];
                            const int slot = (j + 1) & (NC - 1);
                            R mn[K];
                            col_dists(j + 1, mn, true);
                            const R tbn = ring.t[slot];
                            L.prep(mn, tbn, ring.del[slot], zd0, min_[c], tbj, args.nu, pre);
                            tbj = tbn;
                        }
                    } else if (!check || j < ncols) {
                        zbot[c] = L.chain2(pre, zin[c]);
                        mbot[c] = L.mr[K - 1];
                        if (check && owner && j == ncols - 1) args.out[0] = L.z_at(own_q);
                        const int slot = (j + 1) & (NC - 1);
                        R mn[K];
                        col_dists(j + 1, mn, true);
                        const R tbn = ring.t[slot];
                        L.prep(mn, tbn, ring.del[slot], zin[c], min_[c], tbj, args.nu, pre);
                        tbj = tbn;
                    }
                }
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const int j = C * (t - 31) + c;
                    // predicated, not branched: a lane-31-only branch makes
                    // every step a divergent region (BSSY/BSYNC + branch stalls)
                    const bool w = ow && (!check || j < ncols) && (!fill || j >= 0);
                    st_pred(oz + (j & omask), zbot[c], w);
                    st_pred(om + (j & omask), mbot[c], w);
                }
            };
            // full groups: lane 0's last column in the group is < ncols - 1
            while (C * (st + CHS) < ncols) {
                const int st0 = st;
                preamble(st);
                if (to_ring) {  // lane 31 writes columns < C*(st0 + CHS - 31) this group
                    const int need = C * (st0 + CHS - 31) - ZRS;
                    while (TWB_DBG_NOSYNC < 2 && ld_acquire_cta(&cons[warp + 1]) < need &&
                           !s_abort_seen())
                        spin_pause();
                }
                if (st0 < 32) {
                    for (int i = 0; i < CHS; ++i) body(st0 + i, false, true);
                } else {
#pragma unroll UNROLL
                    for (int i = 0; i < CHS; ++i) body(st0 + i, false, false);
                }
                st += CHS;
                const int done = C * (st - 31);  // lane 31 finished columns [0, done)
                if (done > 0) {
                    if (to_ring) {
                        if (lane == 31) st_release_cta(&prog[warp + 1], done);
                    } else if (to_global &&
                               (done <= CHG_RAMP || (done & (args.chg - 1)) < GCOLS)) {
                        // every group while the next stripe starts up, then
                        // every chg columns
                        if (lane == 31) publish_gpu(prog_out, gbase_out + done, sys_out);
                    }
                }
            }
            // drain: per-step flow control, lanes predicated on their columns
            for (; st < nsteps; ++st) {
                preamble(st);
                body(st, true, false);
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const int j = C * (st - 31) + c;
                    if (j >= 0 && j < ncols) publish(j);
                }
            }
        }
        for (; st < nsteps; ++st) generic(st);
        cp_async_wait<0>();
        __syncwarp();
        if (args.dbg && lane == 0) {
            if (warp == 0) args.dbg[s * 4 + 2] = globaltimer();
            if (warp == wact - 1) args.dbg[s * 4 + 3] = globaltimer();
        }
    }
}

}  // namespace twb
