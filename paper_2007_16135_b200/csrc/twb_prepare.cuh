// Per-series precompute (the reference's prepare_series, core.py:218-234,
// with K.consecutive_costs, _kernels.py:51-58) fused with the input check
// that picks the DP kernels' proven-safe or NaN-exact mode.
//
// One launch covers one or two segments (a pair's two series, or a packed
// CSR list of series). A CTA takes tiles of PREP_TILE x PREP_SPT consecutive samples:
// the tile's raw values and timestamps, plus the sample before it, are
// staged in shared memory by bulk asynchronous copies (cp.async.bulk, TMA
// engine, completion on an mbarrier; the < 16-byte unaligned head and tail of
// each range are loaded by threads), so every HBM byte is read once and the
// previous sample of the consecutive cost comes from shared memory. Each
// thread then computes one sample:
//   Del[o] = (lp(v_i - v_{i-1}) + nu*|t_i - t_{i-1}|) + lam   (core.py:233)
// with v_{-1} = 0, t_{-1} = 0 for a series' first sample (C:163-174), and
// writes the prepared row o = i + k + 1 (sample i of series k); the series'
// first sample also writes its virtual row o - 1 (V = virt, T = 0,
// Del = +inf). The input check (every |x| < limit; fp values also 0 or >= tiny)
// is a warp vote and one atomicOr per warp that finds a violation.
//
// Bound: HBM. Algorithmic bytes per sample: reads (d + 1) * sizeof(T),
// writes d * sizeof(R) + sizeof(R) + sizeof(Z) (+ d * sizeof(R) for the
// dim-major copy of the runtime-d kernels).
#pragma once

#include "twb_device.cuh"

namespace twb {

constexpr int PREP_TILE = 256;  // threads per CTA
constexpr int PREP_SPT = 4;     // samples per thread and tile (tile = 1024 samples)
constexpr int PREP_DMAX = 64;   // staged dimensions (larger d: values read from global)

template <typename T, typename R, typename Z>
struct PrepSeg {
    const T* v;          // (ntot, d) raw samples
    const T* t;          // (ntot)
    const int64_t* off;  // (nseries + 1) device offsets, or null with uniform_n
    int64_t nseries, ntot, uniform_n;
    R* V;                // (ntot + nseries, d) prepared
    R* Tm;               // (ntot + nseries)
    Z* Del;              // (ntot + nseries)
    R* Vt;               // optional dim-major copy, leading dimension ldt
    int64_t ldt;
    int64_t tiles;       // ceil(ntot / (PREP_TILE * PREP_SPT))
};

template <typename T, typename R, typename Z>
struct PrepArgs {
    PrepSeg<T, R, Z> seg[2];
    int nseg;
    int d;
    double nu, lam;
    int p;
    double virt;         // virtual row value: 0 (reference layout) or +inf (DP kernels' copy)
    double limit, tiny;  // input check: |x| < limit, and x == 0 or |x| >= tiny (values)
    int* flag;           // |= 1 when a check fails (null: no check)
    int staged;          // values staged in (dynamic) shared memory
};

__device__ __forceinline__ double lp_rt(const double* x, const double* y, int d, int p) {
    if (d == 1) return fabs(x[0] - y[0]);
    if (p == 1) {
        double acc = fabs(x[0] - y[0]);
        for (int k = 1; k < d; ++k) acc = __dadd_rn(acc, fabs(x[k] - y[k]));
        return acc;
    }
    if (p == 2) {
        double d0 = x[0] - y[0];
        double acc = __dmul_rn(d0, d0);
        for (int k = 1; k < d; ++k) {
            double dk = x[k] - y[k];
            acc = __dadd_rn(acc, __dmul_rn(dk, dk));
        }
        return __dsqrt_rn(acc);
    }
    double acc = 0.0;
    for (int k = 0; k < d; ++k) acc = __dadd_rn(acc, int_power(fabs(x[k] - y[k]), p));
    return pow(acc, 1.0 / (double)p);
}

// ---- bulk asynchronous copies (TMA engine) ---------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TWB_MBAR_WAIT%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TWB_MBAR_WAIT%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Staging of elements [e0, e1) of src into buf: element e lands at byte
// (address(src + e) - base) of buf, base = address(src + e0) rounded down to
// 16. The 16-byte-aligned interior goes by one bulk copy (issued by thread 0
// after it armed the barrier with every copy's byte count); the unaligned head
// and tail (< 16 bytes each) are loaded by threads 1.. with plain loads.
template <typename T>
struct Staged {
    const T* src;
    unsigned char* buf;
    uintptr_t base, b0;
    unsigned bytes;  // bulk part
    int64_t e0, nh, t0, nt;
    __device__ __forceinline__ void plan(unsigned char* buf_, const T* src_, int64_t e0_, int64_t e1) {
        src = src_;
        buf = buf_;
        e0 = e0_;
        const uintptr_t a0 = (uintptr_t)(src + e0), a1 = (uintptr_t)(src + e1);
        base = a0 & ~(uintptr_t)15;
        b0 = (a0 + 15) & ~(uintptr_t)15;
        const uintptr_t b1 = a1 & ~(uintptr_t)15;
        bytes = b1 > b0 ? (unsigned)(b1 - b0) : 0u;
        nh = min((int64_t)((b0 - a0) / sizeof(T)), e1 - e0);
        t0 = bytes ? (int64_t)((b1 - a0) / sizeof(T)) : nh;
        nt = (e1 - e0) - t0;
    }
    __device__ __forceinline__ void issue(uint64_t* bar) const {
        if (threadIdx.x == 0 && bytes) bulk_g2s(buf + (b0 - base), (const void*)b0, bytes, bar);
        const int tid = (int)threadIdx.x - 1;
        if (tid >= 0 && tid < nh) put(e0 + tid);
        if (tid >= 0 && tid < nt) put(e0 + t0 + tid);
    }
    __device__ __forceinline__ void put(int64_t e) const {
        *reinterpret_cast<T*>(buf + ((uintptr_t)(src + e) - base)) = src[e];
    }
    __device__ __forceinline__ T at(int64_t e) const {  // after the barrier
        return *reinterpret_cast<const T*>(buf + ((uintptr_t)(src + e) - base));
    }
};

__device__ __forceinline__ bool value_bad(double a, double limit, double tiny) {
    a = fabs(a);
    return !(a < limit) || (a != 0.0 && a < tiny);
}

// lp distance of sample i to sample i-1 (zero vector before a series' first
// sample), lp_dist's operation order (_kernels.py:24-48); D > 0: compile-time
// dimension (registers), D == 0: runtime d, read element by element.
template <int D, typename GC, typename GP>
__device__ __forceinline__ double consecutive_cost(GC cur, GP prev, bool first, int d, int p) {
    if constexpr (D > 0) {
        double x[D], y[D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            x[c] = cur(c);
            y[c] = first ? 0.0 : prev(c);
        }
        return lp_rt(x, y, D, p);
    } else {
        if (d == 1) return fabs(cur(0) - (first ? 0.0 : prev(0)));
        double acc = 0.0;
        for (int c = 0; c < d; ++c) {
            const double df = cur(c) - (first ? 0.0 : prev(c));
            if (p == 1 || p == 2) {
                const double term = p == 1 ? fabs(df) : __dmul_rn(df, df);
                acc = c == 0 ? term : __dadd_rn(acc, term);
            } else {
                acc = __dadd_rn(acc, int_power(fabs(df), p));
            }
        }
        return p == 1 ? acc : p == 2 ? __dsqrt_rn(acc) : pow(acc, 1.0 / (double)p);
    }
}

// D: compile-time dimension (1..4) or 0 (runtime args.d). A tile is
// PREP_TILE * PREP_SPT samples; thread t handles samples t, t + PREP_TILE, ...
// of it (consecutive threads, consecutive samples: coalesced stores).
// Dynamic shared memory: the staged values of a tile,
// (PREP_TILE * PREP_SPT + 1) * d * sizeof(T) + 32 bytes, when args.staged
// (else values are read from global memory).
template <typename T, typename R, typename Z, int D>
__global__ void __launch_bounds__(PREP_TILE) prepare_kernel(const PrepArgs<T, R, Z> args) {
    constexpr int TS = PREP_TILE * PREP_SPT;
    extern __shared__ __align__(16) unsigned char sv[];
    __shared__ __align__(16) unsigned char st_[(TS + 1) * sizeof(T) + 32];
    __shared__ __align__(8) uint64_t bar;
    const int d = D > 0 ? D : args.d;
    const bool staged_v = args.staged != 0;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    unsigned phase = 0;
    const int64_t ntiles = args.seg[0].tiles + (args.nseg > 1 ? args.seg[1].tiles : 0);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int sg = tile < args.seg[0].tiles ? 0 : 1;
        const PrepSeg<T, R, Z>& S = args.seg[sg];
        const int64_t i0 = (tile - (sg ? args.seg[0].tiles : 0)) * TS;
        const int64_t i1 = min(i0 + TS, S.ntot);
        const int64_t j0 = i0 > 0 ? i0 - 1 : 0;  // the sample before the tile
        __syncthreads();  // every thread is done with the previous tile's buffers
        if (threadIdx.x == 0) fence_proxy_async_smem();
        Staged<T> stv, stt;
        stt.plan(st_, S.t, j0, i1);
        if (staged_v) stv.plan(sv, S.v, j0 * d, i1 * d);
        if (threadIdx.x == 0) mbar_arrive_tx(&bar, stt.bytes + (staged_v ? stv.bytes : 0u));
        stt.issue(&bar);
        if (staged_v) stv.issue(&bar);
        __syncthreads();  // the threads' head / tail stores
        mbar_wait(&bar, phase);
        phase ^= 1;
        // shared-memory views in element units: element e of the arrays sits at
        // tv[e - j0] / vv[e - j0*d]
        const T* tv = reinterpret_cast<const T*>(st_ + ((uintptr_t)(S.t + j0) - stt.base));
        const T* vv = staged_v ? reinterpret_cast<const T*>(sv + ((uintptr_t)(S.v + j0 * d) - stv.base))
                               : nullptr;
        bool bad = false;
#pragma unroll
        for (int m = 0; m < PREP_SPT; ++m) {
            const int64_t i = i0 + threadIdx.x + m * PREP_TILE;
            if (i >= i1) break;
            // series of sample i: one series (a pair's) -> 0; equal lengths ->
            // a division (32-bit when it fits); ragged -> binary search
            int64_t k = 0, start = 0;
            if (S.nseries > 1) {
                if (S.uniform_n > 0) {
                    k = (S.ntot < (1ll << 31)) ? (int64_t)((unsigned)i / (unsigned)S.uniform_n)
                                               : i / S.uniform_n;
                    start = k * S.uniform_n;
                } else {  // last k with off[k] <= i
                    int64_t lo = 0, hi = S.nseries;
                    while (hi - lo > 1) {
                        const int64_t mid = (lo + hi) >> 1;
                        if (S.off[mid] <= i) lo = mid; else hi = mid;
                    }
                    k = lo;
                    start = S.off[k];
                }
            }
            const bool first = i == start;
            const int li = (int)(i - j0);  // position in the staged tile
            const double ti = (double)tv[li];
            const double tp = first ? 0.0 : (double)tv[li - 1];
            bad |= args.flag && value_bad(ti, args.limit, 0.0);
            const T* x = staged_v ? vv + (size_t)li * d : S.v + i * d;  // sample i
            const T* y = x - d;                                         // sample i - 1
            auto cur = [&](int c) { return (double)x[c]; };
            auto prev = [&](int c) { return (double)y[c]; };
            const double cost = consecutive_cost<D>(cur, prev, first, d, args.p);
            if (args.flag)
                for (int c = 0; c < d; ++c) bad |= value_bad(cur(c), args.limit, args.tiny);
            const double gap = fabs(ti - tp);
            const int64_t o = i + k + 1;
            S.Tm[o] = (R)ti;
            S.Del[o] = (Z)__dadd_rn(__dadd_rn(cost, __dmul_rn(args.nu, gap)), args.lam);  // core.py:233
            for (int c = 0; c < d; ++c) S.V[o * d + c] = (R)x[c];
            if (S.Vt)  // dim-major copy: consecutive threads, consecutive rows
                for (int c = 0; c < d; ++c) S.Vt[c * S.ldt + o] = (R)x[c];
            if (first) {  // the series' virtual row o - 1
                for (int c = 0; c < d; ++c) S.V[(o - 1) * d + c] = (R)args.virt;
                if (S.Vt)
                    for (int c = 0; c < d; ++c) S.Vt[c * S.ldt + o - 1] = (R)args.virt;
                S.Tm[o - 1] = R(0);
                S.Del[o - 1] = (Z)dinf();
            }
        }
        if (args.flag) {
            if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(args.flag, 1);
        }
    }
}

}  // namespace twb
