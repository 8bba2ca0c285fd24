// Host-side launchers (templates instantiated per D / precision in
// twb_inst_*.cu so the 100+ kernel variants compile in parallel).
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <cstdio>
#include <vector>

#include <cstdint>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "twb_kernels.cuh"

namespace twb {

struct WaveCfg {
    int warps;  // warps per CTA
    int k;      // rows per lane
};

// Per-call launch bookkeeping: kernel count, and (when timing is on) CUDA
// events bracketing the main DP kernel on its stream.
struct LaunchCtx {
    int64_t launches = 0;
    bool timing = false;
    int64_t wave_stripes = 0, wave_rows = 0, wave_ctas = 0;  // shape of the last sweep
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    void before(cudaStream_t st) {
        if (timing) cudaEventRecord(ev0, st);
    }
    void after(cudaStream_t st) {
        ++launches;
        if (timing) cudaEventRecord(ev1, st);
    }
};

// Scratch allocation hook provided by the API layer (stream-ordered).
struct Alloc {
    void* (*fn)(void* ctx, size_t bytes);
    void* ctx;
    void* get(size_t bytes) const { return fn(ctx, bytes); }
};

// One kernel of a CTA ring that spans several kernels (one per device, or
// several on one device): its device, stream, the prepared series on that
// device, its result slot and scratch allocator.
template <typename R, typename Z>
struct WavePart {
    int device;
    cudaStream_t st;
    PreparedT<R, Z> A, B;
    Z* out;
    Alloc alloc;
};
template <typename R, typename Z>
struct CtaRing {
    int nparts;
    WavePart<R, Z>* parts;
    int* abort;             // host-mapped flag, raised by a timed-out wait
    long long timeout_ns;
    int owner = -1;         // out: the part whose out slot holds the distance
};

template <typename R, typename Z>
struct WaveProblem {
    PreparedT<R, Z> A, B;
    int64_t nA, nB;
    double nu;
    int p;
    Z* out;  // device, one value
    int dd = 0;  // components per sample (used by the D == 0 kernels)
    CtaRing<R, Z>* ring = nullptr;  // multi-kernel ring (A, B, out, alloc, st per part)
    const int* gate = nullptr;      // device flag: run only if (*gate & 1) == gate_want
    int gate_want = 0;
};

// Batch kernel variants (lanes per series LW, rows per lane K): row-side
// series of <= 32 / 64 / 128 samples -> LW = 16, K = 2 / 4 / 8 (two series
// per warp); <= 256 -> LW = 32, K = 8. 4 warps per CTA, persistent grid with an
// atomic task counter. The host groups rows by batch_lanes(max_rows).
constexpr int BATCH_WARPS = 4;
constexpr int BATCH_KMAX = 8;
// Runtime-d (D == 0) kernels keep each warp's A rows (K * d * 32 values) in
// shared memory while the CTA's total stays within these budgets; larger
// blocks go to per-warp global scratch (L1/L2-resident for moderate d).
constexpr size_t DYN_BATCH_SMEM_MAX = 100 * 1024;  // keeps >= 2 CTAs per SM
constexpr size_t DYN_WAVE_SMEM_MAX = 200 * 1024;

template <int D, int P, bool E, bool N1, typename R, typename Z>
cudaError_t run_batch(BatchArgs<R, Z> a, int64_t max_rows, const Alloc& alloc, cudaStream_t st,
                      LaunchCtx* ctx) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    auto go = [&](auto kern, int K) -> cudaError_t {
        size_t smem = batch_smem<D, R, Z>(BATCH_WARPS);
        bool rows_global = false;
        if constexpr (D == 0) {
            const size_t rows = (size_t)BATCH_WARPS * K * a.dd * 32 * sizeof(R);
            rows_global = smem + rows > DYN_BATCH_SMEM_MAX;
            if (!rows_global) smem += rows;
        }
        a.arows = nullptr;
        int occ = 0;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, BATCH_WARPS * 32, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
        int64_t want = (a.ntasks + BATCH_WARPS - 1) / BATCH_WARPS;
        int64_t grid = (int64_t)sms * occ;
        if (want < grid) grid = want;
        if (grid < 1) grid = 1;
        if (rows_global) {
            a.arows = (R*)alloc.get((size_t)grid * BATCH_WARPS * K * a.dd * 32 * sizeof(R));
            if (!a.arows) return cudaErrorMemoryAllocation;
        }
        ctx->before(st);
        kern<<<(unsigned)grid, BATCH_WARPS * 32, smem, st>>>(a);
        ctx->after(st);
        return cudaGetLastError();
    };
    if (batch_lanes(max_rows) == 8) return go(batch_kernel<D, 4, 8, P, E, N1, BATCH_WARPS, R, Z>, 4);
    if (max_rows <= 16 * 2) return go(batch_kernel<D, 2, 16, P, E, N1, BATCH_WARPS, R, Z>, 2);
    if (max_rows <= 16 * 4) return go(batch_kernel<D, 4, 16, P, E, N1, BATCH_WARPS, R, Z>, 4);
    if (max_rows <= 16 * 8) return go(batch_kernel<D, 8, 16, P, E, N1, BATCH_WARPS, R, Z>, 8);
    if (max_rows <= 32 * 8) return go(batch_kernel<D, 8, 32, P, E, N1, BATCH_WARPS, R, Z>, 8);
    return cudaErrorInvalidValue;
}

// Wavefront variants (rows per lane K, warps per CTA W, CTAs per SM MINB);
// run_wave picks one by the row-side length.
template <int D, int K, int C, int P, bool E, bool N1, int W, int MINB, typename R, typename Z>
cudaError_t run_wave_cfg(const WaveProblem<R, Z>& pr, const Alloc& alloc, cudaStream_t st,
                         LaunchCtx* ctx) {
    auto kern = wave_kernel<D, K, C, P, E, N1, W, MINB, R, Z>;
    size_t smem = wave_smem<D, R, Z, C, K>(W);
    bool rows_global = false;  // D == 0: the A rows in per-warp global blocks
    if constexpr (D == 0) {
        const size_t rows = (size_t)W * 32 * K * pr.dd * sizeof(R);
        rows_global = smem + rows > DYN_WAVE_SMEM_MAX;
        if (!rows_global) smem += rows;
    }
    // The parts of the ring: one (this device, this stream) unless pr.ring.
    std::vector<WavePart<R, Z>> parts;
    if (pr.ring) {
        parts.assign(pr.ring->parts, pr.ring->parts + pr.ring->nparts);
    } else {
        int dev = 0;
        cudaGetDevice(&dev);
        parts.push_back(WavePart<R, Z>{dev, st, pr.A, pr.B, pr.out, alloc});
    }
    const int np = (int)parts.size();
    int cur_dev = 0;
    cudaGetDevice(&cur_dev);
    // SM slots per part (parts sharing a device split it)
    std::vector<int64_t> capp(np);
    int64_t cap = 0;
    // SM slots of this kernel per device, queried once per device (the batch
    // path launches one sweep per long pair: the attribute call and the
    // occupancy query would otherwise dominate its host time)
    static std::atomic<int> slots_cache[64];
    for (int q = 0; q < np; ++q) {
        int share = 0;
        for (int r = 0; r < np; ++r) share += parts[r].device == parts[q].device;
        const int dv = parts[q].device;
        // (runtime-d kernels: shared memory depends on d, no cache)
        int slots = D == 0 || dv < 0 || dv >= 64 ? 0 : slots_cache[dv].load(std::memory_order_relaxed);
        if (slots <= 0) {
            int sms = 0, occ = 0;
            cudaError_t e = cudaSetDevice(dv);
            if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dv);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, W * 32, smem);
            if (e != cudaSuccess) return e;
            if (occ < 1) return cudaErrorLaunchOutOfResources;
            slots = sms * occ;
            if (dv >= 0 && dv < 64) slots_cache[dv].store(slots, std::memory_order_relaxed);
        }
        capp[q] = (int64_t)slots / share;
        cap += capp[q];
    }
    cudaSetDevice(cur_dev);
    // Stripe height: ws active warps of 32*K rows (ws <= W). Every stripe
    // sweeps all nB+1 columns, so a round of G co-resident stripes costs about
    // nB steps however many rows it holds, and the pipeline fill adds
    // ~(32 + CHS) steps per warp of the whole first round. Pick ws so the
    // stripes fill every SM slot in the fewest rounds (e.g. n = 1M, K = 8:
    // 7 warps -> 559 stripes = 3.8 rounds of 148, instead of 8 warps -> 489
    // stripes on only 123 SMs).
    int64_t H = 0, S = 0, G = 0;
    double best = 0;
    // TWB_WAVE_WS=<n> pins the active warps per stripe (tuning experiments).
    int ws_pin = 0;
    if (const char* env = getenv("TWB_WAVE_WS")) ws_pin = atoi(env);
    // Per-step time grows with the SM's load once its FP64 pipe is busy:
    // factor max(1, ws*K*F/400)^0.75, F ~ FP64 instructions per cell (fitted
    // to B200 sweeps, e.g. n = 100k: d = 1 best at 1024-row stripes, d = 3 at
    // 512; n = 300k d = 3 at 1024; n = 1M at 12 x 6 rows).
    const double F = D == 0 ? 3.0 * pr.dd + 12.0
                     : D == 1 ? 10.0 : D == 2 ? 20.0 : D == 3 ? 24.0 : 27.0;
    for (int ws = W; ws >= 1; --ws) {
        if (ws_pin > 0 && ws != (ws_pin < W ? ws_pin : W)) continue;
        // above 4, whole multiples of 4 warps: one warp short on a
        // sub-partition makes the others the pipeline's slow stage
        // (n = 100k: 9 warps 270 GCUPS vs 8 warps 331)
        if (ws_pin == 0 && ws > 4 && ws % 4 != 0) continue;
        const int64_t h = (int64_t)ws * 32 * K;
        const int64_t s = (pr.nA + h - 1) / h;
        const int64_t r = (s + cap - 1) / cap;
        const int64_t g = (s + r - 1) / r;
        const double load = std::max(1.0, ws * K * F / 400.0);
        const double cost = ((double)r * (double)(pr.nB + 32) +
                             (double)g * (double)(ws * (32 + CHS) + CHG)) * pow(load, 0.75) +
                            (double)(W - ws) * 1e-6;  // ties -> more warps
        if (H == 0 || cost < best) {
            best = cost;
            H = h;
            S = s;
            G = g;
        }
    }
    // Ring positions per part, in proportion to their SM slots; parts left
    // without a CTA drop out of the ring.
    std::vector<int64_t> gp(np, 0);
    {
        int64_t given = 0;
        for (int q = 0; q < np; ++q) given += gp[q] = std::min(capp[q], G * capp[q] / cap);
        for (int q = 0; given < G; q = (q + 1) % np)
            if (gp[q] < capp[q]) ++gp[q], ++given;
    }
    std::vector<int> live;
    for (int q = 0; q < np; ++q)
        if (gp[q] > 0) live.push_back(q);
    const int nl = (int)live.size();
    // Bottom-row publish granularity: every st.release.gpu costs the
    // producing warp a GPU-scope fence, but a coarse publish leaves the next
    // CTA waiting for data that exists, and its stalls travel down the chain.
    // B200 sweep (profiles/r02_wave_ab.log, r02I): 32 columns is best or tied
    // everywhere -- n = 1M d = 3 490.0 vs 484.9 GCUPS at the former 256,
    // n = 300k d = 3 420.6 vs 387.8, 1024 costs 3.4 %, 4096 15 %.
    // TWB_WAVE_CHG overrides.
    int chg = 32;
    if (const char* env = getenv("TWB_WAVE_CHG")) chg = atoi(env);
    if (chg < CHS || (chg & (chg - 1))) chg = 32;
    const size_t ncols = (size_t)(pr.nB + 1);
    std::vector<WaveArgs<R, Z>> args(nl);
    int64_t cta0 = 0;
    const int64_t pos_last = ((pr.nA - 1) / H) % G;  // ring position of the last stripe
    for (int l = 0; l < nl; ++l) {
        const WavePart<R, Z>& pt = parts[live[l]];
        WaveArgs<R, Z>& a = args[l];
        cudaSetDevice(pt.device);
        a.A = pt.A;
        a.B = pt.B;
        a.nA = pr.nA;
        a.nB = pr.nB;
        a.S = S;
        a.H = H;
        a.chg = chg;
        a.nu = pr.nu;
        a.p = pr.p;
        a.out = pt.out;
        const int64_t g = gp[live[l]];
        a.gbuf = (Z*)pt.alloc.get(sizeof(Z) * (size_t)g * ncols);
        a.gmbuf = (R*)pt.alloc.get(sizeof(R) * (size_t)g * ncols);
        a.gprog = (long long*)pt.alloc.get(sizeof(long long) * (size_t)g);
        if (!a.gbuf || !a.gprog || !a.gmbuf) return cudaErrorMemoryAllocation;
        cudaError_t e = cudaMemsetAsync(a.gprog, 0, sizeof(long long) * (size_t)g, pt.st);
        if (e != cudaSuccess) return e;
        a.cta0 = cta0;
        a.GT = G;
        if (pos_last >= cta0 && pos_last < cta0 + g && pr.ring) pr.ring->owner = live[l];
        cta0 += g;
        a.sys = nl > 1;
        a.abort = nl > 1 ? pr.ring->abort : nullptr;
        a.timeout_ns = pr.ring ? pr.ring->timeout_ns : 0;
        a.dbg = nullptr;
        a.gate = pr.gate;
        a.gate_want = pr.gate_want;
        a.dd = pr.dd;
        a.arows = nullptr;
        if (rows_global) {
            a.arows = (R*)pt.alloc.get((size_t)g * W * 32 * K * pr.dd * sizeof(R));
            if (!a.arows) return cudaErrorMemoryAllocation;
        }
    }
    for (int l = 0; l < nl; ++l) {  // the last CTA of each part feeds the next part's CTA 0
        const WaveArgs<R, Z>& nx = args[(l + 1) % nl];
        args[l].next_z = nx.gbuf;
        args[l].next_m = nx.gmbuf;
        args[l].next_prog = nx.gprog;
    }
    if (pr.gate == nullptr || pr.gate_want == 0) {  // the main sweep (not the gated NaN-exact one)
        ctx->wave_stripes = S;
        ctx->wave_rows = H;
        ctx->wave_ctas = G;
    }
    // TWB_DBG_TIMES=<file>: per-stripe timestamps (single kernel; diagnostics, synchronises)
    const char* dbg_path = nl == 1 && !pr.ring ? getenv("TWB_DBG_TIMES") : nullptr;
    if (dbg_path) args[0].dbg = (long long*)alloc.get(sizeof(long long) * (4 + 2 * W) * (size_t)S);
    // A ring over several kernels: part l's last CTA writes into part l+1's
    // inbox and progress counters, which were allocated and zeroed on part
    // l+1's stream. Every part's stream waits for all parts' set-up before
    // any kernel of the ring starts.
    if (nl > 1) {
        std::vector<cudaEvent_t> ready(nl, nullptr);
        cudaError_t e0 = cudaSuccess;
        for (int l = 0; l < nl && e0 == cudaSuccess; ++l) {
            const WavePart<R, Z>& pt = parts[live[l]];
            cudaSetDevice(pt.device);
            e0 = cudaEventCreateWithFlags(&ready[l], cudaEventDisableTiming);
            if (e0 == cudaSuccess) e0 = cudaEventRecord(ready[l], pt.st);
        }
        for (int l = 0; l < nl && e0 == cudaSuccess; ++l) {
            const WavePart<R, Z>& pt = parts[live[l]];
            cudaSetDevice(pt.device);
            for (int m = 0; m < nl && e0 == cudaSuccess; ++m)
                if (m != l) e0 = cudaStreamWaitEvent(pt.st, ready[m], 0);
        }
        for (int l = 0; l < nl; ++l)
            if (ready[l]) {
                cudaSetDevice(parts[live[l]].device);
                cudaEventDestroy(ready[l]);
            }
        if (e0 != cudaSuccess) {
            cudaSetDevice(cur_dev);
            return e0;
        }
    }
    // Cooperative launch: every CTA of a kernel is co-resident (CTA b spins on
    // CTA b-1); the kernels of a ring are launched in ring order.
    cudaError_t e = cudaSuccess;
    for (int l = 0; l < nl && e == cudaSuccess; ++l) {
        const WavePart<R, Z>& pt = parts[live[l]];
        cudaSetDevice(pt.device);
        void* params[] = {(void*)&args[l]};
        if (l == 0) ctx->before(pt.st);
        e = cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)gp[live[l]]),
                                        dim3(W * 32), params, smem, pt.st);
        if (l == 0) ctx->after(pt.st);
    }
    cudaSetDevice(cur_dev);
    if (e == cudaSuccess && dbg_path) {
        std::vector<long long> h((size_t)S * (4 + 2 * W));
        cudaMemcpyAsync(h.data(), args[0].dbg, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        if (FILE* f = fopen(dbg_path, "w")) {
            fprintf(f, "# S=%lld G=%lld H=%lld nB=%lld chg=%d\n", (long long)S, (long long)G,
                    (long long)H, (long long)pr.nB, chg);
            for (int64_t k = 0; k < S; ++k) {
                fprintf(f, "%lld %lld %lld %lld %lld", (long long)k, h[k * 4], h[k * 4 + 1],
                        h[k * 4 + 2], h[k * 4 + 3]);
                for (int w = 0; w < W; ++w) fprintf(f, " %lld", h[S * (4 + W) + k * W + w]);
                for (int w = 0; w < W; ++w) fprintf(f, " %lld", h[S * 4 + k * W + w]);
                fprintf(f, "\n");
            }
            fclose(f);
        }
    }
    return e;
}

template <int D, int P, bool E, bool N1, typename R, typename Z>
cudaError_t run_wave_static(const WaveProblem<R, Z>& pr, const Alloc& alloc, cudaStream_t st,
                            LaunchCtx* ctx, int sms);

template <int D, int P, bool E, bool N1, typename R, typename Z>
cudaError_t run_wave(const WaveProblem<R, Z>& pr, const Alloc& alloc, cudaStream_t st,
                     LaunchCtx* ctx) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (pr.ring && pr.ring->nparts > 1) {  // SMs of the whole ring
        sms = 0;
        for (int q = 0; q < pr.ring->nparts; ++q) {
            int share = 0, m = 0;
            for (int r = 0; r < pr.ring->nparts; ++r)
                share += pr.ring->parts[r].device == pr.ring->parts[q].device;
            cudaDeviceGetAttribute(&m, cudaDevAttrMultiProcessorCount, pr.ring->parts[q].device);
            sms += m / share;
        }
    }
    if constexpr (D == 0) {
        // runtime d: 8 warps; 4 rows per lane while the rows fit in shared
        // memory, else 2
        const size_t rows4 = (size_t)8 * 32 * 4 * pr.dd * sizeof(R);
        if (wave_smem<D, R, Z, 1, 4>(8) + rows4 <= DYN_WAVE_SMEM_MAX)
            return run_wave_cfg<D, 4, 1, P, E, N1, 8, 1, R, Z>(pr, alloc, st, ctx);
        return run_wave_cfg<D, 2, 1, P, E, N1, 8, 1, R, Z>(pr, alloc, st, ctx);
    } else {
        return run_wave_static<D, P, E, N1, R, Z>(pr, alloc, st, ctx, sms);
    }
}

// Compile-time d (1..4): the configuration by the row-side length.
template <int D, int P, bool E, bool N1, typename R, typename Z>
cudaError_t run_wave_static(const WaveProblem<R, Z>& pr, const Alloc& alloc, cudaStream_t st,
                            LaunchCtx* ctx, int sms) {
    // TWB_WAVE_CFG pins a variant (tuning experiments; proven-safe modes):
    // k<rows per lane>w<warps per CTA>[c<columns per step>]
    if constexpr (!E) {
        if (const char* env = getenv("TWB_WAVE_CFG")) {
            const std::string c(env);
            if (c == "k8w8") return run_wave_cfg<D, 8, 1, P, E, N1, 8, 1, R, Z>(pr, alloc, st, ctx);
            if (c == "k6w12") return run_wave_cfg<D, 6, 1, P, E, N1, 12, 1, R, Z>(pr, alloc, st, ctx);
            if (c == "k4w12") return run_wave_cfg<D, 4, 1, P, E, N1, 12, 1, R, Z>(pr, alloc, st, ctx);
#ifdef TWB_WAVE_EXTRA_CFGS  // tuning builds only
            if (c == "k6w16") return run_wave_cfg<D, 6, 1, P, E, N1, 16, 1, R, Z>(pr, alloc, st, ctx);
            if (c == "k4w16") return run_wave_cfg<D, 4, 1, P, E, N1, 16, 1, R, Z>(pr, alloc, st, ctx);
            if (c == "k8w12") return run_wave_cfg<D, 8, 1, P, E, N1, 12, 1, R, Z>(pr, alloc, st, ctx);
            if (c == "k5w16") return run_wave_cfg<D, 5, 1, P, E, N1, 16, 1, R, Z>(pr, alloc, st, ctx);
#endif
            // C = 2 (two columns per lane step) measured within 3% of C = 1
            // on the B200 (profiles/r01_c2_variants.log): not instantiated.
        }
    }
    // Long row side (>= 1.5 rounds of stripes): 12 warps x 6 rows per lane
    // (12 warps/SM hide the FP64 latency; B200 sweep: n = 1M d = 3 fp64
    // 395 GCUPS vs 376 for 8 x 8, d = 1 920 vs 775, fp32 mode 874 vs 507).
    // Shorter: 4 rows per lane, stripes of up to 12 warps sized by the cost
    // model (n = 300k d = 3: 346 GCUPS; n = 100k: d = 1 331, d = 3 170).
    const int64_t long_rows = (int64_t)sms * 12 * 32 * 6 * 3 / 2;  // 1.5 rounds of k6w12 (511k)
    if constexpr (!E && sizeof(R) == 8) {
        // fp64 mid sizes (B200 sweep, profiles/r01i_sweep_mid_sizes.log): the
        // wavefront depth nA / K dominates, so taller lanes (8 rows) win once
        // there are enough of them; short row sides keep more, shorter warps.
        //   d >= 3: 100k 207 (k8w8) vs 200 (k6w12) vs 152 (k4w12) GCUPS; 300k 382 vs 333 vs 344;
        //           600k 464 vs 415 vs 383; 1M 409 vs 484 vs 401; 30k 62 vs 58 vs 67
        //   d = 1 : 100k 332 vs 357 vs 334; 300k 710 vs 679 vs 667
        //   d = 2 : 100k  84 vs 238 vs 201; 300k 233 vs 366 vs 385
        const int64_t n = pr.nA;
        // round 2: d = 3 100k 178.9 (k8w8) vs 207.7 (k6w12) GCUPS, 300k 402.0
        // vs 358.2, 600k 463.6 vs 425.0 (K = 8 rows in registers); 300k 414.1
        // with the rows in shared memory again (after the staging-wait fix)
        if (D >= 3 && n >= (int64_t)sms * 1350 && n < (int64_t)sms * 5400)
            return run_wave_cfg<D, 8, 1, P, E, N1, 8, 1, R, Z>(pr, alloc, st, ctx);
        if (D >= 3 && n >= (int64_t)sms * 150 && n < (int64_t)sms * 1350)
            return run_wave_cfg<D, 6, 1, P, E, N1, 12, 1, R, Z>(pr, alloc, st, ctx);
        if (D == 1 && n >= (int64_t)sms * 1350 && n < long_rows)
            return run_wave_cfg<D, 8, 1, P, E, N1, 8, 1, R, Z>(pr, alloc, st, ctx);
        if (D <= 2 && n < (int64_t)sms * 1350 && n >= (int64_t)sms * 150)
            return run_wave_cfg<D, 6, 1, P, E, N1, 12, 1, R, Z>(pr, alloc, st, ctx);
    }
    if (pr.nA >= long_rows)
        return run_wave_cfg<D, 6, 1, P, E, N1, 12, 1, R, Z>(pr, alloc, st, ctx);
    return run_wave_cfg<D, 4, 1, P, E, N1, 12, 1, R, Z>(pr, alloc, st, ctx);
}

}  // namespace twb
