// Host-side launchers (templates instantiated per D / precision in
// twb_inst_*.cu so the 100+ kernel variants compile in parallel).
#pragma once

#include <cuda_runtime.h>
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

template <typename R, typename Z>
struct WaveProblem {
    PreparedT<R, Z> A, B;
    int64_t nA, nB;
    double nu;
    int p;
    Z* out;  // device, one value
};

// Batch kernel variants (lanes per series LW, rows per lane K): row-side
// series of <= 32 / 64 / 128 samples -> LW = 16, K = 2 / 4 / 8 (two series
// per warp); <= 256 -> LW = 32, K = 8. 4 warps per CTA, persistent grid with an
// atomic task counter. The host groups rows by batch_lanes(max_rows).
constexpr int BATCH_WARPS = 4;
constexpr int BATCH_KMAX = 8;

template <int D, int P, bool E, bool N1, typename R, typename Z>
cudaError_t run_batch(BatchArgs<R, Z> a, int64_t max_rows, cudaStream_t st, LaunchCtx* ctx) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = batch_smem<D, R, Z>(BATCH_WARPS);
    auto go = [&](auto kern) -> cudaError_t {
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
        ctx->before(st);
        kern<<<(unsigned)grid, BATCH_WARPS * 32, smem, st>>>(a);
        ctx->after(st);
        return cudaGetLastError();
    };
    if (max_rows <= 16 * 2) return go(batch_kernel<D, 2, 16, P, E, N1, BATCH_WARPS, R, Z>);
    if (max_rows <= 16 * 4) return go(batch_kernel<D, 4, 16, P, E, N1, BATCH_WARPS, R, Z>);
    if (max_rows <= 16 * 8) return go(batch_kernel<D, 8, 16, P, E, N1, BATCH_WARPS, R, Z>);
    if (max_rows <= 32 * 8) return go(batch_kernel<D, 8, 32, P, E, N1, BATCH_WARPS, R, Z>);
    return cudaErrorInvalidValue;
}

// Wavefront variants (rows per lane K, warps per CTA W, CTAs per SM MINB);
// run_wave picks one by the row-side length.
template <int D, int K, int C, int P, bool E, bool N1, int W, int MINB, typename R, typename Z>
cudaError_t run_wave_cfg(const WaveProblem<R, Z>& pr, const Alloc& alloc, cudaStream_t st,
                         LaunchCtx* ctx) {
    auto kern = wave_kernel<D, K, C, P, E, N1, W, MINB, R, Z>;
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = wave_smem<D, R, Z, C, K>(W);
    int occ = 0;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, W * 32, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorLaunchOutOfResources;
    // Stripe height: ws active warps of 32*K rows (ws <= W). Every stripe
    // sweeps all nB+1 columns, so a round of G co-resident stripes costs about
    // nB steps however many rows it holds, and the pipeline fill adds
    // ~(32 + CHS) steps per warp of the whole first round. Pick ws so the
    // stripes fill every SM slot in the fewest rounds (e.g. n = 1M, K = 8:
    // 7 warps -> 559 stripes = 3.8 rounds of 148, instead of 8 warps -> 489
    // stripes on only 123 SMs).
    const int64_t cap = (int64_t)sms * occ;
    int64_t H = 0, S = 0, G = 0;
    double best = 0;
    // TWB_WAVE_WS=<n> pins the active warps per stripe (tuning experiments).
    int ws_pin = 0;
    if (const char* env = getenv("TWB_WAVE_WS")) ws_pin = atoi(env);
    // Per-step time grows with the SM's load once its FP64 pipe is busy:
    // factor max(1, ws*K*F/400)^0.75, F ~ FP64 instructions per cell (fitted
    // to B200 sweeps, e.g. n = 100k: d = 1 best at 1024-row stripes, d = 3 at
    // 512; n = 300k d = 3 at 1024; n = 1M at 12 x 6 rows).
    const double F = D == 1 ? 10.0 : D == 2 ? 20.0 : D == 3 ? 24.0 : 27.0;
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
    WaveArgs<R, Z> a;
    a.A = pr.A;
    a.B = pr.B;
    a.nA = pr.nA;
    a.nB = pr.nB;
    a.S = S;
    a.H = H;
    // Bottom-row publish granularity: every st.release.gpu costs the
    // producing warp a GPU-scope fence, so publish every chg columns (more for
    // long rows; the consumer lags far behind anyway). TWB_WAVE_CHG overrides.
    int chg = 32;
    while (chg < 256 && (int64_t)chg * 2048 <= pr.nB) chg *= 2;
    if (const char* env = getenv("TWB_WAVE_CHG")) chg = atoi(env);
    if (chg < 32 || (chg & (chg - 1))) chg = 32;
    a.chg = chg;
    a.nu = pr.nu;
    a.p = pr.p;
    a.out = pr.out;
    a.gbuf = (Z*)alloc.get(sizeof(Z) * (size_t)G * (size_t)(pr.nB + 1));
    a.gmbuf = (R*)alloc.get(sizeof(R) * (size_t)G * (size_t)(pr.nB + 1));
    a.gprog = (long long*)alloc.get(sizeof(long long) * (size_t)G);
    if (!a.gbuf || !a.gprog || !a.gmbuf) return cudaErrorMemoryAllocation;
    e = cudaMemsetAsync(a.gprog, 0, sizeof(long long) * (size_t)G, st);
    if (e != cudaSuccess) return e;
    // TWB_DBG_TIMES=<file>: per-stripe timestamps (diagnostics, synchronises)
    const char* dbg_path = getenv("TWB_DBG_TIMES");
    a.dbg = dbg_path ? (long long*)alloc.get(sizeof(long long) * (4 + 2 * W) * (size_t)S) : nullptr;
    void* params[] = {(void*)&a};
    // Cooperative launch: every CTA must be co-resident (CTA b spins on CTA b-1).
    ctx->before(st);
    e = cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)G), dim3(W * 32), params, smem, st);
    ctx->after(st);
    if (e == cudaSuccess && a.dbg) {
        std::vector<long long> h((size_t)S * (4 + 2 * W));
        cudaMemcpyAsync(h.data(), a.dbg, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, st);
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
cudaError_t run_wave(const WaveProblem<R, Z>& pr, const Alloc& alloc, cudaStream_t st,
                     LaunchCtx* ctx) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
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
    if (pr.nA >= (int64_t)sms * 12 * 32 * 6 * 3 / 2)
        return run_wave_cfg<D, 6, 1, P, E, N1, 12, 1, R, Z>(pr, alloc, st, ctx);
    return run_wave_cfg<D, 4, 1, P, E, N1, 12, 1, R, Z>(pr, alloc, st, ctx);
}

}  // namespace twb
