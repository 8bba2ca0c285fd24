// Longest common subsequence length on B200: the
// reference's lcs_band (pkg/src/twedband/band.py:185-197, kernel
// _kernels.py:193-219, a three-diagonal integer DP) re-designed as a
// bit-parallel sweep (Hyyro's LCS recurrence over 64-bit words).
//
//   V = all ones over the columns (symbols of t); for each row symbol c:
//     U = V & PM[c];  V = (V + U) | (V & ~PM[c])
//   LCS = (number of columns) - popcount(V)
// where PM[c] marks the columns holding c and the + carries across the whole
// bit-vector. Integer arithmetic, so the result equals the reference's DP
// exactly (tests pin it against the reference's values and the C oracle).
//
// Layout and schedule. Columns are the longer sequence (more parallel width),
// rows the shorter one (LCS is symmetric). The bit-vector is cut into 64-bit
// words; lane l of CTA b (one warp per CTA) owns LCS_KW consecutive words and
// keeps them in registers for the whole sweep. Rows stream by: at step st lane
// l handles row st - l, so the carry out of its top word reaches lane l+1 by
// warp shuffle exactly when that lane needs it (the same one-step lane skew as
// the TWED wavefront). Lane 31's carries leave the CTA packed 32 rows per
// word into the next CTA's inbox with a release-published progress counter;
// lane 0 of the next CTA polls it with acquire once per 32 rows. The carry
// chain over a lane's words is one add.cc/addc.cc sequence. Match masks
// PM[c][w] are built once on the device (A x W x 8 bytes) and read through
// the read-only cache.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/twb.h"
#include "twb_launch.cuh"

namespace twb {
int api_fail(int code, const char* msg);
void api_count_launch();
LaunchCtx* api_ctx_begin();
}  // namespace twb

namespace {

using namespace twb;

constexpr int LCS_KW = 2;  // 64-bit words per lane

struct LcsArgs {
    const int32_t* s;        // row symbols, dense codes in [0, A) or -1 (absent from t)
    int64_t ns;
    const uint64_t* pm;      // PM[c * W + w]
    int64_t W;               // words over the columns
    int64_t nt;              // columns
    unsigned* carry;         // (G + 1) inboxes of ceil(ns / 32) packed carry words
    long long* prog;         // G + 1 progress counters (carry words published)
    unsigned long long* ones;
};

// Build PM: thread w sets the bits of its 64 columns.
__global__ void lcs_masks_kernel(const int32_t* __restrict__ t, int64_t nt, int64_t W,
                                 uint64_t* __restrict__ pm) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= W) return;
    for (int j = 0; j < 64; ++j) {
        const int64_t pos = w * 64 + j;
        if (pos >= nt) break;
        const int c = t[pos];
        if (c >= 0) pm[(int64_t)c * W + w] |= 1ull << j;
    }
}

__device__ __forceinline__ long long lcs_ld_acquire(const long long* p) {
    long long v;
    asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void lcs_st_release(long long* p, long long v) {
    asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// V + U + cin over two 64-bit words (one carry chain); returns the carry out.
__device__ __forceinline__ unsigned add2(uint64_t (&S)[2], const uint64_t (&V)[2],
                                         const uint64_t (&U)[2], unsigned cin) {
    unsigned s0l, s0h, s1l, s1h, co;
    asm("{\n\t.reg .u32 t;\n\t"
        "add.cc.u32 t, %5, 0xffffffff;\n\t"  // carry flag = cin (0 or 1)
        "addc.cc.u32 %0, %6, %10;\n\t"
        "addc.cc.u32 %1, %7, %11;\n\t"
        "addc.cc.u32 %2, %8, %12;\n\t"
        "addc.cc.u32 %3, %9, %13;\n\t"
        "addc.u32 %4, 0, 0;\n\t}"
        : "=r"(s0l), "=r"(s0h), "=r"(s1l), "=r"(s1h), "=r"(co)
        : "r"(cin), "r"((unsigned)V[0]), "r"((unsigned)(V[0] >> 32)), "r"((unsigned)V[1]),
          "r"((unsigned)(V[1] >> 32)), "r"((unsigned)U[0]), "r"((unsigned)(U[0] >> 32)),
          "r"((unsigned)U[1]), "r"((unsigned)(U[1] >> 32)));
    S[0] = ((uint64_t)s0h << 32) | s0l;
    S[1] = ((uint64_t)s1h << 32) | s1l;
    return co;
}

__global__ void __launch_bounds__(32) lcs_kernel(const LcsArgs a) {
    static_assert(LCS_KW == 2, "add2 chains two words");
    const int lane = threadIdx.x;
    const int b = blockIdx.x;
    const int G = gridDim.x;
    const int64_t w0 = ((int64_t)b * 32 + lane) * LCS_KW;
    const int64_t nwc = (a.ns + 31) / 32;  // carry words per inbox
    const unsigned* cin_src = a.carry + (int64_t)b * nwc;
    unsigned* cout_dst = a.carry + (int64_t)(b + 1) * nwc;
    bool wok[LCS_KW];
    uint64_t V[LCS_KW];
#pragma unroll
    for (int k = 0; k < LCS_KW; ++k) {
        wok[k] = w0 + k < a.W;
        V[k] = ~0ull;
    }
    unsigned cout_prev = 0, cin_word = 0, cpack = 0;
    const int64_t nsteps = a.ns + 31;
    for (int64_t st = 0; st < nsteps; ++st) {
        const int64_t i = st - lane;  // this lane's row
        unsigned cin = __shfl_up_sync(0xffffffffu, cout_prev, 1);
        if (lane == 0) {
            cin = 0;
            if (b > 0 && st < a.ns) {
                if ((st & 31) == 0) {  // the next 32 rows' carries from CTA b-1
                    while (lcs_ld_acquire(a.prog + b) < (st >> 5) + 1) __nanosleep(32);
                    cin_word = __ldcg(cin_src + (st >> 5));
                }
                cin = (cin_word >> (st & 31)) & 1u;
            }
        }
        unsigned co = 0;
        if (i >= 0 && i < a.ns) {
            const int sym = __ldg(a.s + i);
            uint64_t M[LCS_KW], U[LCS_KW], S[LCS_KW];
#pragma unroll
            for (int k = 0; k < LCS_KW; ++k) {
                M[k] = (sym >= 0 && wok[k]) ? __ldg(a.pm + (int64_t)sym * a.W + w0 + k) : 0ull;
                U[k] = V[k] & M[k];
            }
            co = add2(S, V, U, cin);
#pragma unroll
            for (int k = 0; k < LCS_KW; ++k) V[k] = S[k] | (V[k] & ~M[k]);
            if (lane == 31 && b + 1 < G) {
                cpack |= co << (i & 31);
                if ((i & 31) == 31 || i == a.ns - 1) {
                    cout_dst[i >> 5] = cpack;
                    cpack = 0;
                    lcs_st_release(a.prog + b + 1, (i >> 5) + 1);
                }
            }
        }
        cout_prev = co;
    }
    // columns still set in V are not in the LCS
    unsigned long long ones = 0;
#pragma unroll
    for (int k = 0; k < LCS_KW; ++k) {
        if (!wok[k]) continue;
        uint64_t v = V[k];
        const int64_t w = w0 + k;
        if (w == a.W - 1 && (a.nt & 63)) v &= (1ull << (a.nt & 63)) - 1;
        ones += __popcll(v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ones += __shfl_down_sync(0xffffffffu, ones, o);
    if (lane == 0) atomicAdd(a.ones, ones);
}

#define LCK(...)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (__VA_ARGS__);                                                  \
        if (e_ != cudaSuccess) {                                                         \
            cleanup();                                                                   \
            return api_fail(e_ == cudaErrorMemoryAllocation ? TWB_ENOMEM : TWB_ECUDA,   \
                            cudaGetErrorString(e_));                                     \
        }                                                                                \
    } while (0)

}  // namespace

extern "C" int twb_lcs_i32(const int32_t* s, int64_t ns, const int32_t* t, int64_t nt,
                           int32_t alphabet, int32_t device, int64_t* out) {
    if (!out || ns < 0 || nt < 0 || (ns > 0 && !s) || (nt > 0 && !t))
        return api_fail(TWB_EINVAL, "bad arguments");
    if (alphabet < 0) return api_fail(TWB_EINVAL, "alphabet must be >= 0");
    if (ns == 0 || nt == 0 || alphabet == 0) {  // empty input or no common symbol
        *out = 0;
        return 0;
    }
    if (ns > nt) {  // columns = the longer sequence (LCS is symmetric)
        std::swap(s, t);
        std::swap(ns, nt);
    }
    const int64_t W = (nt + 63) / 64;
    const int64_t G = (W + 32 * LCS_KW - 1) / (32 * LCS_KW);
    if ((double)alphabet * (double)W * 8.0 > 4.0e9)
        return api_fail(TWB_EUNSUP, "alphabet x length too large for the match-mask table (> 4 GB)");
    cudaStream_t st = cudaStreamPerThread;
    void *d_s = nullptr, *d_t = nullptr, *d_pm = nullptr, *d_carry = nullptr, *d_prog = nullptr,
         *d_ones = nullptr;
    auto cleanup = [&]() {
        for (void* p : {d_s, d_t, d_pm, d_carry, d_prog, d_ones})
            if (p) cudaFreeAsync(p, st);
        cudaStreamSynchronize(st);
    };
    LCK(cudaSetDevice(device));
    int sms = 0, occ = 0;
    LCK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    LCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lcs_kernel, 32, 0));
    if (G > (int64_t)sms * occ) {
        cleanup();
        return api_fail(TWB_EUNSUP, "sequence too long for one co-resident sweep");
    }
    const int64_t nwc = (ns + 31) / 32;
    LCK(cudaMallocAsync(&d_s, sizeof(int32_t) * ns, st));
    LCK(cudaMallocAsync(&d_t, sizeof(int32_t) * nt, st));
    LCK(cudaMallocAsync(&d_pm, sizeof(uint64_t) * (size_t)alphabet * W, st));
    LCK(cudaMallocAsync(&d_carry, sizeof(unsigned) * (size_t)(G + 1) * nwc, st));
    LCK(cudaMallocAsync(&d_prog, sizeof(long long) * (G + 1), st));
    LCK(cudaMallocAsync(&d_ones, sizeof(unsigned long long), st));
    LCK(cudaMemcpyAsync(d_s, s, sizeof(int32_t) * ns, cudaMemcpyHostToDevice, st));
    LCK(cudaMemcpyAsync(d_t, t, sizeof(int32_t) * nt, cudaMemcpyHostToDevice, st));
    LCK(cudaMemsetAsync(d_pm, 0, sizeof(uint64_t) * (size_t)alphabet * W, st));
    LCK(cudaMemsetAsync(d_prog, 0, sizeof(long long) * (G + 1), st));
    LCK(cudaMemsetAsync(d_ones, 0, sizeof(unsigned long long), st));
    lcs_masks_kernel<<<(unsigned)((W + 255) / 256), 256, 0, st>>>((const int32_t*)d_t, nt, W,
                                                                 (uint64_t*)d_pm);
    api_count_launch();
    LCK(cudaGetLastError());
    LcsArgs a{(const int32_t*)d_s, ns, (const uint64_t*)d_pm, W, nt, (unsigned*)d_carry,
              (long long*)d_prog, (unsigned long long*)d_ones};
    void* params[] = {(void*)&a};
    LaunchCtx* ctx = api_ctx_begin();
    ctx->before(st);
    // cooperative: CTA b spins on CTA b-1, all must be resident
    LCK(cudaLaunchCooperativeKernel((const void*)lcs_kernel, dim3((unsigned)G), dim3(32), params, 0,
                                    st));
    ctx->after(st);
    unsigned long long ones = 0;
    LCK(cudaMemcpyAsync(&ones, d_ones, sizeof ones, cudaMemcpyDeviceToHost, st));
    cleanup();
    *out = nt - (int64_t)ones;
    return 0;
}
