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
// words; lane l of CTA b (one warp per CTA) owns KW consecutive words (KW = 1
// unless the grid would not be co-resident) and keeps them in registers for
// the whole sweep. Rows stream by: at step st lane l handles row st - l, so
// the carry out of its top word reaches lane l+1 by warp shuffle exactly when
// that lane needs it (the same one-step lane skew as the TWED wavefront). Lane
// 31's carries leave the CTA packed 32 rows per 64-bit slot, tagged with the
// slot index in the same store; the next CTA polls the slot itself, loading it
// one chunk of 32 rows ahead. The carry chain over a lane's words is one
// add.cc/addc.cc sequence. Match masks PM[c][w] are built once on the device
// (A x W x 8 bytes) and each warp keeps its slice in shared memory.
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


struct LcsArgs {
    const int32_t* s;        // row symbols, dense codes in [0, A) or -1 (absent from t)
    int64_t ns;
    const uint64_t* pm;      // PM[c * W + w]
    int64_t W;               // words over the columns
    int64_t nt;              // columns
    // (G + 1) inboxes of ceil(ns / 32) slots: slot k = (k + 1) << 32 | the 32
    // carry bits of rows 32k .. 32k+31 -- tag and payload in one 64-bit store,
    // so the consumer polls the slot itself and no fence is needed
    unsigned long long* carry;
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

__device__ __forceinline__ unsigned long long lcs_ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void lcs_st_pred(unsigned long long* p, unsigned long long v, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
                 "@q st.relaxed.gpu.global.u64 [%0], %1;\n\t}" ::"l"(p), "l"(v), "r"((int)pred)
                 : "memory");
}

// V + U + cin over KW 64-bit words (one carry chain); returns the carry out.
template <int KW>
__device__ __forceinline__ unsigned add_chain(uint64_t (&S)[KW], const uint64_t (&V)[KW],
                                              const uint64_t (&U)[KW], unsigned cin) {
    unsigned co;
    if constexpr (KW == 1) {
        unsigned sl, sh;
        asm("{\n\t.reg .u32 t;\n\t"
            "add.cc.u32 t, %3, 0xffffffff;\n\t"  // carry flag = cin (0 or 1)
            "addc.cc.u32 %0, %4, %6;\n\t"
            "addc.cc.u32 %1, %5, %7;\n\t"
            "addc.u32 %2, 0, 0;\n\t}"
            : "=r"(sl), "=r"(sh), "=r"(co)
            : "r"(cin), "r"((unsigned)V[0]), "r"((unsigned)(V[0] >> 32)), "r"((unsigned)U[0]),
              "r"((unsigned)(U[0] >> 32)));
        S[0] = ((uint64_t)sh << 32) | sl;
    } else {
        static_assert(KW == 2, "one or two words per lane");
        unsigned s0l, s0h, s1l, s1h;
        asm("{\n\t.reg .u32 t;\n\t"
            "add.cc.u32 t, %5, 0xffffffff;\n\t"
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
    }
    return co;
}

// One warp per CTA. Steps run in chunks of 32: at a chunk's start the warp
// stages the symbols of the rows its lanes meet in the chunk (rows outside
// [0, ns) get the code of an all-zero mask, which makes them no-ops: with
// M = 0 and carry-in 0, V and the carry out are unchanged), lane 0 fetches the
// chunk's 32 carry bits from the previous CTA, and the 32 unrolled steps run
// without a branch: mask lookup, carry by shuffle, add chain, update. Lane 31
// publishes its 32 carry-outs of a word at step 30 of the next chunk.
// SPM: the warp's slice of the masks ([A + 1][KW][32 lanes], last row zero)
// lives in shared memory, else it is read through the read-only cache.
template <int KW, bool SPM>
__global__ void __launch_bounds__(32) lcs_kernel(const LcsArgs a, int alphabet) {
    extern __shared__ uint64_t spm[];
    __shared__ int ssym[64];
    const int lane = threadIdx.x;
    const int b = blockIdx.x;
    const int G = gridDim.x;
    const int64_t w0 = ((int64_t)b * 32 + lane) * KW;
    const int64_t nwc = (a.ns + 31) / 32;  // carry words per inbox
    const unsigned long long* cin_src = a.carry + (int64_t)b * nwc;
    unsigned long long* cout_dst = a.carry + (int64_t)(b + 1) * nwc;
    bool wok[KW];
    uint64_t V[KW];
#pragma unroll
    for (int k = 0; k < KW; ++k) {
        wok[k] = w0 + k < a.W;
        V[k] = ~0ull;
    }
    if constexpr (SPM) {
        for (int c = 0; c <= alphabet; ++c)
#pragma unroll
            for (int k = 0; k < KW; ++k)
                spm[((int64_t)c * KW + k) * 32 + lane] =
                    (c < alphabet && wok[k]) ? __ldg(a.pm + (int64_t)c * a.W + w0 + k) : 0ull;
    }
    unsigned co = 0, cp = 0;
    // symbols of rows st0 - 31 .. st0 + 32 (two per lane), loaded one chunk ahead
    auto fetch_syms = [&](int64_t st0, int (&c)[2]) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t r = st0 - 31 + h * 32 + lane;
            c[h] = (r >= 0 && r < a.ns) ? __ldg(a.s + r) : -1;
        }
    };
    int nxt[2];
    fetch_syms(0, nxt);
    unsigned long long cpre = b > 0 ? lcs_ld_relaxed(cin_src) : 0ull;  // next chunk's carry slot
    for (int64_t st0 = 0; st0 <= 32 * nwc; st0 += 32) {
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h)  // -1 (cannot match, or no row) -> the zero mask
            ssym[h * 32 + lane] = nxt[h] < 0 ? alphabet : nxt[h];
        fetch_syms(st0 + 32, nxt);
        unsigned cwin = 0;  // carries into rows st0 .. st0 + 31 (used by lane 0)
        if (b > 0 && st0 < a.ns) {  // warp-uniform: every lane polls the same slot
            // the slot was loaded one chunk ago (its L2 latency hidden behind 32
            // steps); reload only while the producer has not reached it
            const int64_t k = st0 >> 5;
            const unsigned long long tag = (unsigned long long)(k + 1) << 32;
            unsigned long long v = cpre;
            while ((v >> 32 << 32) != tag) {
                __nanosleep(20);
                v = lcs_ld_relaxed(cin_src + k);
            }
            cwin = (unsigned)v;
            if (k + 1 < nwc) cpre = lcs_ld_relaxed(cin_src + k + 1);
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int sym = ssym[j - lane + 31];
            uint64_t M[KW], U[KW], S[KW];
#pragma unroll
            for (int k = 0; k < KW; ++k) {
                if constexpr (SPM) M[k] = spm[((int64_t)sym * KW + k) * 32 + lane];
                else M[k] = (sym < alphabet && wok[k]) ? __ldg(a.pm + (int64_t)sym * a.W + w0 + k) : 0ull;
                U[k] = V[k] & M[k];
            }
            unsigned cin = __shfl_up_sync(0xffffffffu, co, 1);
            cin = lane == 0 ? (cwin >> j) & 1u : cin;
            co = add_chain<KW>(S, V, U, cin);
#pragma unroll
            for (int k = 0; k < KW; ++k) V[k] = S[k] | (V[k] & ~M[k]);
            // lane 31 met row st0 + j - 31: bit (j + 1) & 31 of word ((st0 + j - 31) >> 5)
            if (j == 31) {
                cp = co;
            } else {
                cp |= co << (j + 1);
                if (j == 30) {  // word (st0 >> 5) - 1 complete
                    const int64_t wd = (st0 >> 5) - 1;
                    // predicated, not branched: a divergent region here would
                    // make every shuffle of the chunk a WARPSYNC.COLLECTIVE
                    lcs_st_pred(cout_dst + (wd < 0 ? 0 : wd), (unsigned long long)(wd + 1) << 32 | cp,
                                lane == 31 && b + 1 < G && wd >= 0 && wd < nwc);
                }
            }
        }
    }
    // columns still set in V are not in the LCS
    unsigned long long ones = 0;
#pragma unroll
    for (int k = 0; k < KW; ++k) {
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
    if ((double)alphabet * (double)W * 8.0 > 4.0e9)
        return api_fail(TWB_EUNSUP, "alphabet x length too large for the match-mask table (> 4 GB)");
    cudaStream_t st = cudaStreamPerThread;
    void *d_s = nullptr, *d_t = nullptr, *d_pm = nullptr, *d_carry = nullptr, *d_ones = nullptr;
    auto cleanup = [&]() {
        for (void* p : {d_s, d_t, d_pm, d_carry, d_ones})
            if (p) cudaFreeAsync(p, st);
        cudaStreamSynchronize(st);
    };
    int prev_dev = -1;
    if (cudaGetDevice(&prev_dev) != cudaSuccess) prev_dev = -1;
    struct Restore {
        int d;
        ~Restore() {
            if (d >= 0) cudaSetDevice(d);
        }
    } restore{prev_dev};
    LCK(cudaSetDevice(device));
    int sms = 0;
    LCK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    // The widest variant whose grid is co-resident: one word per lane (the
    // shortest carry chain per step), masks in shared memory when they fit.
    using Kern = void (*)(const LcsArgs, int);
    struct Cand {
        Kern k;
        int kw;
        bool spm;
    };
    const Cand cands[] = {{lcs_kernel<1, true>, 1, true}, {lcs_kernel<1, false>, 1, false},
                          {lcs_kernel<2, true>, 2, true}, {lcs_kernel<2, false>, 2, false}};
    Kern kern = nullptr;
    int64_t G = 0;
    size_t smem = 0;
    for (const Cand& c : cands) {
        const size_t sm = c.spm ? (size_t)(alphabet + 1) * c.kw * 32 * sizeof(uint64_t) : 0;
        if (sm > 200 * 1024) continue;
        if (cudaFuncSetAttribute(c.k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        int occ = 0;
        LCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, c.k, 32, sm));
        const int64_t g = (W + 32 * c.kw - 1) / (32 * c.kw);
        if (occ > 0 && g <= (int64_t)sms * occ) {
            kern = c.k;
            G = g;
            smem = sm;
            break;
        }
    }
    if (!kern) {
        cleanup();
        return api_fail(TWB_EUNSUP, "sequence too long for one co-resident sweep");
    }
    const int64_t nwc = (ns + 31) / 32;
    LCK(cudaMallocAsync(&d_s, sizeof(int32_t) * ns, st));
    LCK(cudaMallocAsync(&d_t, sizeof(int32_t) * nt, st));
    LCK(cudaMallocAsync(&d_pm, sizeof(uint64_t) * (size_t)alphabet * W, st));
    LCK(cudaMallocAsync(&d_carry, sizeof(unsigned long long) * (size_t)(G + 1) * nwc, st));
    LCK(cudaMallocAsync(&d_ones, sizeof(unsigned long long), st));
    LCK(cudaMemcpyAsync(d_s, s, sizeof(int32_t) * ns, cudaMemcpyHostToDevice, st));
    LCK(cudaMemcpyAsync(d_t, t, sizeof(int32_t) * nt, cudaMemcpyHostToDevice, st));
    LCK(cudaMemsetAsync(d_pm, 0, sizeof(uint64_t) * (size_t)alphabet * W, st));
    LCK(cudaMemsetAsync(d_carry, 0, sizeof(unsigned long long) * (size_t)(G + 1) * nwc, st));
    LCK(cudaMemsetAsync(d_ones, 0, sizeof(unsigned long long), st));
    lcs_masks_kernel<<<(unsigned)((W + 255) / 256), 256, 0, st>>>((const int32_t*)d_t, nt, W,
                                                                 (uint64_t*)d_pm);
    api_count_launch();
    LCK(cudaGetLastError());
    LcsArgs a{(const int32_t*)d_s, ns, (const uint64_t*)d_pm, W, nt,
              (unsigned long long*)d_carry, (unsigned long long*)d_ones};
    int alpha = alphabet;
    void* params[] = {(void*)&a, (void*)&alpha};
    LaunchCtx* ctx = api_ctx_begin();
    ctx->before(st);
    // cooperative: CTA b spins on CTA b-1, all must be resident
    LCK(cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)G), dim3(32), params, smem,
                                    st));
    ctx->after(st);
    unsigned long long ones = 0;
    LCK(cudaMemcpyAsync(&ones, d_ones, sizeof ones, cudaMemcpyDeviceToHost, st));
    cleanup();
    *out = nt - (int64_t)ones;
    return 0;
}
