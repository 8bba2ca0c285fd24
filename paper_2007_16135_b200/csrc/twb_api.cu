// C ABI of libtwb200.so (declared in include/twb.h). Host orchestration:
// validation of sizes, device scratch, host<->device copies, precision and
// kernel-variant selection, and the batch task decomposition.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>
#include <functional>
#include <future>
#include <thread>

#include "../../include/twb.h"
#include "twb_dispatch.h"

namespace {

using namespace twb;

thread_local std::string t_err;
thread_local int64_t t_launches = 0;
thread_local LaunchCtx t_ctx;  // main-kernel events of the last call (timing mode)
thread_local bool t_timing = false;

int fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
    return code;
}

#define CK(...)                                                                                \
    do {                                                                                       \
        cudaError_t e_ = (__VA_ARGS__);                                                        \
        if (e_ != cudaSuccess)                                                                 \
            return fail(e_ == cudaErrorMemoryAllocation ? TWB_ENOMEM : TWB_ECUDA,              \
                        "%s: %s (%s:%d)", #__VA_ARGS__, cudaGetErrorString(e_), __FILE__,      \
                        __LINE__);                                                             \
    } while (0)

// Host entry points select their device; the caller's current device is put
// back when the call returns (a library call must not move it).
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Stream-ordered scratch, released (asynchronously) when the call returns.
struct Scratch {
    cudaStream_t st;
    std::vector<void*> ptrs;
    bool failed = false;
    explicit Scratch(cudaStream_t s) : st(s) {}
    void* get(size_t n) {
        void* p = nullptr;
        if (cudaMallocAsync(&p, n ? n : 16, st) != cudaSuccess) {
            failed = true;
            return nullptr;
        }
        ptrs.push_back(p);
        return p;
    }
    template <typename X>
    X* get_n(size_t n) {
        return (X*)get(n * sizeof(X));
    }
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};
void* scratch_alloc(void* ctx, size_t n) { return ((Scratch*)ctx)->get(n); }

// Keep up to 8 GB of freed scratch in the device's stream-ordered pool instead
// of returning it to the driver at every synchronisation (a 1M pair's boundary
// rows are 2.3 GB; re-mapping them cost 12 ms per call and 150-250 ms spikes).
// twb_trim_pool hands the cache back.
constexpr uint64_t POOL_KEEP_BYTES = 8ull << 30;
std::once_flag g_pool_once[64];
void init_pool(int dev) {
    if (dev < 0 || dev >= 64) return;
    std::call_once(g_pool_once[dev], [dev]() {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = POOL_KEEP_BYTES;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
}

// Device-resident entry points run on the caller's current device. Without
// this, the default pool's release threshold (0) hands the 1M pair's boundary
// rows back to the driver at every synchronisation and the next call re-maps
// them (12 ms per call, spikes of 150-250 ms on the B200).
void init_pool_current() {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) init_pool(dev);
}

// ---------------------------------------------------------------------------
// "safe" inputs: every value/time finite with |x| < 2^500 (fp64) or 2^60
// (fp32), nu and lam finite and small. Then no cell candidate can be NaN or
// negative-signed, the DP min is order-free and exact symmetry allows
// swapping the pair. Otherwise the NaN-exact compare chain is used.
// ---------------------------------------------------------------------------
// tiny > 0 (values): nonzero |x| < tiny also counts as unsafe. fp32: the
// kernels take the square root with flush-to-zero (sqrt.approx.ftz) on the
// safe path; with every nonzero |x| >= 2^-30 a nonzero sum of squared
// differences is >= 2^-106, far above the fp32 denormal range. fp64 (tiny =
// 2^-400): a nonzero sum is >= 2^-904, inside the branch-free sqrt's range
// (twb_device.cuh sqrt_fast0).
template <typename T>
__global__ void unsafe_kernel(const T* __restrict__ x, int64_t n, double limit, double tiny,
                              int* flag) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double a = fabs((double)x[i]);
        bad |= !(a < limit) || (a != 0.0 && a < tiny);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <typename T>
__global__ void convert_kernel(const double* __restrict__ in, T* __restrict__ out, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = (T)in[i];
}

// Mirror the strict upper triangle into the lower one (engine.py:223-225).
// 32x32 tiles through shared memory so both the read and the write coalesce.
template <typename T>
__global__ void mirror_kernel(T* m, int64_t n) {
    __shared__ T tile[32][33];
    const int64_t bi = blockIdx.y, bj = blockIdx.x;  // tile (bi, bj) with bj > bi...
    if (bj < bi) return;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = bi * 32 + r, j = bj * 32 + tx;
        if (i < n && j < n) tile[r][tx] = m[i * n + j];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int64_t j = bj * 32 + r, i = bi * 32 + tx;  // write (j, i) = tile[tx][r]
        if (i < n && j < n && j > i) m[j * n + i] = tile[tx][r];
    }
}

// Vt[k * rows + r] = V[r * d + k] (the dim-major copy the runtime-d kernels
// read columns from), 32x32 tiles through shared memory.
template <typename R>
__global__ void transpose_kernel(const R* __restrict__ V, int64_t rows, int d, R* __restrict__ Vt) {
    __shared__ R tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int k0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t r = r0 + i;
        const int k = k0 + threadIdx.x;
        if (r < rows && k < d) tile[i][threadIdx.x] = V[r * d + k];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int k = k0 + i;
        const int64_t r = r0 + threadIdx.x;
        if (r < rows && k < d) Vt[k * rows + r] = tile[threadIdx.x][i];
    }
}

template <typename T>
int check_unsafe(const T* d, int64_t n, double limit, int* dflag, cudaStream_t st,
                 double tiny = 0.0) {
    if (n <= 0) return 0;
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 4096);
    unsafe_kernel<T><<<blocks, 256, 0, st>>>(d, n, limit, tiny, dflag);
    ++t_launches;
    return 0;
}

// The precompute of one or two segments (a pair's two series, or packed CSR
// lists) in one launch, fused with the input check when flag != null
// (twb_prepare.cuh). virt: value of the virtual row 0 of V -- 0 (the
// reference's layout) or +inf (the DP kernels' marker of a virtual column,
// LaneRows::COL0_BY_INF). Vt (optional): the dim-major copy for the
// runtime-d kernels, leading dimension ntot + nseries (every prepared row).
template <typename T, typename R, typename Z>
struct PrepIn {
    const T* v;
    const T* t;
    const int64_t* d_off;  // device offsets (null: uniform_n)
    int64_t nseries, ntot, uniform_n;
    R* V;
    R* Tm;
    Z* Del;
    R* Vt;
};
template <typename T, typename R, typename Z>
int prepare_fused(const PrepIn<T, R, Z>* in, int nseg, int dim, double nu, double lam, int degree,
                  cudaStream_t st, double virt, int* flag, double limit, double tiny) {
    PrepArgs<T, R, Z> a{};
    int64_t tiles = 0;
    for (int k = 0; k < nseg; ++k) {
        PrepSeg<T, R, Z>& g = a.seg[k];
        g.v = in[k].v;
        g.t = in[k].t;
        g.off = in[k].d_off;
        g.nseries = in[k].nseries;
        g.ntot = in[k].ntot;
        g.uniform_n = in[k].uniform_n;
        g.V = in[k].V;
        g.Tm = in[k].Tm;
        g.Del = in[k].Del;
        g.Vt = in[k].Vt;
        g.ldt = in[k].ntot + in[k].nseries;
        g.tiles = (in[k].ntot + PREP_TILE * PREP_SPT - 1) / (PREP_TILE * PREP_SPT);
        tiles += g.tiles;
    }
    a.nseg = nseg;
    a.d = dim;
    a.nu = nu;
    a.lam = lam;
    a.p = degree;
    a.virt = virt;
    a.flag = flag;
    a.limit = limit;
    a.tiny = tiny;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    a.staged = dim <= PREP_DMAX && (size_t)(PREP_TILE * PREP_SPT + 1) * dim * sizeof(T) + 32 <= 160 * 1024;
    const size_t smem = a.staged ? (size_t)(PREP_TILE * PREP_SPT + 1) * dim * sizeof(T) + 32 : 0;
    // 8 CTAs of 256 threads per SM (the thread limit) while the staging fits:
    // each keeps one tile's bulk loads in flight
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms * 8));
    auto go = [&](auto kern) -> int {
        // static staging (times, ~8 KB) + dynamic: opt in above 32 KB of dynamic
        if (smem > 32 * 1024)
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<(unsigned)grid, PREP_TILE, smem, st>>>(a);
        ++t_launches;
        CK(cudaGetLastError());
        return 0;
    };
    switch (dim) {
        case 1: return go(prepare_kernel<T, R, Z, 1>);
        case 2: return go(prepare_kernel<T, R, Z, 2>);
        case 3: return go(prepare_kernel<T, R, Z, 3>);
        case 4: return go(prepare_kernel<T, R, Z, 4>);
    }
    return go(prepare_kernel<T, R, Z, 0>);
}
template <typename T, typename R, typename Z>
int prepare(const T* values, const T* times, const int64_t* d_off, int64_t nseries, int64_t ntot,
            int64_t uniform_n, int dim, double nu, double lam, int degree, R* V, R* Tm, Z* Del,
            cudaStream_t st, double virt = HUGE_VAL, R* Vt = nullptr) {
    const PrepIn<T, R, Z> in{values, times, d_off, nseries, ntot, uniform_n, V, Tm, Del, Vt};
    return prepare_fused<T, R, Z>(&in, 1, dim, nu, lam, degree, st, virt, nullptr, 0.0, 0.0);
}

// Launch bookkeeping for the next main-kernel launch: counts every launch
// and, in timing mode, brackets it with events (read by twb_last_kernel_ms).
LaunchCtx* ctx_begin() {
    t_launches += t_ctx.launches;
    t_ctx.launches = 0;
    t_ctx.timing = t_timing;
    if (t_timing && !t_ctx.ev0) {
        cudaEventCreate(&t_ctx.ev0);
        cudaEventCreate(&t_ctx.ev1);
    }
    return &t_ctx;
}

// Dimensions 1..4 have compile-time kernels; any other d (and every d with
// TWB_FORCE_DYN=1, a test hook) runs the runtime-d kernels (D == 0).
bool use_dyn(int dim) {
    static const bool force = getenv("TWB_FORCE_DYN") && atoi(getenv("TWB_FORCE_DYN")) != 0;
    return dim > 4 || force;
}

template <typename R, typename Z>
cudaError_t call_wave(int dim, int P, bool E, bool N1, const WaveProblem<R, Z>& pr, Scratch& sc,
                      cudaStream_t st) {
    Alloc al{scratch_alloc, &sc};
    if (use_dyn(dim)) {
        WaveProblem<R, Z> p2 = pr;
        p2.dd = dim;
        return wave_d<0, R, Z>(P, E, N1, p2, al, st, ctx_begin());
    }
    switch (dim) {
        case 1: return wave_d<1, R, Z>(P, E, N1, pr, al, st, ctx_begin());
        case 2: return wave_d<2, R, Z>(P, E, N1, pr, al, st, ctx_begin());
        case 3: return wave_d<3, R, Z>(P, E, N1, pr, al, st, ctx_begin());
        case 4: return wave_d<4, R, Z>(P, E, N1, pr, al, st, ctx_begin());
    }
    return cudaErrorInvalidValue;
}

template <typename R, typename Z>
cudaError_t call_batch(int dim, int P, bool E, bool N1, const BatchArgs<R, Z>& a, int64_t max_rows,
                       Scratch& sc, cudaStream_t st) {
    Alloc al{scratch_alloc, &sc};
    if (use_dyn(dim)) {
        BatchArgs<R, Z> a2 = a;
        a2.dd = dim;
        return batch_d<0, R, Z>(P, E, N1, a2, max_rows, al, st, ctx_begin());
    }
    switch (dim) {
        case 1: return batch_d<1, R, Z>(P, E, N1, a, max_rows, al, st, ctx_begin());
        case 2: return batch_d<2, R, Z>(P, E, N1, a, max_rows, al, st, ctx_begin());
        case 3: return batch_d<3, R, Z>(P, E, N1, a, max_rows, al, st, ctx_begin());
        case 4: return batch_d<4, R, Z>(P, E, N1, a, max_rows, al, st, ctx_begin());
    }
    return cudaErrorInvalidValue;
}

int check_params(int64_t nA, int64_t nB, int dim, double nu, double lam, int degree) {
    if (nA < 1 || nB < 1) return fail(TWB_EINVAL, "a time series needs at least one sample");
    if (dim < 1) return fail(TWB_EINVAL, "samples need at least one component");
    if (!(nu >= 0)) return fail(TWB_EINVAL, "nu must be >= 0, got %g", nu);
    if (!(lam >= 0)) return fail(TWB_EINVAL, "lam must be >= 0, got %g", lam);
    if (degree < 1) return fail(TWB_EINVAL, "degree must be a positive integer, got %d", degree);
    return 0;
}

// Kernel variant flags from the parameters and the input check.
struct Variant {
    int P;
    bool E, N1;
};
Variant pick_variant(int dim, int degree, double nu, double lam, bool unsafe_inputs, double limit) {
    Variant v;
    v.P = dim == 1 ? 2 : (degree <= 2 ? degree : 0);
    bool params_ok = std::isfinite(nu) && std::isfinite(lam) && nu < limit && lam < limit;
    v.E = unsafe_inputs || !params_ok || v.P == 0;
    v.N1 = !v.E && nu == 1.0;
    return v;
}

// Values below the limit keep every sum of squared differences finite and,
// in fp64, inside the branch-free square root's range (<= 2^1004): d terms of
// (2 * limit)^2 each, so the limit shrinks with d above 4.
template <typename T>
double safe_limit(int dim = 1) {
    double lim = sizeof(T) == 8 ? 0x1p500 : 0x1p60;
    for (int d = 4; d < dim; d *= 4) lim *= 0.5;
    return lim;
}
template <typename R>
constexpr double safe_tiny() {
    return sizeof(R) == 8 ? 0x1p-400 : 0x1p-30;
}

// ---------------------------------------------------------------------------
// Single pair. Inputs are device pointers (raw samples); out is a device
// pointer to one double.
// ---------------------------------------------------------------------------
template <typename T, typename R, typename Z>
int twed_pair_dev(const T* dA, int64_t nA, const T* dTA, const T* dB, int64_t nB, const T* dTB,
                  int dim, double nu, double lam, int degree, cudaStream_t st, double* d_out) {
    init_pool_current();
    Scratch sc(st);
    int* dflag = sc.get_n<int>(1);
    if (sc.failed) return fail(TWB_ENOMEM, "device scratch allocation failed");
    CK(cudaMemsetAsync(dflag, 0, sizeof(int), st));
    const double lim = safe_limit<R>(dim);

    const bool dyn = use_dyn(dim);
    R* V[2] = {sc.get_n<R>((nA + 1) * dim), sc.get_n<R>((nB + 1) * dim)};
    R* Tm[2] = {sc.get_n<R>(nA + 1), sc.get_n<R>(nB + 1)};
    Z* Del[2] = {sc.get_n<Z>(nA + 1), sc.get_n<Z>(nB + 1)};
    R* Vt[2] = {nullptr, nullptr};
    if (dyn) {
        Vt[0] = sc.get_n<R>((nA + 1) * dim);
        Vt[1] = sc.get_n<R>((nB + 1) * dim);
    }
    Z* zout = sc.get_n<Z>(1);
    if (sc.failed) return fail(TWB_ENOMEM, "device scratch allocation failed");
    int rc;
    {  // both series and the input check in one launch
        const PrepIn<T, R, Z> in[2] = {{dA, dTA, nullptr, 1, nA, nA, V[0], Tm[0], Del[0], Vt[0]},
                                       {dB, dTB, nullptr, 1, nB, nB, V[1], Tm[1], Del[1], Vt[1]}};
        if ((rc = prepare_fused<T, R, Z>(in, 2, dim, nu, lam, degree, st, HUGE_VAL, dflag, lim,
                                         safe_tiny<R>())))
            return rc;
    }
    const int64_t ldt[2] = {nA + 1, nB + 1};
    // No host round trip: the data-dependent choice between the proven-safe
    // sweep and the NaN-exact one is made on the device. Both are launched,
    // gated on the check's flag; the one not wanted returns at once. The call
    // stays asynchronous on the caller's stream (and capturable in a CUDA
    // graph). The safe sweep goes last so kernel timing brackets it.
    auto sweep = [&](const Variant& v, const int* gate, int want) -> int {
        // Rows = the longer series (more stripes for the SMs). Exact symmetry
        // twed(a,b) == twed(b,a) makes the swap bit-identical when the min is
        // order-free (not in the NaN-exact mode).
        int ra = 0, rb = 1;
        int64_t na = nA, nb = nB;
        if (!v.E && nB > nA && !getenv("TWB_NO_SWAP")) {  // env: tuning experiments
            ra = 1;
            rb = 0;
            std::swap(na, nb);
        }
        WaveProblem<R, Z> pr;
        pr.A = {V[ra], Tm[ra], Del[ra], Vt[ra], ldt[ra]};
        pr.B = {V[rb], Tm[rb], Del[rb], Vt[rb], ldt[rb]};
        pr.nA = na;
        pr.nB = nb;
        pr.nu = nu;
        pr.p = degree;
        pr.out = zout;
        pr.gate = gate;
        pr.gate_want = want;
        // The sweep's boundary rows come from their own scratch, returned to
        // the stream-ordered pool right after the launch: the gated sweep that
        // follows on the same stream reuses the same memory (one set of
        // boundary rows per call, not two).
        Scratch wsc(st);
        CK(call_wave<R, Z>(dim, v.P, v.E, v.N1, pr, wsc, st));
        if (wsc.failed) return fail(TWB_ENOMEM, "device scratch allocation failed");
        return 0;
    };
    const Variant v_safe = pick_variant(dim, degree, nu, lam, false, lim);
    if (v_safe.E) {  // parameters alone rule the safe sweep out
        if ((rc = sweep(v_safe, nullptr, 0))) return rc;
    } else {
        if ((rc = sweep(pick_variant(dim, degree, nu, lam, true, lim), dflag, 1))) return rc;
        if ((rc = sweep(v_safe, dflag, 0))) return rc;
    }
    static_assert(sizeof(Z) == 8, "pairs accumulate in fp64");
    CK(cudaMemcpyAsync(d_out, zout, sizeof(double), cudaMemcpyDeviceToDevice, st));
    return 0;
}

template <typename T>
int twed_pair_host(const T* A, int64_t nA, const T* TA, const T* B, int64_t nB, const T* TB,
                   int dim, double nu, double lam, int degree, int device, double* out) {
    int rc = check_params(nA, nB, dim, nu, lam, degree);
    if (rc) return rc;
    if (!A || !TA || !B || !TB || !out) return fail(TWB_EINVAL, "null pointer argument");
    DeviceGuard device_guard;
    CK(cudaSetDevice(device));
    init_pool(device);
    cudaStream_t st = cudaStreamPerThread;
    Scratch sc(st);
    T* dA = sc.get_n<T>(nA * dim);
    T* dTA = sc.get_n<T>(nA);
    T* dB = sc.get_n<T>(nB * dim);
    T* dTB = sc.get_n<T>(nB);
    double* dout = sc.get_n<double>(1);
    if (sc.failed) return fail(TWB_ENOMEM, "device allocation failed");
    CK(cudaMemcpyAsync(dA, A, sizeof(T) * nA * dim, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dTA, TA, sizeof(T) * nA, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dB, B, sizeof(T) * nB * dim, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dTB, TB, sizeof(T) * nB, cudaMemcpyHostToDevice, st));
    if constexpr (sizeof(T) == 8)
        rc = twed_pair_dev<T, double, double>(dA, nA, dTA, dB, nB, dTB, dim, nu, lam, degree, st, dout);
    else
        rc = twed_pair_dev<T, float, double>(dA, nA, dTA, dB, nB, dTB, dim, nu, lam, degree, st, dout);
    if (rc) return rc;
    CK(cudaMemcpyAsync(out, dout, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return 0;
}

// ---------------------------------------------------------------------------
// One pair on several devices: the wavefront's ring of
// CTAs spans one kernel per device; every part holds the prepared series, the
// stripes go round-robin over the whole ring, and the last CTA of each part
// writes its bottom row straight into the next part's inbox (peer memory over
// NVLink, system-scope release/acquire on the progress counter). A device may
// appear more than once (several kernels on one GPU, each on its own stream):
// the same protocol on one GPU, which is how it is tested here.
// ---------------------------------------------------------------------------
template <typename T>
int twed_pair_multi(const T* A, int64_t nA, const T* TA, const T* B, int64_t nB, const T* TB,
                    int dim, double nu, double lam, int degree, const int32_t* devices,
                    int32_t ndev, double* out) {
    using R = T;
    using Z = double;
    int rc = check_params(nA, nB, dim, nu, lam, degree);
    if (rc) return rc;
    if (!A || !TA || !B || !TB || !out || !devices) return fail(TWB_EINVAL, "null pointer argument");
    if (ndev < 1 || ndev > 64) return fail(TWB_EINVAL, "ndev must be in [1, 64], got %d", ndev);
    DeviceGuard device_guard;
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    for (int q = 0; q < ndev; ++q)
        if (devices[q] < 0 || devices[q] >= count)
            return fail(TWB_EINVAL, "device %d out of range (%d devices)", devices[q], count);
    // the producer part q writes into part q+1's memory
    for (int q = 0; q < ndev; ++q) {
        const int a = devices[q], b = devices[(q + 1) % ndev];
        if (a == b) continue;
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, a, b));
        if (!ok) return fail(TWB_EUNSUP, "device %d cannot access device %d (no peer access)", a, b);
        CK(cudaSetDevice(a));
        cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) return fail(TWB_ECUDA, "enable peer access %d -> %d: %s", a, b, cudaGetErrorString(e));
    }
    struct Part {
        int dev;
        cudaStream_t st = nullptr;
        Scratch* sc = nullptr;
        R* V[2];
        R* Tm[2];
        Z* Del[2];
        R* Vt[2] = {nullptr, nullptr};
        Z* zout;
        int* dflag;
    };
    std::vector<Part> parts(ndev);
    int* abort_flag = nullptr;
    auto cleanup = [&]() {
        for (Part& q : parts) {
            if (!q.st) continue;
            cudaSetDevice(q.dev);
            cudaStreamSynchronize(q.st);
            delete q.sc;
            cudaStreamSynchronize(q.st);
            cudaStreamDestroy(q.st);
        }
        if (abort_flag) cudaFreeHost(abort_flag);
    };
    struct Guard {
        std::function<void()> f;
        ~Guard() { f(); }
    } guard{cleanup};
    const double lim = safe_limit<R>(dim);
    const bool dyn = use_dyn(dim);
    const int64_t ldt[2] = {nA + 1, nB + 1};
    for (int q = 0; q < ndev; ++q) {
        Part& pt = parts[q];
        pt.dev = devices[q];
        CK(cudaSetDevice(pt.dev));
        init_pool(pt.dev);
        CK(cudaStreamCreateWithFlags(&pt.st, cudaStreamNonBlocking));
        pt.sc = new Scratch(pt.st);
        Scratch& sc = *pt.sc;
        T* dA = sc.get_n<T>(nA * dim);
        T* dTA = sc.get_n<T>(nA);
        T* dB = sc.get_n<T>(nB * dim);
        T* dTB = sc.get_n<T>(nB);
        pt.dflag = sc.get_n<int>(1);
        pt.V[0] = sc.get_n<R>((nA + 1) * dim);
        pt.V[1] = sc.get_n<R>((nB + 1) * dim);
        pt.Tm[0] = sc.get_n<R>(nA + 1);
        pt.Tm[1] = sc.get_n<R>(nB + 1);
        pt.Del[0] = sc.get_n<Z>(nA + 1);
        pt.Del[1] = sc.get_n<Z>(nB + 1);
        if (dyn) {
            pt.Vt[0] = sc.get_n<R>((nA + 1) * dim);
            pt.Vt[1] = sc.get_n<R>((nB + 1) * dim);
        }
        pt.zout = sc.get_n<Z>(1);
        if (sc.failed) return fail(TWB_ENOMEM, "device allocation failed on device %d", pt.dev);
        CK(cudaMemcpyAsync(dA, A, sizeof(T) * nA * dim, cudaMemcpyHostToDevice, pt.st));
        CK(cudaMemcpyAsync(dTA, TA, sizeof(T) * nA, cudaMemcpyHostToDevice, pt.st));
        CK(cudaMemcpyAsync(dB, B, sizeof(T) * nB * dim, cudaMemcpyHostToDevice, pt.st));
        CK(cudaMemcpyAsync(dTB, TB, sizeof(T) * nB, cudaMemcpyHostToDevice, pt.st));
        CK(cudaMemsetAsync(pt.dflag, 0, sizeof(int), pt.st));
        const PrepIn<T, R, Z> in[2] = {
            {dA, dTA, nullptr, 1, nA, nA, pt.V[0], pt.Tm[0], pt.Del[0], pt.Vt[0]},
            {dB, dTB, nullptr, 1, nB, nB, pt.V[1], pt.Tm[1], pt.Del[1], pt.Vt[1]}};
        if ((rc = prepare_fused<T, R, Z>(in, 2, dim, nu, lam, degree, pt.st, HUGE_VAL, pt.dflag, lim,
                                         safe_tiny<R>())))
            return rc;
    }
    int hflag = 0;
    CK(cudaSetDevice(parts[0].dev));
    CK(cudaMemcpyAsync(&hflag, parts[0].dflag, sizeof(int), cudaMemcpyDeviceToHost, parts[0].st));
    CK(cudaStreamSynchronize(parts[0].st));
    Variant v = pick_variant(dim, degree, nu, lam, hflag != 0, lim);
    int ra = 0, rb = 1;
    int64_t na = nA, nb = nB;
    if (!v.E && nB > nA) {  // rows = the longer series (exact symmetry, safe mode)
        ra = 1;
        rb = 0;
        std::swap(na, nb);
    }
    CK(cudaHostAlloc((void**)&abort_flag, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
    *abort_flag = 0;
    std::vector<WavePart<R, Z>> wp(ndev);
    for (int q = 0; q < ndev; ++q) {
        Part& pt = parts[q];
        CK(cudaStreamSynchronize(pt.st));  // inputs prepared on every part
        wp[q] = WavePart<R, Z>{pt.dev, pt.st, {pt.V[ra], pt.Tm[ra], pt.Del[ra], pt.Vt[ra], ldt[ra]},
                               {pt.V[rb], pt.Tm[rb], pt.Del[rb], pt.Vt[rb], ldt[rb]}, pt.zout,
                               Alloc{scratch_alloc, pt.sc}};
    }
    long long timeout_ms = 20000;
    if (const char* env = getenv("TWB_RING_TIMEOUT_MS")) timeout_ms = atoll(env);
    CtaRing<R, Z> ring{ndev, wp.data(), abort_flag, timeout_ms * 1000000LL};
    WaveProblem<R, Z> pr;
    pr.A = wp[0].A;
    pr.B = wp[0].B;
    pr.nA = na;
    pr.nB = nb;
    pr.nu = nu;
    pr.p = degree;
    pr.out = wp[0].out;
    pr.ring = &ring;
    CK(cudaSetDevice(parts[0].dev));
    CK(call_wave<R, Z>(dim, v.P, v.E, v.N1, pr, *parts[0].sc, parts[0].st));
    for (Part& pt : parts) {
        CK(cudaSetDevice(pt.dev));
        CK(cudaStreamSynchronize(pt.st));
        if (pt.sc->failed) return fail(TWB_ENOMEM, "device scratch allocation failed on device %d", pt.dev);
    }
    if (*(volatile int*)abort_flag)
        return fail(TWB_ECUDA, "multi-device sweep aborted: a stripe waited %lld ms for its producer "
                    "(kernels of the ring not co-resident?)", timeout_ms);
    if (ring.owner < 0) return fail(TWB_ECUDA, "multi-device sweep: no owner of the last stripe");
    const Part& own = parts[ring.owner];
    CK(cudaSetDevice(own.dev));
    CK(cudaMemcpyAsync(out, own.zout, sizeof(double), cudaMemcpyDeviceToHost, own.st));
    CK(cudaStreamSynchronize(own.st));
    return 0;
}

// ---------------------------------------------------------------------------
// All-pairs matrix (engine.py:183-226). Device inputs, host offsets, device
// output block (row_end - row_begin) x nBB of type O.
// ---------------------------------------------------------------------------
constexpr int64_t BATCH_ROWS_MAX = 32 * BATCH_KMAX;  // row-side length of the warp kernel

template <typename T, typename R, typename Z, typename O>
int twed_batch_dev_impl(const T* dAA, const int64_t* a_off, int64_t nAA, const T* dTAA,
                        const T* dBB, const int64_t* b_off, int64_t nBB, const T* dTBB, int dim,
                        double nu, double lam, int degree, int tri, int64_t row_begin,
                        int64_t row_end, cudaStream_t st, O* d_out) {
    const bool self = dBB == nullptr;
    if (self) {
        dBB = dAA;
        dTBB = dTAA;
        b_off = a_off;
        nBB = nAA;
    }
    const int64_t nrows = row_end - row_begin;
    Scratch sc(st);
    // prepared offsets on the host
    std::vector<int64_t> a_poff(nAA + 1), b_poff(nBB + 1);
    int64_t amax = 0, bmax = 0;
    for (int64_t k = 0; k <= nAA; ++k) a_poff[k] = a_off[k] + k;
    for (int64_t k = 0; k <= nBB; ++k) b_poff[k] = b_off[k] + k;
    for (int64_t k = 0; k < nAA; ++k) amax = std::max(amax, a_off[k + 1] - a_off[k]);
    for (int64_t k = 0; k < nBB; ++k) bmax = std::max(bmax, b_off[k + 1] - b_off[k]);
    auto uniform = [](const int64_t* off, int64_t n) -> int64_t {
        int64_t len = off[1] - off[0];
        for (int64_t k = 1; k < n; ++k)
            if (off[k + 1] - off[k] != len) return 0;
        return len;
    };
    const int64_t totA = a_off[nAA], totB = b_off[nBB];

    int* dflag = sc.get_n<int>(1);
    int64_t* d_aoff = sc.get_n<int64_t>(nAA + 1);
    int64_t* d_boff = sc.get_n<int64_t>(nBB + 1);
    int64_t* d_apoff = sc.get_n<int64_t>(nAA + 1);
    int64_t* d_bpoff = sc.get_n<int64_t>(nBB + 1);
    R* VA = sc.get_n<R>((totA + nAA) * dim);
    R* TmA = sc.get_n<R>(totA + nAA);
    Z* DelA = sc.get_n<Z>(totA + nAA);
    R *VB = VA, *TmB = TmA;
    Z* DelB = DelA;
    if (!self) {
        VB = sc.get_n<R>((totB + nBB) * dim);
        TmB = sc.get_n<R>(totB + nBB);
        DelB = sc.get_n<Z>(totB + nBB);
    }
    // runtime-d kernels read the columns (the B side) dim-major
    R* VtB = use_dyn(dim) ? sc.get_n<R>((totB + nBB) * dim) : nullptr;
    [[maybe_unused]] const int64_t ldtB = totB + nBB;
    if (sc.failed) return fail(TWB_ENOMEM, "device scratch allocation failed");
    CK(cudaMemsetAsync(dflag, 0, sizeof(int), st));
    CK(cudaMemcpyAsync(d_aoff, a_off, sizeof(int64_t) * (nAA + 1), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_apoff, a_poff.data(), sizeof(int64_t) * (nAA + 1), cudaMemcpyHostToDevice, st));
    if (!self) {
        CK(cudaMemcpyAsync(d_boff, b_off, sizeof(int64_t) * (nBB + 1), cudaMemcpyHostToDevice, st));
    }
    CK(cudaMemcpyAsync(d_bpoff, b_poff.data(), sizeof(int64_t) * (nBB + 1), cudaMemcpyHostToDevice, st));
    const double lim = safe_limit<R>(dim);
    int rc;
    {  // both lists and the input check in one launch
        const PrepIn<T, R, Z> in[2] = {
            {dAA, dTAA, d_aoff, nAA, totA, uniform(a_off, nAA), VA, TmA, DelA, self ? VtB : nullptr},
            {dBB, dTBB, d_boff, nBB, totB, uniform(b_off, nBB), VB, TmB, DelB, VtB}};
        if ((rc = prepare_fused<T, R, Z>(in, self ? 1 : 2, dim, nu, lam, degree, st, HUGE_VAL, dflag,
                                         lim, safe_tiny<R>())))
            return rc;
    }
    int hflag = 0;
    CK(cudaMemcpyAsync(&hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));

    // Output block: the kernel writes only solved entries (+ mirror).
    const bool mirror = tri && row_begin == 0 && row_end == nAA;
    Z* zout = nullptr;
    if constexpr (std::is_same<Z, O>::value) {
        zout = d_out;
    } else {
        zout = sc.get_n<Z>((size_t)nrows * nBB);
        if (sc.failed) return fail(TWB_ENOMEM, "device scratch allocation failed");
    }
    CK(cudaMemsetAsync(zout, 0, sizeof(Z) * (size_t)nrows * nBB, st));

    // Task decomposition: rows short enough for the warp kernel get chunks of
    // `chunk` B series; longer rows are solved pair by pair (wave kernel).
    double avg_b = (double)totB / (double)nBB;
    int chunk = (int)std::lround(3072.0 / (avg_b + 1.0));
    chunk = std::max(1, std::min(chunk, MAX_CHUNK));
    // Rows longer than the warp kernel's reach go to the wavefront kernel; the
    // others are grouped 32/LW consecutive rows per warp (row groups, see
    // batch_kernel). A group's tasks cover the columns of its first row.
    std::vector<int64_t> long_rows;
    int64_t max_rows = 1;
    for (int64_t li = 0; li < nrows; ++li) {
        const int64_t na = a_off[row_begin + li + 1] - a_off[row_begin + li];
        if (na <= BATCH_ROWS_MAX) max_rows = std::max(max_rows, na);
        else long_rows.push_back(li);
    }
    const int64_t groups_per_warp = 32 / batch_lanes(max_rows);
    const int64_t ngroups = (nrows + groups_per_warp - 1) / groups_per_warp;
    std::vector<int64_t> prefix(ngroups + 1, 0);
    for (int64_t g = 0; g < ngroups; ++g) {
        bool any_short = false;
        for (int64_t li = g * groups_per_warp; li < std::min(nrows, (g + 1) * groups_per_warp); ++li)
            any_short |= a_off[row_begin + li + 1] - a_off[row_begin + li] <= BATCH_ROWS_MAX;
        const int64_t jfirst = tri ? row_begin + g * groups_per_warp : 0;
        const int64_t nt = any_short && nBB > jfirst ? (nBB - jfirst + chunk - 1) / chunk : 0;
        prefix[g + 1] = prefix[g] + nt;
    }
    CK(cudaStreamSynchronize(st));  // hflag (and the host vectors stay alive)
    const Variant v = pick_variant(dim, degree, nu, lam, hflag != 0, lim);

    if (prefix[ngroups] > 0) {
        int64_t* d_prefix = sc.get_n<int64_t>(ngroups + 1);
        unsigned long long* d_counter = sc.get_n<unsigned long long>(1);
        if (sc.failed) return fail(TWB_ENOMEM, "device scratch allocation failed");
        CK(cudaMemcpyAsync(d_prefix, prefix.data(), sizeof(int64_t) * (ngroups + 1),
                           cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(d_counter, 0, sizeof(unsigned long long), st));
        BatchArgs<R, Z> a;
        a.A = {VA, TmA, DelA};
        a.B = {VB, TmB, DelB, VtB, ldtB};
        a.a_poff = d_apoff;
        a.b_poff = d_bpoff;
        a.nBB = nBB;
        a.row_begin = row_begin;
        a.nrows = nrows;
        a.task_prefix = d_prefix;
        a.ngroups = ngroups;
        a.ntasks = prefix[ngroups];
        a.chunk = chunk;
        a.tri = tri;
        a.mirror = mirror;
        a.out = zout;
        a.ld = nBB;
        a.nu = nu;
        a.p = degree;
        a.counter = d_counter;
        CK(call_batch<R, Z>(dim, v.P, v.E, v.N1, a, max_rows, sc, st));
        if (sc.failed) return fail(TWB_ENOMEM, "device scratch allocation failed");
    }
    // Long row-side series: one wavefront solve per pair. A pair of a few
    // thousand samples fills only a CTA or two, so the pairs are spread over a
    // pool of streams and their (cooperative, small-grid) sweeps run side by
    // side; the pool joins back into the caller's stream.
    if (!long_rows.empty()) {
        if constexpr (!std::is_same<Z, double>::value) {
            // the wave kernel needs Z = double; Z = float is only selected when
            // every series is short
            return fail(TWB_EUNSUP, "internal: fp32 accumulator with long series");
        } else {
            int64_t npairs = 0;
            for (int64_t li : long_rows) npairs += nBB - (tri ? row_begin + li : 0);
            const int ns = (int)std::min<int64_t>(32, std::max<int64_t>(npairs, 1));
            std::vector<cudaStream_t> pool(ns, nullptr);
            cudaEvent_t fork = nullptr;
            auto release = [&]() {
                for (int k = 0; k < ns; ++k) {
                    if (!pool[k]) continue;
                    cudaEvent_t joined;
                    if (cudaEventCreateWithFlags(&joined, cudaEventDisableTiming) == cudaSuccess) {
                        cudaEventRecord(joined, pool[k]);
                        cudaStreamWaitEvent(st, joined, 0);
                        cudaEventDestroy(joined);
                    }
                    cudaStreamSynchronize(pool[k]);
                    cudaStreamDestroy(pool[k]);
                }
                if (fork) cudaEventDestroy(fork);
            };
            struct PoolGuard {
                std::function<void()> f;
                ~PoolGuard() { f(); }
            } pool_guard{release};
            CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
            CK(cudaEventRecord(fork, st));  // inputs prepared, zout allocated
            for (int k = 0; k < ns; ++k) {
                CK(cudaStreamCreateWithFlags(&pool[k], cudaStreamNonBlocking));
                CK(cudaStreamWaitEvent(pool[k], fork, 0));
            }
            int64_t q = 0;
            for (int64_t li : long_rows) {
                const int64_t i = row_begin + li;
                const int64_t jfirst = tri ? i : 0;
                for (int64_t j = jfirst; j < nBB; ++j, ++q) {
                    const int k = (int)(q % ns);
                    Scratch pair_sc(pool[k]);  // freed stream-ordered after the pair
                    WaveProblem<R, double> pr;
                    pr.A = {VA + a_poff[i] * dim, TmA + a_poff[i], DelA + a_poff[i]};
                    pr.B = {VB + b_poff[j] * dim, TmB + b_poff[j], DelB + b_poff[j],
                            VtB ? VtB + b_poff[j] : nullptr, ldtB};
                    pr.nA = a_off[i + 1] - a_off[i];
                    pr.nB = b_off[j + 1] - b_off[j];
                    pr.nu = nu;
                    pr.p = degree;
                    pr.out = zout + li * nBB + j;
                    CK(call_wave<R, double>(dim, v.P, v.E, v.N1, pr, pair_sc, pool[k]));
                    if (pair_sc.failed) return fail(TWB_ENOMEM, "device scratch allocation failed");
                    if (mirror && j != i)
                        CK(cudaMemcpyAsync(zout + j * nBB + i, zout + li * nBB + j, sizeof(double),
                                           cudaMemcpyDeviceToDevice, pool[k]));
                }
            }
        }
    }
    if constexpr (!std::is_same<Z, O>::value) {
        const int64_t n = nrows * nBB;
        int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
        convert_kernel<O><<<std::max(blocks, 1), 256, 0, st>>>((const double*)zout, d_out, n);
        ++t_launches;
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(st));  // scratch (host vectors) lifetime
    return 0;
}

int check_batch(const int64_t* a_off, int64_t nAA, const int64_t* b_off, int64_t nBB, int dim,
                double nu, double lam, int degree, int64_t row_begin, int64_t row_end) {
    if (!a_off || nAA < 1 || (b_off && nBB < 1)) return fail(TWB_EINVAL, "batch lists must be nonempty");
    // CSR offsets start at 0 (the packed arrays hold exactly off[n] samples)
    if (a_off[0] != 0 || (b_off && b_off[0] != 0))
        return fail(TWB_EINVAL, "CSR offsets must start at 0 (a_off[0] = %lld)", (long long)a_off[0]);
    for (int64_t k = 0; k < nAA; ++k)
        if (a_off[k + 1] - a_off[k] < 1) return fail(TWB_EINVAL, "a time series needs at least one sample");
    if (b_off)
        for (int64_t k = 0; k < nBB; ++k)
            if (b_off[k + 1] - b_off[k] < 1)
                return fail(TWB_EINVAL, "a time series needs at least one sample");
    if (row_begin < 0 || row_end > nAA || row_begin >= row_end)
        return fail(TWB_EINVAL, "row range [%lld, %lld) outside [0, %lld)", (long long)row_begin,
                    (long long)row_end, (long long)nAA);
    return check_params(1, 1, dim, nu, lam, degree);
}

template <typename T, typename O>
int twed_batch_dev(const T* dAA, const int64_t* a_off, int64_t nAA, const T* dTAA, const T* dBB,
                   const int64_t* b_off, int64_t nBB, const T* dTBB, int dim, double nu, double lam,
                   int degree, int tri, int64_t row_begin, int64_t row_end, cudaStream_t st,
                   O* d_out) {
    const bool self = dBB == nullptr;
    int rc = check_batch(a_off, nAA, self ? nullptr : b_off, nBB, dim, nu, lam, degree, row_begin,
                         row_end);
    if (rc) return rc;
    if (tri && !self) return fail(TWB_EINVAL, "symmetric=True requires both lists to be the same collection");
    if (!dAA || !dTAA || !d_out || (!self && (!dTBB || !b_off)))
        return fail(TWB_EINVAL, "null pointer argument");
    init_pool_current();
    if constexpr (sizeof(T) == 8) {
        return twed_batch_dev_impl<T, double, double, O>(dAA, a_off, nAA, dTAA, dBB, b_off, nBB,
                                                         dTBB, dim, nu, lam, degree, tri, row_begin,
                                                         row_end, st, d_out);
    } else {
        // fp32 mode: fp32 accumulator when every series is short (error grows
        // with the path length), fp64 accumulator otherwise.
        int64_t mx = 0;
        for (int64_t k = 0; k < nAA; ++k) mx = std::max(mx, a_off[k + 1] - a_off[k]);
        if (!self)
            for (int64_t k = 0; k < nBB; ++k) mx = std::max(mx, b_off[k + 1] - b_off[k]);
        if (mx <= 4096 / 2 && mx <= BATCH_ROWS_MAX)
            return twed_batch_dev_impl<T, float, float, O>(dAA, a_off, nAA, dTAA, dBB, b_off, nBB,
                                                           dTBB, dim, nu, lam, degree, tri,
                                                           row_begin, row_end, st, d_out);
        return twed_batch_dev_impl<T, float, double, O>(dAA, a_off, nAA, dTAA, dBB, b_off, nBB,
                                                        dTBB, dim, nu, lam, degree, tri, row_begin,
                                                        row_end, st, d_out);
    }
}

// A large result (cfg5: 400 MB) usually lands in freshly allocated host
// memory, whose first-touch page faults would otherwise be taken inside the
// device-to-host copy (cfg5 e2e 491 -> 428 ms). Two host threads take them
// while the kernels run; the caller waits on the future before its copies,
// which then overwrite every byte. TWB_PREFAULT=0 disables it.
constexpr size_t PREFAULT_MIN_BYTES = (size_t)64 << 20;
std::shared_future<void> prefault_async(void* out, size_t bytes) {
    static const bool on = !getenv("TWB_PREFAULT") || atoi(getenv("TWB_PREFAULT")) != 0;
    if (!on || bytes < PREFAULT_MIN_BYTES) {
        std::promise<void> done;
        done.set_value();
        return done.get_future().share();
    }
    return std::async(std::launch::async, [out, bytes]() {
               volatile char* p = reinterpret_cast<volatile char*>(out);
               const size_t half = bytes / 2 / 4096 * 4096;
               std::thread second([=]() {
                   for (size_t i = half; i < bytes; i += 4096) p[i] = 0;
               });
               for (size_t i = 0; i < half; i += 4096) p[i] = 0;
               second.join();
           }).share();
}

template <typename T, typename O>
int twed_batch_host(const T* AA, const int64_t* a_off, int64_t nAA, const T* TAA, const T* BB,
                    const int64_t* b_off, int64_t nBB, const T* TBB, int dim, double nu, double lam,
                    int degree, int tri, int64_t row_begin, int64_t row_end, int device, O* out) {
    const bool self = BB == nullptr;
    int rc = check_batch(a_off, nAA, self ? nullptr : b_off, nBB, dim, nu, lam, degree, row_begin,
                         row_end);
    if (rc) return rc;
    if (!AA || !TAA || !out || (!self && (!TBB || !b_off))) return fail(TWB_EINVAL, "null pointer argument");
    DeviceGuard device_guard;
    CK(cudaSetDevice(device));
    init_pool(device);
    cudaStream_t st = cudaStreamPerThread;
    Scratch sc(st);
    const int64_t totA = a_off[nAA];
    const int64_t totB = self ? 0 : b_off[nBB];
    const int64_t ncols = self ? nAA : nBB;
    T* dA = sc.get_n<T>(totA * dim);
    T* dTA = sc.get_n<T>(totA);
    T* dB = self ? nullptr : sc.get_n<T>(totB * dim);
    T* dTB = self ? nullptr : sc.get_n<T>(totB);
    O* dout = sc.get_n<O>((size_t)(row_end - row_begin) * ncols);
    if (sc.failed) return fail(TWB_ENOMEM, "device allocation failed");
    CK(cudaMemcpyAsync(dA, AA, sizeof(T) * totA * dim, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dTA, TAA, sizeof(T) * totA, cudaMemcpyHostToDevice, st));
    if (!self) {
        CK(cudaMemcpyAsync(dB, BB, sizeof(T) * totB * dim, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dTB, TBB, sizeof(T) * totB, cudaMemcpyHostToDevice, st));
    }
    const size_t out_bytes = sizeof(O) * (size_t)(row_end - row_begin) * ncols;
    std::shared_future<void> faulted = prefault_async(out, out_bytes);
    rc = twed_batch_dev<T, O>(dA, a_off, nAA, dTA, dB, b_off, nBB, dTB, dim, nu, lam, degree, tri,
                              row_begin, row_end, st, dout);
    if (rc) return rc;
    faulted.wait();
    CK(cudaMemcpyAsync(out, dout, out_bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return 0;
}

// ---------------------------------------------------------------------------
// All-pairs matrix over several devices in one call (SURVEY.md §8(b) C-ABI
// form `devices, ndev`; §8(e) sharding): contiguous row blocks balanced by
// work (pairs x row length; j >= i pairs for the triangle), one host thread
// per device, no collective. Each device writes its rows straight into the
// caller's matrix; for the triangle it also writes the mirror of its rows'
// upper part: the diagonal square is mirrored on the device and the strip
// right of it goes back transposed into the columns of its rows -- the
// reference's mirror (engine.py:223-225) without a host pass over the matrix.
// ---------------------------------------------------------------------------
// m (rows x ld, row-major): the square [0, n) x [c0, c0 + n) mirrored, upper
// -> lower (32x32 tiles through shared memory).
template <typename T>
__global__ void mirror_block_kernel(T* m, int64_t ld, int64_t c0, int64_t n) {
    __shared__ T tile[32][33];
    const int64_t bi = blockIdx.y, bj = blockIdx.x;
    if (bj < bi) return;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = bi * 32 + r, j = bj * 32 + tx;
        if (i < n && j < n) tile[r][tx] = m[i * ld + c0 + j];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int64_t j = bj * 32 + r, i = bi * 32 + tx;
        if (i < n && j < n && j > i) m[j * ld + c0 + i] = tile[tx][r];
    }
}
// dst (cols x rows) = transpose of src (rows x cols, leading dimension lds).
template <typename T>
__global__ void transpose_block_kernel(const T* __restrict__ src, int64_t lds, int64_t rows,
                                       int64_t cols, T* __restrict__ dst) {
    __shared__ T tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = src[r * lds + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) dst[c * rows + r] = tile[threadIdx.x][i];
    }
}

template <typename T, typename O>
int twed_batch_multi(const T* AA, const int64_t* a_off, int64_t nAA, const T* TAA, const T* BB,
                     const int64_t* b_off, int64_t nBB, const T* TBB, int dim, double nu, double lam,
                     int degree, int tri, const int32_t* devices, int32_t ndev, O* out) {
    const bool self = BB == nullptr;
    int rc = check_batch(a_off, nAA, self ? nullptr : b_off, nBB, dim, nu, lam, degree, 0, nAA);
    if (rc) return rc;
    if (tri && !self) return fail(TWB_EINVAL, "symmetric=True requires both lists to be the same collection");
    if (!AA || !TAA || !out || (!self && (!TBB || !b_off)) || !devices || ndev < 1)
        return fail(TWB_EINVAL, "null pointer argument or empty device list");
    int ndevs = 0;
    CK(cudaGetDeviceCount(&ndevs));
    for (int k = 0; k < ndev; ++k)
        if (devices[k] < 0 || devices[k] >= ndevs)
            return fail(TWB_EINVAL, "device %d out of range (%d devices)", devices[k], ndevs);
    const int64_t ncols = self ? nAA : nBB;
    if (ndev == 1)
        return twed_batch_host<T, O>(AA, a_off, nAA, TAA, BB, b_off, nBB, TBB, dim, nu, lam, degree,
                                     tri, 0, nAA, devices[0], out);
    // row blocks of equal work: row i costs len_i * (sum of its columns' lengths)
    const int64_t* coff = self ? a_off : b_off;
    std::vector<double> suffix(ncols + 1, 0.0);  // column lengths summed from j on
    for (int64_t j = ncols - 1; j >= 0; --j) suffix[j] = suffix[j + 1] + (double)(coff[j + 1] - coff[j]);
    std::vector<double> w(nAA + 1, 0.0);
    for (int64_t i = 0; i < nAA; ++i)
        w[i + 1] = w[i] + (double)(a_off[i + 1] - a_off[i]) * (tri ? suffix[i] : suffix[0]);
    std::vector<int64_t> lo(ndev + 1, 0);
    for (int k = 1; k < ndev; ++k) {
        const double target = w[nAA] * k / ndev;
        lo[k] = std::max(lo[k - 1], (int64_t)(std::lower_bound(w.begin(), w.end(), target) - w.begin()));
        lo[k] = std::min(lo[k], nAA);
    }
    lo[ndev] = nAA;
    std::vector<int> rcs(ndev, 0);
    std::vector<std::string> msgs(ndev);
    // every block's copies wait for the whole matrix to be faulted in (a
    // device also writes into other blocks' rows: the transposed strip)
    std::shared_future<void> faulted = prefault_async(out, sizeof(O) * (size_t)nAA * ncols);
    auto block = [&](int k) -> int {
        const int64_t r0 = lo[k], r1 = lo[k + 1];
        if (r1 <= r0) return 0;
        const int64_t rows = r1 - r0;
        CK(cudaSetDevice(devices[k]));
        init_pool(devices[k]);
        cudaStream_t st = cudaStreamPerThread;
        Scratch sc(st);
        const int64_t totA = a_off[nAA], totB = self ? 0 : b_off[nBB];
        T* dA = sc.get_n<T>(totA * dim);
        T* dTA = sc.get_n<T>(totA);
        T* dB = self ? nullptr : sc.get_n<T>(totB * dim);
        T* dTB = self ? nullptr : sc.get_n<T>(totB);
        O* dout = sc.get_n<O>((size_t)rows * ncols);
        const int64_t strip = tri ? ncols - r1 : 0;  // columns right of the diagonal square
        O* dtr = strip > 0 ? sc.get_n<O>((size_t)rows * strip) : nullptr;
        if (sc.failed) return fail(TWB_ENOMEM, "device allocation failed on device %d", devices[k]);
        CK(cudaMemcpyAsync(dA, AA, sizeof(T) * totA * dim, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dTA, TAA, sizeof(T) * totA, cudaMemcpyHostToDevice, st));
        if (!self) {
            CK(cudaMemcpyAsync(dB, BB, sizeof(T) * totB * dim, cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(dTB, TBB, sizeof(T) * totB, cudaMemcpyHostToDevice, st));
        }
        int rc2 = twed_batch_dev<T, O>(dA, a_off, nAA, dTA, dB, b_off, nBB, dTB, dim, nu, lam, degree,
                                       tri, r0, r1, st, dout);
        if (rc2) return rc2;
        faulted.wait();
        if (!tri) {
            CK(cudaMemcpyAsync(out + r0 * ncols, dout, sizeof(O) * (size_t)rows * ncols,
                               cudaMemcpyDeviceToHost, st));
        } else {
            // the diagonal square, mirrored on the device
            dim3 g1((unsigned)((rows + 31) / 32), (unsigned)((rows + 31) / 32));
            mirror_block_kernel<O><<<g1, dim3(32, 8), 0, st>>>(dout, ncols, r0, rows);
            ++t_launches;
            CK(cudaGetLastError());
            // rows r0..r1, columns r0.. (upper part + mirrored square)
            CK(cudaMemcpy2DAsync(out + r0 * ncols + r0, sizeof(O) * ncols, dout + r0,
                                 sizeof(O) * ncols, sizeof(O) * (ncols - r0), rows,
                                 cudaMemcpyDeviceToHost, st));
            if (strip > 0) {  // columns r1.. of these rows -> rows r1.. of columns r0..r1
                dim3 g2((unsigned)((strip + 31) / 32), (unsigned)((rows + 31) / 32));
                transpose_block_kernel<O><<<g2, dim3(32, 8), 0, st>>>(dout + r1, ncols, rows, strip, dtr);
                ++t_launches;
                CK(cudaGetLastError());
                CK(cudaMemcpy2DAsync(out + r1 * ncols + r0, sizeof(O) * ncols, dtr, sizeof(O) * rows,
                                     sizeof(O) * rows, strip, cudaMemcpyDeviceToHost, st));
            }
        }
        CK(cudaStreamSynchronize(st));
        return 0;
    };
    std::vector<std::thread> workers;
    for (int k = 0; k < ndev; ++k)
        workers.emplace_back([&, k]() {
            DeviceGuard guard;
            rcs[k] = block(k);
            if (rcs[k]) msgs[k] = t_err;
        });
    for (auto& t : workers) t.join();
    for (int k = 0; k < ndev; ++k)
        if (rcs[k]) return fail(rcs[k], "device %d: %s", devices[k], msgs[k].c_str());
    return 0;
}

template <typename T>
int mirror_dev(T* d, int64_t n, cudaStream_t st) {
    if (!d || n < 1) return fail(TWB_EINVAL, "bad matrix");
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
    mirror_kernel<T><<<grid, dim3(32, 8), 0, st>>>(d, n);
    ++t_launches;
    CK(cudaGetLastError());
    return 0;
}

// Pipe-throughput probe: independent add chains per thread, enough warps to
// saturate the pipe; returns lane-ops/s (one add = one op). This is the
// measured denominator of the ALU roofline (MEASURED_PEAKS.json only has HBM
// and bf16 tensor peaks).
template <typename T>
__global__ void add_probe_kernel(T* sink, int iters, T seed) {
    T a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
      a6 = a0 + 6, a7 = a0 + 7;
    const T inc = seed * (T)1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a0 += inc; a1 += inc; a2 += inc; a3 += inc; a4 += inc; a5 += inc; a6 += inc; a7 += inc;
        }
    }
    T r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (r == (T)-1) sink[0] = r;  // keep the chains alive
}

// sqrt_fast (twb_device.cuh) against __dsqrt_rn on hashed bit patterns: half
// uniform over every non-negative double (all exponents, denormals, inf, NaN),
// half uniform mantissas over exponents [2^-80, 2^80). Counts bit mismatches
// where sqrt_fast_ok holds, and how many inputs took the fast path.
__device__ __forceinline__ unsigned long long splitmix(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
__global__ void sqrt_check_kernel(int64_t n, unsigned long long seed, unsigned long long* bad,
                                  unsigned long long* fast) {
    unsigned long long nb = 0, nf = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        unsigned long long h = splitmix(seed ^ (unsigned long long)i);
        unsigned long long bits = h & 0x7fffffffffffffffull;
        if (i & 1) {
            const unsigned long long e = 0x3ff - 80 + ((h >> 52) % 160);
            bits = (e << 52) | (h & 0x000fffffffffffffull);
        }
        const double x = __longlong_as_double((long long)bits);
        if (sqrt_fast_ok(x)) {
            ++nf;
            nb += __double_as_longlong(sqrt_fast(x)) != __double_as_longlong(__dsqrt_rn(x));
        }
        // the K-wide form on the safe-mode domain {0} U [2^-904, 2^1004)
        // (twb_device.cuh sqrt_fast0_k), zero included in every vector
        const unsigned hx = (unsigned)(bits >> 32);
        const double xs = (hx >= 0x07700000u && hx < 0x7eb00000u) ? x : 1.0 + (double)(i & 1023);
        const double v[4] = {xs, 0.0, __dmul_rn(xs, 0.25), __dadd_rn(xs, 1.0)};
        double o[4];
        sqrt_fast0_k<4>(v, o);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            nb += __double_as_longlong(o[q]) != __double_as_longlong(__dsqrt_rn(v[q]));
    }
    atomicAdd(bad, nb);
    atomicAdd(fast, nf);
}

}  // namespace

// Hooks for the other translation units of the library (twb_lcs.cu): the
// thread-local error text, launch count and kernel-timing context.
namespace twb {
int api_fail(int code, const char* msg) { return fail(code, "%s", msg); }
void api_count_launch() { ++t_launches; }
LaunchCtx* api_ctx_begin() { return ctx_begin(); }
}  // namespace twb

// The single-pair precompute exactly as twb_twed_dev runs it (both series and
// the input check in one launch), into caller buffers: the DP kernels' layout
// (virtual row +inf). For timing and inspection of the HBM-bound precompute.
template <typename T, typename R>
int prepare_pair_dev(const T* A, const T* TA, int64_t nA, const T* B, const T* TB, int64_t nB,
                     int dim, double nu, double lam, int degree, R* VA, R* TmA, double* DelA, R* VB,
                     R* TmB, double* DelB, int* flag, void* stream) {
    int rc = check_params(nA, nB, dim, nu, lam, degree);
    if (rc) return rc;
    if (!A || !TA || !B || !TB || !VA || !TmA || !DelA || !VB || !TmB || !DelB || !flag)
        return fail(TWB_EINVAL, "null pointer argument");
    cudaStream_t st = (cudaStream_t)stream;
    const PrepIn<T, R, double> in[2] = {{A, TA, nullptr, 1, nA, nA, VA, TmA, DelA, nullptr},
                                        {B, TB, nullptr, 1, nB, nB, VB, TmB, DelB, nullptr}};
    CK(cudaMemsetAsync(flag, 0, sizeof(int), st));
    return prepare_fused<T, R, double>(in, 2, dim, nu, lam, degree, st, HUGE_VAL, flag,
                                       safe_limit<R>(dim), safe_tiny<R>());
}

extern "C" {

int64_t twb_selftest_sqrt(int64_t n, uint64_t seed, int32_t device, int64_t* fast_count) {
    if (n < 1) return fail(TWB_EINVAL, "n must be >= 1");
    DeviceGuard device_guard;
    CK(cudaSetDevice(device));
    cudaStream_t st = cudaStreamPerThread;
    unsigned long long* d = nullptr;
    CK(cudaMallocAsync(&d, 2 * sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), st));
    sqrt_check_kernel<<<148 * 8, 256, 0, st>>>(n, seed, d, d + 1);
    ++t_launches;
    CK(cudaGetLastError());
    unsigned long long h[2] = {0, 0};
    CK(cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(d, st));
    CK(cudaStreamSynchronize(st));
    if (fast_count) *fast_count = (int64_t)h[1];
    return (int64_t)h[0];
}

double twb_probe_add_rate(int fp64, int device) {
    DeviceGuard device_guard;
    if (cudaSetDevice(device) != cudaSuccess) return -1.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaStream_t st = cudaStreamPerThread;
    void* sink = nullptr;
    if (cudaMallocAsync(&sink, 16, st) != cudaSuccess) return -1.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, threads = 512, blocks = sms * 4;
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0, st);
        if (fp64) add_probe_kernel<double><<<blocks, threads, 0, st>>>((double*)sink, iters, 1.0);
        else add_probe_kernel<float><<<blocks, threads, 0, st>>>((float*)sink, iters, 1.0f);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(sink, st);
    cudaStreamSynchronize(st);
    if (cudaGetLastError() != cudaSuccess) return -1.0;
    const double ops = (double)blocks * threads * iters * 64.0;
    return ops / (best * 1e-3);
}

int twb_version(void) { return 200; }

int twb_trim_pool(int device) {
    cudaMemPool_t pool;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, device);
    if (e == cudaSuccess) e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemPoolTrimTo(pool, 0);
    cudaSetDevice(cur);
    if (e != cudaSuccess) return fail(TWB_ECUDA, "twb_trim_pool(%d): %s", device, cudaGetErrorString(e));
    return TWB_OK;
}

size_t twb_last_error(char* buf, size_t len) {
    if (buf && len) {
        size_t n = std::min(len - 1, t_err.size());
        memcpy(buf, t_err.data(), n);
        buf[n] = 0;
    }
    return t_err.size();
}

int twb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int64_t twb_take_launch_count(void) {
    int64_t n = t_launches + t_ctx.launches;
    t_launches = 0;
    t_ctx.launches = 0;
    return n;
}

void twb_set_kernel_timing(int enable) { t_timing = enable != 0; }

void twb_last_wave_shape(int64_t* stripes, int64_t* rows_per_stripe, int64_t* ctas) {
    if (stripes) *stripes = t_ctx.wave_stripes;
    if (rows_per_stripe) *rows_per_stripe = t_ctx.wave_rows;
    if (ctas) *ctas = t_ctx.wave_ctas;
}

float twb_last_kernel_ms(void) {
    if (!t_timing || !t_ctx.ev1) return -1.f;
    if (cudaEventSynchronize(t_ctx.ev1) != cudaSuccess) return -1.f;
    float ms = -1.f;
    if (cudaEventElapsedTime(&ms, t_ctx.ev0, t_ctx.ev1) != cudaSuccess) return -1.f;
    return ms;
}

int twb_twed_f64(const double* A, int64_t nA, const double* TA, const double* B, int64_t nB,
                 const double* TB, int32_t dim, double nu, double lam, int32_t degree,
                 int32_t device, double* out) {
    return twed_pair_host<double>(A, nA, TA, B, nB, TB, dim, nu, lam, degree, device, out);
}

int twb_twed_f32(const float* A, int64_t nA, const float* TA, const float* B, int64_t nB,
                 const float* TB, int32_t dim, double nu, double lam, int32_t degree,
                 int32_t device, double* out) {
    return twed_pair_host<float>(A, nA, TA, B, nB, TB, dim, nu, lam, degree, device, out);
}

int twb_twed_dev_f64(const double* dA, int64_t nA, const double* dTA, const double* dB, int64_t nB,
                     const double* dTB, int32_t dim, double nu, double lam, int32_t degree,
                     void* stream, double* d_out) {
    int rc = check_params(nA, nB, dim, nu, lam, degree);
    if (rc) return rc;
    if (!dA || !dTA || !dB || !dTB || !d_out) return fail(TWB_EINVAL, "null pointer argument");
    return twed_pair_dev<double, double, double>(dA, nA, dTA, dB, nB, dTB, dim, nu, lam, degree,
                                                 (cudaStream_t)stream, d_out);
}

int twb_twed_dev_f32(const float* dA, int64_t nA, const float* dTA, const float* dB, int64_t nB,
                     const float* dTB, int32_t dim, double nu, double lam, int32_t degree,
                     void* stream, double* d_out) {
    int rc = check_params(nA, nB, dim, nu, lam, degree);
    if (rc) return rc;
    if (!dA || !dTA || !dB || !dTB || !d_out) return fail(TWB_EINVAL, "null pointer argument");
    return twed_pair_dev<float, float, double>(dA, nA, dTA, dB, nB, dTB, dim, nu, lam, degree,
                                               (cudaStream_t)stream, d_out);
}

int twb_twed_multi_f64(const double* A, int64_t nA, const double* TA, const double* B, int64_t nB,
                       const double* TB, int32_t dim, double nu, double lam, int32_t degree,
                       const int32_t* devices, int32_t ndev, double* out) {
    return twed_pair_multi<double>(A, nA, TA, B, nB, TB, dim, nu, lam, degree, devices, ndev, out);
}

int twb_twed_multi_f32(const float* A, int64_t nA, const float* TA, const float* B, int64_t nB,
                       const float* TB, int32_t dim, double nu, double lam, int32_t degree,
                       const int32_t* devices, int32_t ndev, double* out) {
    return twed_pair_multi<float>(A, nA, TA, B, nB, TB, dim, nu, lam, degree, devices, ndev, out);
}

int twb_twed_batch_f64(const double* AA, const int64_t* a_off, int64_t nAA, const double* TAA,
                       const double* BB, const int64_t* b_off, int64_t nBB, const double* TBB,
                       int32_t dim, double nu, double lam, int32_t degree, int32_t tri,
                       int64_t row_begin, int64_t row_end, int32_t device, double* out) {
    return twed_batch_host<double, double>(AA, a_off, nAA, TAA, BB, b_off, nBB, TBB, dim, nu, lam,
                                           degree, tri, row_begin, row_end, device, out);
}

int twb_twed_batch_multi_f64(const double* AA, const int64_t* a_off, int64_t nAA, const double* TAA,
                             const double* BB, const int64_t* b_off, int64_t nBB, const double* TBB,
                             int32_t dim, double nu, double lam, int32_t degree, int32_t tri,
                             const int32_t* devices, int32_t ndev, double* out) {
    return twed_batch_multi<double, double>(AA, a_off, nAA, TAA, BB, b_off, nBB, TBB, dim, nu, lam,
                                            degree, tri, devices, ndev, out);
}
int twb_twed_batch_multi_f32(const float* AA, const int64_t* a_off, int64_t nAA, const float* TAA,
                             const float* BB, const int64_t* b_off, int64_t nBB, const float* TBB,
                             int32_t dim, double nu, double lam, int32_t degree, int32_t tri,
                             const int32_t* devices, int32_t ndev, float* out) {
    return twed_batch_multi<float, float>(AA, a_off, nAA, TAA, BB, b_off, nBB, TBB, dim, nu, lam,
                                          degree, tri, devices, ndev, out);
}

int twb_twed_batch_f32(const float* AA, const int64_t* a_off, int64_t nAA, const float* TAA,
                       const float* BB, const int64_t* b_off, int64_t nBB, const float* TBB,
                       int32_t dim, double nu, double lam, int32_t degree, int32_t tri,
                       int64_t row_begin, int64_t row_end, int32_t device, float* out) {
    return twed_batch_host<float, float>(AA, a_off, nAA, TAA, BB, b_off, nBB, TBB, dim, nu, lam,
                                         degree, tri, row_begin, row_end, device, out);
}

int twb_twed_batch_dev_f64(const double* dAA, const int64_t* a_off, int64_t nAA, const double* dTAA,
                           const double* dBB, const int64_t* b_off, int64_t nBB, const double* dTBB,
                           int32_t dim, double nu, double lam, int32_t degree, int32_t tri,
                           int64_t row_begin, int64_t row_end, void* stream, double* d_out) {
    return twed_batch_dev<double, double>(dAA, a_off, nAA, dTAA, dBB, b_off, nBB, dTBB, dim, nu, lam,
                                          degree, tri, row_begin, row_end, (cudaStream_t)stream,
                                          d_out);
}

int twb_twed_batch_dev_f32(const float* dAA, const int64_t* a_off, int64_t nAA, const float* dTAA,
                           const float* dBB, const int64_t* b_off, int64_t nBB, const float* dTBB,
                           int32_t dim, double nu, double lam, int32_t degree, int32_t tri,
                           int64_t row_begin, int64_t row_end, void* stream, float* d_out) {
    return twed_batch_dev<float, float>(dAA, a_off, nAA, dTAA, dBB, b_off, nBB, dTBB, dim, nu, lam,
                                        degree, tri, row_begin, row_end, (cudaStream_t)stream, d_out);
}

int twb_mirror_upper_dev_f64(double* d_out, int64_t n, void* stream) {
    return mirror_dev<double>(d_out, n, (cudaStream_t)stream);
}
int twb_mirror_upper_dev_f32(float* d_out, int64_t n, void* stream) {
    return mirror_dev<float>(d_out, n, (cudaStream_t)stream);
}

int twb_band_solve_f64(const double* va, const double* ta, const double* dela, int64_t na,
                       const double* vb, const double* tb, const double* delb, int64_t nb,
                       int32_t dim, double nu, int32_t degree, int32_t device, double* out) {
    int rc = check_params(na, nb, dim, nu, 0.0, degree);
    if (rc) return rc;
    if (!va || !ta || !dela || !vb || !tb || !delb || !out) return fail(TWB_EINVAL, "null pointer argument");
    DeviceGuard device_guard;
    CK(cudaSetDevice(device));
    init_pool(device);
    cudaStream_t st = cudaStreamPerThread;
    Scratch sc(st);
    double* d[6] = {sc.get_n<double>((na + 1) * dim), sc.get_n<double>(na + 1),
                    sc.get_n<double>(na + 1),         sc.get_n<double>((nb + 1) * dim),
                    sc.get_n<double>(nb + 1),         sc.get_n<double>(nb + 1)};
    double* dout = sc.get_n<double>(1);
    int* dflag = sc.get_n<int>(1);
    if (sc.failed) return fail(TWB_ENOMEM, "device allocation failed");
    const double* h[6] = {va, ta, dela, vb, tb, delb};
    const int64_t n[6] = {(na + 1) * dim, na + 1, na + 1, (nb + 1) * dim, nb + 1, nb + 1};
    for (int k = 0; k < 6; ++k)
        CK(cudaMemcpyAsync(d[k], h[k], sizeof(double) * n[k], cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(dflag, 0, sizeof(int), st));
    const double lim = safe_limit<double>(dim);
    for (int k = 0; k < 6; ++k) {
        const bool is_del = k == 2 || k == 5;  // del[0] = +inf by construction
        const bool is_val = k == 0 || k == 3;
        check_unsafe(d[k] + (is_del ? 1 : 0), n[k] - (is_del ? 1 : 0), lim, dflag, st,
                     is_val ? safe_tiny<double>() : 0.0);
    }
    // the DP kernels' copy marks the virtual row 0 with +inf (COL0_BY_INF)
    static const double infs[4] = {HUGE_VAL, HUGE_VAL, HUGE_VAL, HUGE_VAL};
    for (int k = 0; k < 2; ++k) {
        double* v0 = d[3 * k];
        for (int c = 0; c < dim; c += 4)
            CK(cudaMemcpyAsync(v0 + c, infs, sizeof(double) * std::min(4, dim - c),
                               cudaMemcpyHostToDevice, st));
    }
    double* vt[2] = {nullptr, nullptr};
    if (use_dyn(dim)) {
        vt[0] = sc.get_n<double>((na + 1) * dim);
        vt[1] = sc.get_n<double>((nb + 1) * dim);
        if (sc.failed) return fail(TWB_ENOMEM, "device allocation failed");
        for (int k = 0; k < 2; ++k) {
            const int64_t rows = k ? nb + 1 : na + 1;
            dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((dim + 31) / 32));
            transpose_kernel<double><<<grid, dim3(32, 8), 0, st>>>(d[3 * k], rows, dim, vt[k]);
            ++t_launches;
            CK(cudaGetLastError());
        }
    }
    int hflag = 0;
    CK(cudaMemcpyAsync(&hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const Variant v = pick_variant(dim, degree, nu, 0.0, hflag != 0, lim);
    WaveProblem<double, double> pr;
    pr.A = {d[0], d[1], d[2], vt[0], na + 1};
    pr.B = {d[3], d[4], d[5], vt[1], nb + 1};
    pr.nA = na;
    pr.nB = nb;
    if (!v.E && nb > na) {
        std::swap(pr.A, pr.B);
        std::swap(pr.nA, pr.nB);
    }
    pr.nu = nu;
    pr.p = degree;
    pr.out = dout;
    CK(call_wave<double, double>(dim, v.P, v.E, v.N1, pr, sc, st));
    if (sc.failed) return fail(TWB_ENOMEM, "device scratch allocation failed");
    CK(cudaMemcpyAsync(out, dout, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return 0;
}

int twb_prepare_pair_dev_f64(const double* A, const double* TA, int64_t nA, const double* B,
                             const double* TB, int64_t nB, int32_t dim, double nu, double lam,
                             int32_t degree, double* VA, double* TmA, double* DelA, double* VB,
                             double* TmB, double* DelB, int32_t* unsafe_flag, void* stream) {
    return prepare_pair_dev<double, double>(A, TA, nA, B, TB, nB, dim, nu, lam, degree, VA, TmA,
                                            DelA, VB, TmB, DelB, unsafe_flag, stream);
}
int twb_prepare_pair_dev_f32(const float* A, const float* TA, int64_t nA, const float* B,
                             const float* TB, int64_t nB, int32_t dim, double nu, double lam,
                             int32_t degree, float* VA, float* TmA, double* DelA, float* VB,
                             float* TmB, double* DelB, int32_t* unsafe_flag, void* stream) {
    return prepare_pair_dev<float, float>(A, TA, nA, B, TB, nB, dim, nu, lam, degree, VA, TmA,
                                          DelA, VB, TmB, DelB, unsafe_flag, stream);
}

int twb_prepare_series_f64(const double* values, const double* times, int64_t n, int32_t dim,
                           double nu, double lam, int32_t degree, int32_t device, double* ext_values,
                           double* ext_times, double* deletion) {
    if (n < 1 || dim < 1 || degree < 1) return fail(TWB_EINVAL, "bad series");
    DeviceGuard device_guard;
    CK(cudaSetDevice(device));
    init_pool(device);
    cudaStream_t st = cudaStreamPerThread;
    Scratch sc(st);
    double* dv = sc.get_n<double>(n * dim);
    double* dt = sc.get_n<double>(n);
    double* V = sc.get_n<double>((n + 1) * dim);
    double* Tm = sc.get_n<double>(n + 1);
    double* Del = sc.get_n<double>(n + 1);
    if (sc.failed) return fail(TWB_ENOMEM, "device allocation failed");
    CK(cudaMemcpyAsync(dv, values, sizeof(double) * n * dim, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dt, times, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    int rc = prepare<double, double, double>(dv, dt, nullptr, 1, n, n, dim, nu, lam, degree, V, Tm,
                                             Del, st, 0.0);
    if (rc) return rc;
    CK(cudaMemcpyAsync(ext_values, V, sizeof(double) * (n + 1) * dim, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ext_times, Tm, sizeof(double) * (n + 1), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(deletion, Del, sizeof(double) * (n + 1), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return 0;
}

}  // extern "C"
