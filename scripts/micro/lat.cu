// Latency microbenchmarks (one warp): dependent chains of FP64 ops on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2007_16135_b200/csrc/twb_device.cuh"
using namespace twb;
#define N 4096
__global__ void k_dadd(double* o, double x, long long* t) {
  double a = x + threadIdx.x; long long t0 = clock64();
  #pragma unroll 16
  for (int i = 0; i < N; ++i) a = __dadd_rn(a, x);
  long long t1 = clock64(); o[threadIdx.x] = a; if (threadIdx.x == 0) *t = t1 - t0; }
__global__ void k_dmul(double* o, double x, long long* t) {
  double a = x + threadIdx.x; long long t0 = clock64();
  #pragma unroll 16
  for (int i = 0; i < N; ++i) a = __dmul_rn(a, x);
  long long t1 = clock64(); o[threadIdx.x] = a; if (threadIdx.x == 0) *t = t1 - t0; }
__global__ void k_min(double* o, double x, long long* t) {  // DADD + DSETP + 2 FSEL chain
  double a = x + threadIdx.x, b = 1.5 * x; long long t0 = clock64();
  #pragma unroll 16
  for (int i = 0; i < N; ++i) { double d = __dadd_rn(a, x); a = (b < d) ? b : d; b = __dadd_rn(b, 1e-300); }
  long long t1 = clock64(); o[threadIdx.x] = a; if (threadIdx.x == 0) *t = t1 - t0; }
__global__ void k_imin(double* o, double x, long long* t) {  // DADD + int64 min chain
  double a = x + threadIdx.x, b = 1.5 * x; long long t0 = clock64();
  #pragma unroll 16
  for (int i = 0; i < N; ++i) { double d = __dadd_rn(a, x); a = __longlong_as_double(min(__double_as_longlong(b), __double_as_longlong(d))); b = __dadd_rn(b, 1e-300); }
  long long t1 = clock64(); o[threadIdx.x] = a; if (threadIdx.x == 0) *t = t1 - t0; }
__global__ void k_sqrt(double* o, double x, long long* t) {
  double a = x + threadIdx.x; long long t0 = clock64();
  #pragma unroll 4
  for (int i = 0; i < N; ++i) a = sqrt_fast(a) + 1.0;
  long long t1 = clock64(); o[threadIdx.x] = a; if (threadIdx.x == 0) *t = t1 - t0; }
__global__ void k_dsqrt(double* o, double x, long long* t) {
  double a = x + threadIdx.x; long long t0 = clock64();
  #pragma unroll 4
  for (int i = 0; i < N; ++i) a = __dsqrt_rn(a) + 1.0;
  long long t1 = clock64(); o[threadIdx.x] = a; if (threadIdx.x == 0) *t = t1 - t0; }
__global__ void k_shfl(double* o, double x, long long* t) {
  double a = x + threadIdx.x; long long t0 = clock64();
  #pragma unroll 16
  for (int i = 0; i < N; ++i) a = __shfl_up_sync(0xffffffffu, a, 1);
  long long t1 = clock64(); o[threadIdx.x] = a; if (threadIdx.x == 0) *t = t1 - t0; }
__global__ void k_fadd(double* o, double x, long long* t) {
  float a = x + threadIdx.x; float y = x; long long t0 = clock64();
  #pragma unroll 16
  for (int i = 0; i < N; ++i) a = __fadd_rn(a, y);
  long long t1 = clock64(); o[threadIdx.x] = a; if (threadIdx.x == 0) *t = t1 - t0; }
// throughput: 8 independent chains per thread, W warps
template <int W>
__global__ void k_dadd_tp(double* o, double x, long long* t) {
  double a0 = x + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  __syncthreads(); long long t0 = clock64();
  for (int i = 0; i < N; ++i) { a0 = __dadd_rn(a0, x); a1 = __dadd_rn(a1, x); a2 = __dadd_rn(a2, x); a3 = __dadd_rn(a3, x); a4 = __dadd_rn(a4, x); a5 = __dadd_rn(a5, x); a6 = __dadd_rn(a6, x); a7 = __dadd_rn(a7, x); }
  __syncthreads(); long long t1 = clock64();
  o[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7; if (threadIdx.x == 0) *t = t1 - t0; }
int main() {
  double* o; long long* t; cudaMalloc(&o, 8 * 1024); cudaMalloc(&t, 8);
  long long h;
#define RUN(K, name, per) K<<<1, 32>>>(o, 1.0000001, t); K<<<1, 32>>>(o, 1.0000001, t); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("%-28s %7.2f cycles/op\n", name, (double)h / (N * (per)));
  RUN(k_dadd, "DADD dep chain", 1)
  RUN(k_dmul, "DMUL dep chain", 1)
  RUN(k_fadd, "FADD dep chain", 1)
  RUN(k_min, "DADD+min(DSETP,FSEL) chain", 1)
  RUN(k_imin, "DADD+int64 min chain", 1)
  RUN(k_sqrt, "sqrt_fast+DADD chain", 1)
  RUN(k_dsqrt, "__dsqrt_rn+DADD chain", 1)
  RUN(k_shfl, "SHFL.UP (f64) chain", 1)
  k_dadd_tp<1><<<1, 32>>>(o, 1.0, t); k_dadd_tp<1><<<1, 32>>>(o, 1.0, t); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("DADD tp 1 warp x8 chains: %.2f cycles/warp-instr\n", (double)h / (N * 8));
  k_dadd_tp<1><<<1, 128>>>(o, 1.0, t); k_dadd_tp<1><<<1, 128>>>(o, 1.0, t); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("DADD tp 4 warps x8 chains: %.2f cycles per 4 warp-instr\n", (double)h / (N * 8));
  k_dadd_tp<1><<<1, 256>>>(o, 1.0, t); k_dadd_tp<1><<<1, 256>>>(o, 1.0, t); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("DADD tp 8 warps x8 chains: %.2f cycles per 8 warp-instr\n", (double)h / (N * 8));
  k_dadd_tp<1><<<1, 1024>>>(o, 1.0, t); k_dadd_tp<1><<<1, 1024>>>(o, 1.0, t); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("DADD tp 32 warps x8 chains: %.2f cycles per 8 chains x 32 warps /32\n", (double)h / (N * 8));
  cudaError_t e = cudaDeviceSynchronize(); printf("%s\n", cudaGetErrorString(e));
}
