// Throughput microbenchmarks on sm_100a: many warps, independent work.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2007_16135_b200/csrc/twb_device.cuh"
using namespace twb;
#define ITERS 2048
__device__ __forceinline__ double rsq(double a){ double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); return r; }
__global__ void k_mufu(double* o, double x) {
  double a0 = x + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  for (int i = 0; i < ITERS; ++i) { a0 = rsq(a0); a1 = rsq(a1); a2 = rsq(a2); a3 = rsq(a3); }
  o[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3; }
__global__ void k_sqrtf(double* o, double x) {
  double a0 = x + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  for (int i = 0; i < ITERS; ++i) { a0 = sqrt_fast(a0) + 2.0; a1 = sqrt_fast(a1) + 2.0; a2 = sqrt_fast(a2) + 2.0; a3 = sqrt_fast(a3) + 2.0; }
  o[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3; }
__global__ void k_sqrts(double* o, double x) {
  double a0 = x + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  for (int i = 0; i < ITERS; ++i) { a0 = sqrt_safe(a0) + 2.0; a1 = sqrt_safe(a1) + 2.0; a2 = sqrt_safe(a2) + 2.0; a3 = sqrt_safe(a3) + 2.0; }
  o[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3; }
__global__ void k_dsetp(double* o, double x) {
  double a0 = x + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b = x * 0.5;
  for (int i = 0; i < ITERS; ++i) { a0 = a0 < b ? a0 : b; a1 = a1 < b ? a1 : b; a2 = a2 < b ? a2 : b; a3 = a3 < b ? a3 : b; b = b + 1e-300; }
  o[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3; }
__global__ void k_dfma(double* o, double x) {
  double a0 = x + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  for (int i = 0; i < ITERS; ++i) { a0 = __fma_rn(a0, x, x); a1 = __fma_rn(a1, x, x); a2 = __fma_rn(a2, x, x); a3 = __fma_rn(a3, x, x); }
  o[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3; }
// a TWED-like cell, d = 3: sumsq + sqrt_safe + 9 DADD + 2 min
__global__ void k_cell(double* o, double x) {
  double z0 = x + threadIdx.x, z1 = z0 + 1, z2 = z0 + 2, z3 = z0 + 3;
  const double a0 = x, a1 = 2 * x, a2 = 3 * x;
  double b0 = threadIdx.x * 1e-3, b1 = b0 + 1, b2 = b0 + 2;
  for (int i = 0; i < ITERS; ++i) {
    #define CELL(z) { double d0 = a0 - b0, d1 = a1 - b1, d2 = a2 - b2; \
      double acc = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)); \
      double m = sqrt_safe(acc); double g = __dadd_rn(fabs(a0 - b2), fabs(a1 - b0)); \
      double match = __dadd_rn(__dadd_rn(__dadd_rn(z, m), m), g); double db = z + b1; double da = z + b0; \
      double t = match < db ? match : db; z = t < da ? t : da; }
    CELL(z0) CELL(z1) CELL(z2) CELL(z3)
    b0 += 1e-9; b1 += 1e-9; b2 += 1e-9;
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = z0 + z1 + z2 + z3; }
int main() {
  double* o; cudaMalloc(&o, 8 * 148 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
#define RUN(K, name, ops_per_iter) for (int w : {4, 8, 16, 32}) { K<<<148, 32 * w>>>(o, 1.0000001); cudaEventRecord(e0); K<<<148, 32 * w>>>(o, 1.0000001); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); \
   double n = 148.0 * 32 * w * ITERS * ops_per_iter; printf("%-12s warps/SM=%2d: %8.3f G/s  (%.2f per SM-clk @1.965GHz)\n", name, w, n / ms / 1e6, n / (ms * 1e-3) / (148 * 1.965e9)); }
  RUN(k_mufu, "MUFU.RSQ64H", 4)
  RUN(k_sqrtf, "sqrt_fast", 4)
  RUN(k_sqrts, "sqrt_safe", 4)
  RUN(k_dsetp, "min DSETP", 4)
  RUN(k_dfma, "DFMA", 4)
  RUN(k_cell, "cell d=3", 4)
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
