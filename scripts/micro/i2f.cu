#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_i2f(double* o, int x) {
  int a0 = x + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < ITERS; ++i) {
    s0 = (double)(a0 ^ i); s1 = (double)(a1 ^ i); s2 = (double)(a2 ^ i); s3 = (double)(a3 ^ i);
    a0 += (int)s1; a1 += (int)s2; a2 += 3; a3 += 5;
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void k_i2f_only(double* o, int x) {
  int a = x + threadIdx.x;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  #pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    s0 = __dadd_rn(s0, (double)(a + i)); s1 = __dadd_rn(s1, (double)(a - i)); s2 = __dadd_rn(s2, (double)(a ^ i)); s3 = __dadd_rn(s3, (double)(a | i));
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void k_dadd_only(double* o, int x) {
  double a = x + threadIdx.x;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  #pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    s0 = __dadd_rn(s0, a); s1 = __dadd_rn(s1, a); s2 = __dadd_rn(s2, a); s3 = __dadd_rn(s3, a);
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
int main() {
  double* o; cudaMalloc(&o, 8 * 148 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
#define RUN(K, name, per) for (int w : {8, 16, 32}) { K<<<148, 32 * w>>>(o, 1); cudaEventRecord(e0); K<<<148, 32 * w>>>(o, 1); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); \
   double n = 148.0 * 32 * w * ITERS * per; printf("%-26s warps/SM=%2d: %.2f per SM-clk\n", name, w, n / (ms * 1e-3) / (148 * 1.965e9)); }
  RUN(k_dadd_only, "DADD x4", 4)
  RUN(k_i2f_only, "I2F.F64+DADD x4 (per pair)", 4)
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
