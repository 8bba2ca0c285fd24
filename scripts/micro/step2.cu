// Emulate a lane step processing C adjacent columns (split recurrence).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2007_16135_b200/csrc/twb_device.cuh"
using namespace twb;
#define ITERS 512
template <int K, int C>
__global__ void __launch_bounds__(512) k_step(double* o, const double* __restrict__ in, double x) {
  double a[K][3], da[K], ta[K], zl[K], mr[K], gr[K];
  for (int q = 0; q < K; ++q) { a[q][0] = in[q]; a[q][1] = in[q+1]; a[q][2] = in[q+2]; da[q] = in[q+3]; ta[q] = in[q+5]; zl[q] = in[q+4]; mr[q] = 0; gr[q] = 0; }
  double zbot[C], mbot[C];
  for (int c = 0; c < C; ++c) { zbot[c] = x; mbot[c] = 0; }
  double b0 = threadIdx.x * 1e-3, tb = 0.5, delb = 0.25, zprev = 0, mprev = 0, tbprev = 0, tup = 0.1;
  for (int it = 0; it < ITERS; ++it) {
    double zin[C], min_[C];
    for (int c = 0; c < C; ++c) { zin[c] = __shfl_up_sync(0xffffffffu, zbot[c], 1); min_[c] = __shfl_up_sync(0xffffffffu, mbot[c], 1); }
    for (int c = 0; c < C; ++c) {
      const double bb0 = b0 + c, bb1 = bb0 + 1, bb2 = bb0 + 2, tbc = tb + c, delbc = delb + c * 1e-9;
      double mn[K];
      for (int q = 0; q < K; ++q) {
        double d0 = a[q][0] - bb0, d1 = a[q][1] - bb1, d2 = a[q][2] - bb2;
        mn[q] = sqrt_safe(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)));
      }
      // cell (q, c): z_up = row above same column; z_left = zl[q] (previous column); z_diag
      double zu = zin[c], zd = zprev, mu = mprev, gu = tup - tbprev;
      for (int q = 0; q < K; ++q) {
        const double g = ta[q] - tbc;
        const double gs = __dadd_rn(fabs(g), fabs(gu));
        const double match = __dadd_rn(__dadd_rn(__dadd_rn(zd, mn[q]), mu), gs);
        const double del_b = zl[q] + delbc;
        const double pre = match < del_b ? match : del_b;
        const double del_a = zu + da[q];
        const double z = pre < del_a ? pre : del_a;
        zd = zl[q]; mu = mr[q]; gu = gr[q];
        zl[q] = z; mr[q] = mn[q]; gr[q] = g; zu = z;
      }
      zprev = zin[c]; mprev = min_[c]; tbprev = tbc;
      zbot[c] = zu; mbot[c] = mr[K - 1];
    }
    b0 += 1e-9 * C; tb += C; delb += 1e-12;
  }
  double s = 0; for (int q = 0; q < K; ++q) s += zl[q];
  o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o; double* in; cudaMalloc(&o, 8 * 148 * 1024 * 4); cudaMalloc(&in, 8 * 64);
  double h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0 + i * 0.37; cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
#define RUN(K, C) for (int w : {4, 8, 12, 16}) { k_step<K, C><<<148, 32 * w>>>(o, in, 1.0); cudaEventRecord(e0); k_step<K, C><<<148, 32 * w>>>(o, in, 1.0); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); \
   double n = 148.0 * 32 * w * ITERS * K * C; printf("K=%d C=%d warps/SM=%2d: %7.1f GCUPS (%.2f cells per SM-clk; %.0f cyc/step/warp)\n", K, C, w, n / ms / 1e6, n / (ms * 1e-3) / (148 * 1.965e9), (ms * 1e-3 * 1.965e9) / ITERS); }
  RUN(8, 1) RUN(8, 2) RUN(4, 1) RUN(4, 2) RUN(4, 4) RUN(2, 4) RUN(6, 2)
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
