// Emulate one lane's step: K-row min-plus chain + K independent distance cells.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2007_16135_b200/csrc/twb_device.cuh"
using namespace twb;
#define ITERS 1024
template <int K, int MODE>
__global__ void k_step(double* o, const double* __restrict__ in, double x) {
  double a[K][3], da[K], zl[K], mr[K], pre[K];
  for (int q = 0; q < K; ++q) { a[q][0] = in[q]; a[q][1] = in[q+1]; a[q][2] = in[q+2]; da[q] = in[q+3]; zl[q] = in[q+4]; mr[q] = 0; pre[q] = 1e300; }
  double zup = x, tb = 0.5, delb = 0.25;
  double b0 = threadIdx.x * 1e-3, b1 = b0 + 1, b2 = b0 + 2;
  for (int it = 0; it < ITERS; ++it) {
    // chain for this column
    double zu = __shfl_up_sync(0xffffffffu, zup, 1);
    for (int q = 0; q < K; ++q) {
      const double del_a = zu + da[q];
      double z;
      if (MODE == 1) z = __longlong_as_double(min(__double_as_longlong(pre[q]), __double_as_longlong(del_a)));
      else z = pre[q] < del_a ? pre[q] : del_a;
      zl[q] = z; zu = z;
    }
    zup = zu;
    // next column distances + prep
    double mn[K];
    for (int q = 0; q < K; ++q) {
      double d0 = a[q][0] - b0, d1 = a[q][1] - b1, d2 = a[q][2] - b2;
      double acc = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
      if (MODE == 2) { double r = sqrt_fast(acc); mn[q] = (__double2hiint(acc) == 0) ? 0.0 : r; }
      else mn[q] = sqrt_safe(acc);
    }
    for (int q = K - 1; q >= 0; --q) {
      const double g = __dadd_rn(fabs(a[q][0] - tb), fabs(a[q][1] - tb));
      const double zd = q > 0 ? zl[q - 1] : zup;
      const double m_up = q > 0 ? mr[q - 1] : 0.0;
      const double match = __dadd_rn(__dadd_rn(__dadd_rn(zd, mn[q]), m_up), g);
      const double del_b = zl[q] + delb;
      if (MODE == 1) pre[q] = __longlong_as_double(min(__double_as_longlong(match), __double_as_longlong(del_b)));
      else pre[q] = match < del_b ? match : del_b;
      mr[q] = mn[q];
    }
    b0 += 1e-9; b1 += 1e-9; b2 += 1e-9; tb += 1.0; delb += 1e-12;
  }
  double s = 0; for (int q = 0; q < K; ++q) s += zl[q] + pre[q];
  o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o; double* in; cudaMalloc(&o, 8 * 148 * 1024 * 4); cudaMalloc(&in, 8 * 64);
  double h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0 + i * 0.37; cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
#define RUN(K, M, name) for (int w : {1, 2, 4, 8, 16}) { k_step<K, M><<<148, 32 * w>>>(o, in, 1.0); cudaEventRecord(e0); k_step<K, M><<<148, 32 * w>>>(o, in, 1.0); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); \
   double n = 148.0 * 32 * w * ITERS * K; printf("%-22s K=%d warps/SM=%2d: %7.1f GCUPS (%.2f cells per SM-clk; %.0f cyc/step/warp)\n", name, K, w, n / ms / 1e6, n / (ms * 1e-3) / (148 * 1.965e9), (ms * 1e-3 * 1.965e9) / ITERS); }
  RUN(8, 0, "sqrt_safe dsetp")
  RUN(8, 1, "sqrt_safe intmin")
  RUN(8, 2, "sqrt_fast+0sel dsetp")
  RUN(4, 0, "sqrt_safe dsetp")
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
