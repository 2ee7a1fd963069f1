// DFMA throughput probe: independent accumulator chains per thread vs resident warps per SM, with
// the multiplier either a kernel parameter (uniform register / constant bank, like the stencil
// coefficients) or a register. Prints TFLOP/s per configuration. Build: nvcc -arch=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>

struct Coef { double c[32]; };

template <int CH, bool UNIFORM>
__global__ void k_dfma(const __grid_constant__ Coef C, double* out, int iters) {
  double acc[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) acc[k] = threadIdx.x * 1e-9 + k;
  double x = 1.0 + threadIdx.x * 1e-12;
  double creg[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) creg[k] = C.c[k] + threadIdx.x * 1e-15;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int k = 0; k < CH; ++k) acc[k] = fma(UNIFORM ? C.c[(j * CH + k) & 31] : creg[(j + k) & 3], x, acc[k]);
    x = x * 0.9999999;
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += acc[k];
  if (s == 12345.678) out[0] = s;
}

template <int CH, bool U>
void run(int warps_per_sm, int sms) {
  Coef C;
  for (int k = 0; k < 32; ++k) C.c[k] = 1e-3 * (k + 1);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 128, blocks = sms * warps_per_sm * 32 / threads, iters = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_dfma<CH, U><<<blocks, threads>>>(C, out, 10);
  cudaEventRecord(a);
  k_dfma<CH, U><<<blocks, threads>>>(C, out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * blocks * threads * (double)iters * 8 * CH;
  printf("chains %2d  %s  warps/SM %2d  %.1f TFLOP/s\n", CH, U ? "uniform" : "register", warps_per_sm,
         flops / ms / 1e9);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {8, 16, 32}) {
    run<6, true>(w, sms);
    run<12, true>(w, sms);
    run<18, true>(w, sms);
    run<18, false>(w, sms);
  }
  return 0;
}
