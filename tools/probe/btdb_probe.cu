// Tensor-core decision probe for the batched hex8 element tangent K_e = sum_q B_q^T (w D_q B_q)
// (north_star (2): tensor cores only if the batched B^T D B is a dense contraction worth it).
//
// Per element the contraction is one [24 x 48] x [48 x 24] product (the 8 Gauss points' 6-row
// strain blocks stacked along k): 27 648 FMA, 576 outputs (4.6 KB of fp64 written per element).
// Three measurements on the same device:
//   1. peak DFMA (FP64 CUDA-core pipe) and peak DMMA (mma.sync.m8n8k4.f64, FP64 tensor pipe):
//      independent accumulator chains, no memory traffic;
//   2. the element contraction on CUDA cores: one warp per element, operands in shared memory,
//      18 outputs per lane (864 DFMA each), K_e streamed out;
//   3. the same contraction on the FP64 tensor pipe: 9 output tiles x 12 k-steps = 108 DMMA per
//      warp, same shared operands, same stores.
// Operands are synthesised per element in shared memory (so both variants read identical data and
// neither is HBM-bound on the inputs); the checksum of K guards against dead-code elimination and
// compares the two variants. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void k_peak_dfma(double* out, int iters) {
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = fma(r[k], 0.999999, 1e-7);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_peak_dmma(double* out, int iters) {
  double d[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) d[k][0] = d[k][1] = threadIdx.x * 1e-3 + k;
  const double a = 0.999 + threadIdx.x * 1e-9, b = 1e-3;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(d[k][0], d[k][1], a, b);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  if (s == 12345.678) out[0] = s;
}

constexpr int WPB = 2;  // warps (elements in flight) per block (36 KB of operands)

// G (24 x 48, "B^T" of the 8 Gauss points) and H (48 x 24, "w D B") of element e in shared memory.
__device__ __forceinline__ void synth(double* G, double* H, long e, int lane) {
  for (int i = lane; i < 24 * 48; i += 32) {
    const int r = i / 48, c = i % 48;
    G[i] = 1e-3 * ((r * 7 + c * 3 + (int)(e & 15)) % 17) - 8e-3;
    H[c * 24 + r] = 1e-3 * ((r * 5 + c * 11 + (int)(e & 7)) % 13) - 6e-3;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(32 * WPB) k_btdb_dfma(double* K, long n_elem, double* sum) {
  __shared__ double sG[WPB][24 * 48], sH[WPB][48 * 24];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* G = sG[w];
  double* H = sH[w];
  double chk = 0;
  for (long e = blockIdx.x * (long)WPB + w; e < n_elem; e += (long)gridDim.x * WPB) {
    synth(G, H, e, lane);
    double acc[18];
#pragma unroll
    for (int t = 0; t < 18; ++t) acc[t] = 0;
    // outputs o = lane + 32 t (t < 18): row o / 24, col o % 24
    for (int k = 0; k < 48; ++k) {
#pragma unroll
      for (int t = 0; t < 18; ++t) {
        const int o = lane + 32 * t;
        acc[t] = fma(G[(o / 24) * 48 + k], H[k * 24 + o % 24], acc[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < 18; ++t) {
      __stcs(&K[e * 576 + lane + 32 * t], acc[t]);
      chk += acc[t];
    }
    __syncwarp();
  }
  if (chk != 0) atomicAdd(sum, chk);
}

__global__ void __launch_bounds__(32 * WPB) k_btdb_dmma(double* K, long n_elem, double* sum) {
  __shared__ double sG[WPB][24 * 48], sH[WPB][48 * 24];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* G = sG[w];
  double* H = sH[w];
  const int g = lane >> 2, q = lane & 3;  // fragment coordinates
  double chk = 0;
  for (long e = blockIdx.x * (long)WPB + w; e < n_elem; e += (long)gridDim.x * WPB) {
    synth(G, H, e, lane);
    double d[9][2];
#pragma unroll
    for (int t = 0; t < 9; ++t) d[t][0] = d[t][1] = 0;
#pragma unroll
    for (int kk = 0; kk < 12; ++kk) {
      double a[3], b[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) a[i] = G[(8 * i + g) * 48 + 4 * kk + q];   // A: row g, col q
#pragma unroll
      for (int j = 0; j < 3; ++j) b[j] = H[(4 * kk + q) * 24 + 8 * j + g];   // B: row q, col g
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) dmma(d[3 * i + j][0], d[3 * i + j][1], a[i], b[j]);
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int r = 8 * i + g, c = 8 * j + 2 * q;
        __stcs(reinterpret_cast<double2*>(&K[e * 576 + r * 24 + c]), make_double2(d[3 * i + j][0], d[3 * i + j][1]));
        chk += d[3 * i + j][0] + d[3 * i + j][1];
      }
    __syncwarp();
  }
  if (chk != 0) atomicAdd(sum, chk);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double *out, *sum, *K;
  CK(cudaMalloc(&out, 8));
  CK(cudaMalloc(&sum, 8));
  const long n_run = 1L << 19;  // 524 288 elements: 2.4 GB of K written per launch
  CK(cudaMalloc(&K, n_run * 576 * sizeof(double)));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float ms = 0;
  const int iters = 4096;
  // 1. pipe peaks
  k_peak_dfma<<<sms * 8, 256>>>(out, iters);
  CK(cudaEventRecord(a));
  for (int r = 0; r < 5; ++r) k_peak_dfma<<<sms * 8, 256>>>(out, iters);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&ms, a, b));
  const double dfma_tf = 2.0 * 8 * iters * 256.0 * sms * 8 * 5 / (ms * 1e-3) / 1e12;
  k_peak_dmma<<<sms * 8, 256>>>(out, iters);
  CK(cudaEventRecord(a));
  for (int r = 0; r < 5; ++r) k_peak_dmma<<<sms * 8, 256>>>(out, iters);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&ms, a, b));
  const double dmma_tf = 2.0 * 256 * 8 * iters * (256 / 32.0) * sms * 8 * 5 / (ms * 1e-3) / 1e12;
  std::printf("peak FP64: DFMA %.1f TFLOP/s, DMMA (m8n8k4) %.1f TFLOP/s\n", dfma_tf, dmma_tf);
  // 2./3. element contraction
  const double flop = 2.0 * 27648 * n_run, bytes = 576.0 * 8 * n_run;
  double cs[2] = {0, 0};
  for (int v = 0; v < 2; ++v) {
    for (int blocks_per_sm : {2, 4, 6}) {
      const int grid = sms * blocks_per_sm;
      CK(cudaMemset(sum, 0, 8));
      if (v == 0) k_btdb_dfma<<<grid, 32 * WPB>>>(K, n_run, sum);
      else k_btdb_dmma<<<grid, 32 * WPB>>>(K, n_run, sum);
      CK(cudaGetLastError());
      CK(cudaEventRecord(a));
      for (int r = 0; r < 3; ++r) {
        if (v == 0) k_btdb_dfma<<<grid, 32 * WPB>>>(K, n_run, sum);
        else k_btdb_dmma<<<grid, 32 * WPB>>>(K, n_run, sum);
      }
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      CK(cudaMemcpy(&cs[v], sum, 8, cudaMemcpyDeviceToHost));
      const double t = ms * 1e-3 / 3;
      std::printf("B^T D B %s  %d blocks/SM: %.3f ms per %ld elements = %.2f G elem/s, %.1f TFLOP/s (%.0f%% of "
                  "the %s peak), K stores %.0f GB/s\n",
                  v == 0 ? "DFMA" : "DMMA", blocks_per_sm, t * 1e3, n_run, n_run / t / 1e9, flop / t / 1e12,
                  100.0 * flop / t / 1e12 / (v == 0 ? dfma_tf : dmma_tf), v == 0 ? "DFMA" : "DMMA", bytes / t / 1e9);
    }
  }
  std::printf("checksums (4 launches each): DFMA %.17g DMMA %.17g rel diff %.2e\n", cs[0], cs[1],
              (cs[0] - cs[1]) / (cs[0] != 0 ? cs[0] : 1.0));
  return 0;
}
