// Deterministic grid-wide reduction of NV doubles (last-block-done pattern).
#pragma once

#include "common.cuh"

namespace afem {

// Block-wide sum of NV values per thread; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV]) {
  __shared__ double sh[NV][kRedThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double t = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) sh[k][w] = t;
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double t = lane < (int)(blockDim.x >> 5) ? sh[k][lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      v[k] = t;
    }
  }
  __syncthreads();
}

// Every block contributes v; returns true in the last block, where v (thread 0) holds the grid sum
// of all blocks, reduced in a fixed order. partials needs gridDim.x*NV doubles.
template <int NV>
__device__ __forceinline__ bool grid_reduce(double (&v)[NV], double* partials, unsigned int* counter) {
  __shared__ bool last;
  block_reduce<NV>(v);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) partials[k * gridDim.x + blockIdx.x] = v[k];
    __threadfence();
    const unsigned int t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
    for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x) s += __ldcg(&partials[k * gridDim.x + b]);
    v[k] = s;
  }
  block_reduce<NV>(v);
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

// Cross-kernel fixed-order reduction: every block of a kernel stores its block sum in
// mine[bid]; the last block to finish (ticket) adds prior[0..nprior) then mine[0..nmine) in index
// order and writes out[0]. Deterministic for fixed launch shapes.
__device__ __forceinline__ void block_to_slot_and_finish(double v, double* mine, int bid, int nmine,
                                                         const double* prior, int nprior, unsigned int* counter,
                                                         double* out) {
  __shared__ bool last;
  double a[1] = {v};
  block_reduce<1>(a);
  if (threadIdx.x == 0) {
    mine[bid] = a[0];
    __threadfence();
    last = atomicAdd(counter, 1u) == static_cast<unsigned>(nmine - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double s = 0.0;
  // fixed assignment of partials to threads, then a fixed-shape block reduction
  for (int b = threadIdx.x; b < nprior; b += blockDim.x) s += __ldcg(&prior[b]);
  for (int b = threadIdx.x; b < nmine; b += blockDim.x) s += __ldcg(&mine[b]);
  a[0] = s;
  block_reduce<1>(a);
  if (threadIdx.x == 0) {
    out[0] = a[0];
    *counter = 0u;
  }
}

}  // namespace afem
