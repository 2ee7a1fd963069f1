// BLAS-1 on the device (linalg.hpp:41-58). Reductions are deterministic: a fixed grid of
// kRedBlocks blocks accumulates in grid-stride order, each block tree-reduces, and the last block
// to finish (threadfence + ticket) reduces the per-block partials in a fixed order. The result is
// bitwise reproducible run to run (the reference demands bitwise determinism of its assembly,
// test_assembly.cpp:262-276; we keep the same property for every reduction).
#include "afem_impl.hpp"
#include "reduce.cuh"

namespace afem {
namespace {

__global__ void __launch_bounds__(kRedThreads) k_dot(const double* __restrict__ x, const double* __restrict__ y,
                                                     int64_t n, double* partials, unsigned int* counter,
                                                     double* out, int sqrt_out) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += x[i] * y[i];
  double v[1] = {s};
  if (grid_reduce<1>(v, partials, counter)) {
    if (threadIdx.x == 0) out[0] = sqrt_out ? sqrt(v[0]) : v[0];
  }
}

__global__ void __launch_bounds__(kRedThreads) k_free_sq(const double* __restrict__ r, const uint8_t* __restrict__ mask,
                                                         int64_t n, double* partials, unsigned int* counter,
                                                         double* out) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!mask[i]) s += r[i] * r[i];
  double v[1] = {s};
  if (grid_reduce<1>(v, partials, counter)) {
    if (threadIdx.x == 0) out[0] = sqrt(v[0]);
  }
}

__global__ void k_axpy(double a, const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += a * x[i];
}

__global__ void k_axpy_dev(const double* alpha, double scale, const double* __restrict__ x, double* __restrict__ y,
                           int64_t n) {
  const double a = scale * alpha[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += a * x[i];
}

__global__ void k_fill(double v, double* y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = v;
}

}  // namespace

unsigned red_grid(int64_t n) { return grid_for(n, kRedThreads, kRedBlocks); }

void dot_dev(Ctx& c, const double* x, const double* y, int64_t n, double* out_dev) {
  launch(c, k_dot, red_grid(n), kRedThreads, 0, x, y, n, c.red_partials.p, c.red_counter.p, out_dev, 0);
}

static double fetch(Ctx& c, const double* d) {
  double h = 0.0;
  AFEM_CK(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  return h;
}

double dot(Ctx& c, const double* x, const double* y, int64_t n) {
  dot_dev(c, x, y, n, c.red_out.p);
  return fetch(c, c.red_out.p);
}

double free_norm(Ctx& c, const double* r, const uint8_t* mask, int64_t n) {
  launch(c, k_free_sq, red_grid(n), kRedThreads, 0, r, mask, n, c.red_partials.p, c.red_counter.p, c.red_out.p);
  return fetch(c, c.red_out.p);
}

void axpy(Ctx& c, double a, const double* x, double* y, int64_t n) {
  launch(c, k_axpy, grid_for(n, 256, 148 * 16), 256, 0, a, x, y, n);
}

void add_scaled_dev(Ctx& c, const double* alpha_dev, double scale, const double* x, double* y, int64_t n) {
  launch(c, k_axpy_dev, grid_for(n, 256, 148 * 16), 256, 0, alpha_dev, scale, x, y, n);
}

void copy(Ctx& c, const double* x, double* y, int64_t n) {
  if (x != y) AFEM_CK(cudaMemcpyAsync(y, x, n * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
}

void fill(Ctx& c, double v, double* y, int64_t n) { launch(c, k_fill, grid_for(n, 256, 148 * 16), 256, 0, v, y, n); }

}  // namespace afem
