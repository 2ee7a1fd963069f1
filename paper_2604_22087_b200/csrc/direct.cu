// Banded direct solvers (BandedFactorization, krylov.hpp:196-307; run_solver's DIRECT_CHOL /
// DIRECT_LU branch, backend.hpp:245-269) on the device CSR.
//
// The band (bandwidth = max |i - j| over the pattern, as the reference) is factored in place by ONE
// persistent CTA: right-looking elimination, one pivot per step, the bw x bw trailing update spread
// over the block, a block barrier per step; then forward / backward substitution, one row per step
// with a block-wide dot product. LU is the reference's unpivoted banded LU; Cholesky is computed
// right-looking (the reference's loop is left-looking: same factor up to rounding, same failing
// pivot row). Sequential in n by nature: this completes the reference's solver menu for small
// systems (config 1: 8 450 dofs, bw 133), it is not a throughput path.
#include <algorithm>
#include <cmath>
#include <vector>

#include "afem_impl.hpp"

namespace afem {
namespace {

constexpr int kDirThreads = 1024;

// Scatter the CSR values into band storage. LU: full(i, j) = band[i * W + (j - i + bw)], W = 2bw+1;
// CHOL: lo(i, j) = band[i * W + (j - i + bw)], j <= i only (W = bw + 1, offset bw).
__global__ void k_to_band(SysView s, const double* __restrict__ vals, double* band, int64_t bw, int64_t W, int chol) {
  const int D = s.dim;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s.n_dof; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / D;
    const int a = static_cast<int>(i % D);
    const int64_t a0 = s.adj_ptr[n];
    const int deg = static_cast<int>(s.adj_ptr[n + 1] - a0);
    const int64_t base = (int64_t)D * D * a0 + (int64_t)a * D * deg;
    for (int jj = 0; jj < D * deg; ++jj) {
      const int64_t j = (int64_t)D * s.adj[a0 + jj / D] + jj % D;
      if (chol && j > i) continue;
      band[i * W + (j - i + bw)] = vals[base + jj];
    }
  }
}

__global__ void __launch_bounds__(kDirThreads) k_band_lu(double* band, int64_t n, int64_t bw, int64_t* bad) {
  const int64_t W = 2 * bw + 1;
  auto F = [&](int64_t i, int64_t j) -> double& { return band[i * W + (j - i + bw)]; };
  __shared__ double piv;
  for (int64_t k = 0; k < n; ++k) {
    if (threadIdx.x == 0) piv = F(k, k);
    __syncthreads();
    if (piv == 0.0) {
      if (threadIdx.x == 0) *bad = k;
      return;
    }
    const int64_t m = std::min(n - 1, k + bw) - k;  // rows / cols k+1 .. k+m
    for (int64_t t = threadIdx.x; t < m; t += blockDim.x) F(k + 1 + t, k) /= piv;
    __syncthreads();
    for (int64_t t = threadIdx.x; t < m * m; t += blockDim.x) {
      const int64_t i = k + 1 + t / m, j = k + 1 + t % m;
      F(i, j) -= F(i, k) * F(k, j);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kDirThreads) k_band_chol(double* band, int64_t n, int64_t bw, int64_t* bad) {
  const int64_t W = bw + 1;
  auto L = [&](int64_t i, int64_t j) -> double& { return band[i * W + (j - i + bw)]; };
  __shared__ double d;
  for (int64_t k = 0; k < n; ++k) {
    if (threadIdx.x == 0) {
      const double s = L(k, k);
      d = s > 0.0 ? sqrt(s) : 0.0;
      L(k, k) = d;
    }
    __syncthreads();
    if (!(d > 0.0)) {
      if (threadIdx.x == 0) *bad = k;
      return;
    }
    const int64_t m = std::min(n - 1, k + bw) - k;
    for (int64_t t = threadIdx.x; t < m; t += blockDim.x) L(k + 1 + t, k) /= d;
    __syncthreads();
    for (int64_t t = threadIdx.x; t < m * m; t += blockDim.x) {  // lower triangle of the trailing block
      const int64_t i = k + 1 + t / m, j = k + 1 + t % m;
      if (j <= i) L(i, j) -= L(i, k) * L(j, k);
    }
    __syncthreads();
  }
}

// Block-wide sum (result in every thread).
__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = lane < static_cast<int>(blockDim.x >> 5) ? sh[lane] : 0.0;
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __syncthreads();
  return t;
}

// x = A^-1 b with the factor: forward then backward substitution (krylov.hpp:258-300).
__global__ void __launch_bounds__(kDirThreads) k_band_solve(const double* band, int64_t n, int64_t bw, int chol,
                                                            double* x) {
  __shared__ double sh[32];
  const int64_t W = chol ? bw + 1 : 2 * bw + 1;
  auto B = [&](int64_t i, int64_t j) -> double { return band[i * W + (j - i + bw)]; };
  for (int64_t i = 0; i < n; ++i) {  // L y = b (unit diagonal for LU)
    double s = 0.0;
    for (int64_t j = std::max<int64_t>(0, i - bw) + threadIdx.x; j < i; j += blockDim.x) s += B(i, j) * x[j];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) x[i] = chol ? (x[i] - s) / B(i, i) : x[i] - s;
    __syncthreads();
  }
  for (int64_t i = n - 1; i >= 0; --i) {  // U x = y (CHOL: L^T)
    double s = 0.0;
    const int64_t jmax = std::min(n - 1, i + bw);
    for (int64_t j = i + 1 + threadIdx.x; j <= jmax; j += blockDim.x) s += (chol ? B(j, i) : B(i, j)) * x[j];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) x[i] = (x[i] - s) / B(i, i);
    __syncthreads();
  }
}

}  // namespace

// run_solver's direct branch: returns false (failure set) when the factorisation breaks down.
bool direct_solve(System& s, const double* vals, bool chol, const double* b, double* x, std::string& failure) {
  Ctx& c = *s.ctx;
  const int64_t n = s.n_dof;
  // bandwidth from the pattern (krylov.hpp:205-208): max |i - j| over the node adjacency, in dofs
  std::vector<int64_t> ap(s.n_nodes + 1);
  std::vector<int32_t> adj(s.adj.n);
  AFEM_CK(cudaMemcpyAsync(ap.data(), s.adj_ptr.p, ap.size() * 8, cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaMemcpyAsync(adj.data(), s.adj.p, adj.size() * 4, cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  int64_t bw = 0;
  for (int64_t nd = 0; nd < s.n_nodes; ++nd)
    for (int64_t k = ap[nd]; k < ap[nd + 1]; ++k)
      bw = std::max(bw, std::abs((int64_t)adj[k] - nd) * s.dim + (s.dim - 1));
  const int64_t W = chol ? bw + 1 : 2 * bw + 1;
  if ((double)n * W * 8.0 > 16e9)
    throw CapabilityError("direct solve: the band (" + std::to_string(n) + " x " + std::to_string(W) +
                          ") exceeds the device budget; use an iterative method");
  DevArray<double> band((size_t)n * W);
  DevArray<int64_t> bad(1);
  AFEM_CK(cudaMemsetAsync(band.p, 0, band.bytes(), c.stream));
  const int64_t init = -1;
  AFEM_CK(cudaMemcpyAsync(bad.p, &init, 8, cudaMemcpyHostToDevice, c.stream));
  launch(c, k_to_band, grid_for(n, 256, 148 * 16), 256, 0, s.view(), vals, band.p, bw, W, chol ? 1 : 0);
  if (chol) launch(c, k_band_chol, 1, kDirThreads, 0, band.p, n, bw, bad.p);
  else launch(c, k_band_lu, 1, kDirThreads, 0, band.p, n, bw, bad.p);
  int64_t hb = -1;
  AFEM_CK(cudaMemcpyAsync(&hb, bad.p, 8, cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  if (hb >= 0) {
    failure = chol ? "cholesky: matrix not positive definite at pivot row " + std::to_string(hb)
                   : "lu: zero pivot at row " + std::to_string(hb);
    return false;
  }
  AFEM_CK(cudaMemcpyAsync(x, b, n * 8, cudaMemcpyDeviceToDevice, c.stream));
  launch(c, k_band_solve, 1, kDirThreads, 0, band.p, n, bw, chol ? 1 : 0, x);
  return true;
}

}  // namespace afem
