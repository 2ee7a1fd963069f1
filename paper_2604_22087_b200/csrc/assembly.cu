// General-mesh assembly kernels (any quad4 / hex8 geometry): residual, tangent (CSR values),
// diagonal, matrix-free JVP, Dirichlet elimination and CSR SpMV.
//
// Scatter strategy: node-centric gather. One thread owns a node's dim rows and walks the node's
// incident (element, local node) list in the reference's (batch, element) order (system.cu), so
// every sum is deterministic run to run and associates element contributions exactly like the
// reference's scatter-add (assembly.hpp:130-137) and its stable-sort duplicate summation
// (sparse.hpp:25-27, assembly.hpp:158-172). No fp64 atomics anywhere.
// Each (node, element) pair re-evaluates the element's quadrature loop for its own rows only; the
// structured stencil path (stencil.cu) is the throughput path for the matrix-free operator.
#include <cstdlib>
#include "afem_impl.hpp"

namespace afem {
namespace {

template <int D>
__device__ __forceinline__ void load_coords(const SysView& s, int64_t e, double (&xc)[EL<D>::npe][D]) {
#pragma unroll
  for (int k = 0; k < EL<D>::npe; ++k) {
    const int64_t n = s.conn[e * EL<D>::npe + k];
#pragma unroll
    for (int c = 0; c < D; ++c) xc[k][c] = s.coords[n * D + c];
  }
}

template <int D>
__device__ __forceinline__ void load_dofs(const SysView& s, int64_t e, const double* v, double (&ve)[EL<D>::nd]) {
#pragma unroll
  for (int k = 0; k < EL<D>::npe; ++k) {
    const int64_t n = s.conn[e * EL<D>::npe + k];
#pragma unroll
    for (int c = 0; c < D; ++c) ve[k * D + c] = v[n * D + c];
  }
}

template <int D>
__device__ __forceinline__ void load_dofs_masked(const SysView& s, int64_t e, const double* v, const uint8_t* mask,
                                                 double (&ve)[EL<D>::nd]) {
#pragma unroll
  for (int k = 0; k < EL<D>::npe; ++k) {
    const int64_t n = s.conn[e * EL<D>::npe + k];
#pragma unroll
    for (int c = 0; c < D; ++c) ve[k * D + c] = mask[n * D + c] ? 0.0 : v[n * D + c];
  }
}

__device__ __forceinline__ const double* qp_hist(const SysView& s, int64_t e, int q, int nq) {
  return s.hist ? s.hist + (e * nq + q) * kHist : nullptr;
}

// R(u) rows of node n (assembly.hpp:126-139 with element_internal_force, element.hpp:68-125).
template <int D>
__global__ void __launch_bounds__(128) k_residual(SysView s, const double* u, double* r) {
  constexpr int npe = EL<D>::npe, nq = EL<D>::nq, nd = EL<D>::nd;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < s.n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    double acc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) acc[a] = 0.0;
    int err = 0;
    for (int64_t p = s.inc_ptr[n]; p < s.inc_ptr[n + 1]; ++p) {
      const uint32_t v = s.inc[p];
      const int64_t e = v / npe;
      const int ln = v % npe;
      double xc[npe][D], ue[nd];
      load_coords<D>(s, e, xc);
      load_dofs<D>(s, e, u, ue);
      const DMat m = s.mats[s.phase[e]];
      double f[D];
#pragma unroll
      for (int a = 0; a < D; ++a) f[a] = 0.0;
      for (int q = 0; q < nq; ++q) {
        double g[npe][D], wdet;
        if (!qp_geometry<D>(xc, q, g, wdet)) err |= ERR_DETJ;
        double H[D][D], P[D][D];
        grad_u<D>(ue, g, H);
        piola<D>(m, H, P, err, qp_hist(s, e, q, nq));
#pragma unroll
        for (int a = 0; a < D; ++a) {
          double t = 0.0;
#pragma unroll
          for (int b = 0; b < D; ++b) t += P[a][b] * g[ln][b];
          f[a] += wdet * t;
        }
      }
#pragma unroll
      for (int a = 0; a < D; ++a) acc[a] += f[a];
    }
    if (err) atomicOr(s.err, err);
#pragma unroll
    for (int a = 0; a < D; ++a) r[D * n + a] = acc[a];
  }
}

// Matrix-free K(u) x rows of node n: masked JVP (backend.hpp:130-147).
template <int D>
__global__ void __launch_bounds__(128) k_mf_apply(SysView s, const double* state, const uint8_t* mask,
                                                  const double* x, double* y) {
  constexpr int npe = EL<D>::npe, nq = EL<D>::nq, nd = EL<D>::nd;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < s.n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    double acc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) acc[a] = 0.0;
    int err = 0;
    for (int64_t p = s.inc_ptr[n]; p < s.inc_ptr[n + 1]; ++p) {
      const uint32_t v = s.inc[p];
      const int64_t e = v / npe;
      const int ln = v % npe;
      double xc[npe][D], ue[nd], xe[nd];
      load_coords<D>(s, e, xc);
      load_dofs_masked<D>(s, e, x, mask, xe);
      const DMat m = s.mats[s.phase[e]];
      if (m.model != MODEL_LINEAR) load_dofs<D>(s, e, state, ue);
      double f[D];
#pragma unroll
      for (int a = 0; a < D; ++a) f[a] = 0.0;
      for (int q = 0; q < nq; ++q) {
        double g[npe][D], wdet;
        if (!qp_geometry<D>(xc, q, g, wdet)) err |= ERR_DETJ;
        double H[D][D], dH[D][D], dP[D][D];
        grad_u<D>(xe, g, dH);
        if (m.model != MODEL_LINEAR) grad_u<D>(ue, g, H);
        piola_jvp<D>(m, H, dH, dP, qp_hist(s, e, q, nq));
#pragma unroll
        for (int a = 0; a < D; ++a) {
          double t = 0.0;
#pragma unroll
          for (int b = 0; b < D; ++b) t += dP[a][b] * g[ln][b];
          f[a] += wdet * t;
        }
      }
#pragma unroll
      for (int a = 0; a < D; ++a) acc[a] += f[a];
    }
    if (err) atomicOr(s.err, err);
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int64_t d = D * n + a;
      y[d] = mask[d] ? x[d] : acc[a];
    }
  }
}

// history_commit: advance every J2 quadrature point's committed history to the return-mapped
// state at u (one thread per element, in place: each slot is read and written by its owner only).
template <int D>
__global__ void __launch_bounds__(128) k_history_commit(SysView s, const double* u, double* hist) {
  constexpr int npe = EL<D>::npe, nq = EL<D>::nq, nd = EL<D>::nd;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s.n_elem; e += (int64_t)gridDim.x * blockDim.x) {
    const DMat m = s.mats[s.phase[e]];
    if (m.model != MODEL_J2) continue;
    double xc[npe][D], ue[nd];
    load_coords<D>(s, e, xc);
    load_dofs<D>(s, e, u, ue);
    for (int q = 0; q < nq; ++q) {
      double g[npe][D], wdet;
      qp_geometry<D>(xc, q, g, wdet);
      double H[D][D];
      grad_u<D>(ue, g, H);
      double* hq = hist + (e * nq + q) * kHist;
      j2_commit<D>(m, H, hq, hq);
    }
  }
}

__device__ __forceinline__ int find_pos(const int32_t* adj, int deg, int32_t m) {
  int lo = 0, hi = deg;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (adj[mid] < m) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// K(u) rows of node n into pattern-ordered CSR values (assembly.hpp:144-173).
template <int D>
__global__ void __launch_bounds__(128) k_jacobian(SysView s, const double* u, double* values) {
  constexpr int npe = EL<D>::npe, nq = EL<D>::nq, nd = EL<D>::nd;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < s.n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a0 = s.adj_ptr[n];
    const int deg = static_cast<int>(s.adj_ptr[n + 1] - a0);
    const int64_t base = (int64_t)D * D * a0;
    for (int j = 0; j < D * D * deg; ++j) values[base + j] = 0.0;
    int err = 0;
    for (int64_t p = s.inc_ptr[n]; p < s.inc_ptr[n + 1]; ++p) {
      const uint32_t v = s.inc[p];
      const int64_t e = v / npe;
      const int ln = v % npe;
      double xc[npe][D], ue[nd];
      load_coords<D>(s, e, xc);
      load_dofs<D>(s, e, u, ue);
      const DMat m = s.mats[s.phase[e]];
      int pos[npe];
#pragma unroll
      for (int k = 0; k < npe; ++k) pos[k] = find_pos(s.adj + a0, deg, s.conn[e * npe + k]);
      double K[D][nd];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int j = 0; j < nd; ++j) K[a][j] = 0.0;
      for (int q = 0; q < nq; ++q) {
        double g[npe][D], wdet;
        if (!qp_geometry<D>(xc, q, g, wdet)) err |= ERR_DETJ;
        double H[D][D];
        grad_u<D>(ue, g, H);
        TangentQP<D> t;
        tangent_qp<D>(m, H, t, err, qp_hist(s, e, q, nq));
        double gn[D];
#pragma unroll
        for (int c = 0; c < D; ++c) gn[c] = g[ln][c];
#pragma unroll
        for (int lm = 0; lm < npe; ++lm) {
          double gm[D], blk[D][D];
#pragma unroll
          for (int c = 0; c < D; ++c) gm[c] = g[lm][c];
          tangent_block<D>(t, gn, gm, blk);
#pragma unroll
          for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = 0; b < D; ++b) K[a][lm * D + b] += wdet * blk[a][b];
        }
      }
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const int64_t row = base + (int64_t)a * D * deg;
#pragma unroll
        for (int lm = 0; lm < npe; ++lm)
#pragma unroll
          for (int b = 0; b < D; ++b) values[row + pos[lm] * D + b] += K[a][lm * D + b];
      }
    }
    if (err) atomicOr(s.err, err);
  }
}

// diag K(u) (assembly.hpp:177-188).
template <int D>
__global__ void __launch_bounds__(128) k_diagonal(SysView s, const double* u, double* d) {
  constexpr int npe = EL<D>::npe, nq = EL<D>::nq, nd = EL<D>::nd;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < s.n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    double acc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) acc[a] = 0.0;
    int err = 0;
    for (int64_t p = s.inc_ptr[n]; p < s.inc_ptr[n + 1]; ++p) {
      const uint32_t v = s.inc[p];
      const int64_t e = v / npe;
      const int ln = v % npe;
      double xc[npe][D], ue[nd];
      load_coords<D>(s, e, xc);
      load_dofs<D>(s, e, u, ue);
      const DMat m = s.mats[s.phase[e]];
      double f[D];
#pragma unroll
      for (int a = 0; a < D; ++a) f[a] = 0.0;
      for (int q = 0; q < nq; ++q) {
        double g[npe][D], wdet;
        if (!qp_geometry<D>(xc, q, g, wdet)) err |= ERR_DETJ;
        double H[D][D];
        grad_u<D>(ue, g, H);
        TangentQP<D> t;
        tangent_qp<D>(m, H, t, err, qp_hist(s, e, q, nq));
        double gn[D], blk[D][D];
#pragma unroll
        for (int c = 0; c < D; ++c) gn[c] = g[ln][c];
        tangent_block<D>(t, gn, gn, blk);
#pragma unroll
        for (int a = 0; a < D; ++a) f[a] += wdet * blk[a][a];
      }
#pragma unroll
      for (int a = 0; a < D; ++a) acc[a] += f[a];
    }
    if (err) atomicOr(s.err, err);
#pragma unroll
    for (int a = 0; a < D; ++a) d[D * n + a] = acc[a];
  }
}

// eliminate_dirichlet (assembly.hpp:218-238): one thread per row, slots in column order.
__global__ void k_eliminate(SysView s, double* values, double* res, const double* u) {
  const int D = s.dim;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s.n_dof; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / D;
    const int a = static_cast<int>(i % D);
    const int64_t a0 = s.adj_ptr[n];
    const int deg = static_cast<int>(s.adj_ptr[n + 1] - a0);
    const int64_t row = (int64_t)D * D * a0 + (int64_t)a * D * deg;
    const bool ci = s.mask[i] != 0;
    double ri = res[i];
    for (int jj = 0; jj < D * deg; ++jj) {
      const int64_t j = (int64_t)D * s.adj[a0 + jj / D] + jj % D;
      const bool cj = s.mask[j] != 0;
      const int64_t k = row + jj;
      if (!ci && cj) {
        ri += values[k] * (s.presc[j] - u[j]);
        values[k] = 0.0;
      } else if (ci) {
        values[k] = (i == j) ? 1.0 : 0.0;
      }
    }
    res[i] = ci ? u[i] - s.presc[i] : ri;
  }
}

__global__ void k_constrain(const uint8_t* mask, const double* presc, double* res, const double* u, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (mask[i]) res[i] = u[i] - presc[i];
}

__global__ void k_impose(const uint8_t* mask, const double* presc, double* u, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (mask[i]) u[i] = presc[i];
}

// y = A x over pattern-ordered values: one warp per node (its dim rows are contiguous).
template <int D>
__global__ void __launch_bounds__(256) k_csr_apply(SysView s, const double* __restrict__ values,
                                                   const double* __restrict__ x, double* __restrict__ y,
                                                   const int* skip) {
  if (skip && *skip) return;  // the CG loop's speculative iterations after convergence
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t n = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; n < s.n_nodes; n += warps) {
    const int64_t a0 = s.adj_ptr[n];
    const int deg = static_cast<int>(s.adj_ptr[n + 1] - a0);
    const int len = D * deg;
    double acc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) acc[a] = 0.0;
    for (int jj = lane; jj < len; jj += 32) {
      const double xv = __ldg(&x[(int64_t)D * s.adj[a0 + jj / D] + jj % D]);
#pragma unroll
      for (int a = 0; a < D; ++a) acc[a] += values[(int64_t)D * D * a0 + (int64_t)a * len + jj] * xv;
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double v = acc[a];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) y[D * n + a] = v;
    }
  }
}

// csr_diagonal (krylov.hpp:102-111).
__global__ void k_csr_diagonal(SysView s, const double* values, double* d) {
  const int D = s.dim;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s.n_dof; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / D;
    const int a = static_cast<int>(i % D);
    const int64_t a0 = s.adj_ptr[n];
    const int deg = static_cast<int>(s.adj_ptr[n + 1] - a0);
    const int pos = find_pos(s.adj + a0, deg, static_cast<int32_t>(n));
    double v = 0.0;
    if (pos < deg && s.adj[a0 + pos] == n) v = values[(int64_t)D * D * a0 + (int64_t)a * D * deg + pos * D + a];
    d[i] = v;
  }
}

template <template <int> class K>
struct Dispatch;

inline unsigned node_grid(const System& s, int threads) { return grid_for(s.n_nodes, threads, 148 * 64); }

}  // namespace

void residual(System& s, const double* u, double* r) {
  if (grid_elem_path(s)) {
    grid_residual(s, u, r);
    check_err(s);
    return;
  }
  if (s.dim == 2) launch(*s.ctx, k_residual<2>, node_grid(s, 128), 128, 0, s.view(), u, r);
  else launch(*s.ctx, k_residual<3>, node_grid(s, 128), 128, 0, s.view(), u, r);
  check_err(s);
}

void jacobian(System& s, const double* u, double* values) {
  if (s.dim == 3 && grid_elem_path(s)) {  // 2D keeps the reference's per-element geometry (its solver
    grid_jacobian(s, u, values);           // iteration counts are compared with the reference library)
    check_err(s);
    return;
  }
  if (s.dim == 2) launch(*s.ctx, k_jacobian<2>, node_grid(s, 128), 128, 0, s.view(), u, values);
  else launch(*s.ctx, k_jacobian<3>, node_grid(s, 128), 128, 0, s.view(), u, values);
  check_err(s);
}

void diagonal(System& s, const double* u, double* d) {
  if (grid_elem_path(s)) {
    grid_diagonal(s, u, d);
    check_err(s);
    return;
  }
  if (s.dim == 2) launch(*s.ctx, k_diagonal<2>, node_grid(s, 128), 128, 0, s.view(), u, d);
  else launch(*s.ctx, k_diagonal<3>, node_grid(s, 128), 128, 0, s.view(), u, d);
  check_err(s);
}

// Asynchronous (no error check): used inside Krylov loops; the state was validated at operator
// creation by the diagonal assembly.
void mf_apply_general(System& s, const double* state, const uint8_t* mask, const double* x, double* y) {
  if (grid_elem_path(s)) {
    grid_mf_apply(s, state, mask, x, y);
    return;
  }
  if (s.dim == 2) launch(*s.ctx, k_mf_apply<2>, node_grid(s, 128), 128, 0, s.view(), state, mask, x, y);
  else launch(*s.ctx, k_mf_apply<3>, node_grid(s, 128), 128, 0, s.view(), state, mask, x, y);
}

void history_commit(System& s, const double* u) {
  if (!s.has_history()) return;
  if (s.dim == 3 && grid_elem_path(s)) {
    grid_history_commit(s, u);
    return;
  }
  const unsigned g = grid_for(s.n_elem, 128, 148 * 64);
  if (s.dim == 2) launch(*s.ctx, k_history_commit<2>, g, 128, 0, s.view(), u, s.hist.p);
  else launch(*s.ctx, k_history_commit<3>, g, 128, 0, s.view(), u, s.hist.p);
}

void history_reset(System& s) {
  if (s.has_history()) AFEM_CK(cudaMemsetAsync(s.hist.p, 0, s.hist.bytes(), s.ctx->stream));
}

void eliminate(System& s, double* values, double* residual_, const double* u) {
  launch(*s.ctx, k_eliminate, grid_for(s.n_dof, 256, 148 * 64), 256, 0, s.view(), values, residual_, u);
}

void constrain_residual(System& s, double* residual_, const double* u) {
  launch(*s.ctx, k_constrain, grid_for(s.n_dof, 256, 148 * 64), 256, 0, s.mask.p, s.presc.p, residual_, u, s.n_dof);
}

void impose_dirichlet(System& s, double* u) {
  launch(*s.ctx, k_impose, grid_for(s.n_dof, 256, 148 * 64), 256, 0, s.mask.p, s.presc.p, u, s.n_dof);
}

void csr_apply(System& s, const double* values, const double* x, double* y, const int* skip) {
  const unsigned g = grid_for(s.n_nodes * 32, 256, 148 * 64);
  if (s.dim == 2) launch(*s.ctx, k_csr_apply<2>, g, 256, 0, s.view(), values, x, y, skip);
  else launch(*s.ctx, k_csr_apply<3>, g, 256, 0, s.view(), values, x, y, skip);
}

void csr_diagonal(System& s, const double* values, double* d) {
  launch(*s.ctx, k_csr_diagonal, grid_for(s.n_dof, 256, 148 * 64), 256, 0, s.view(), values, d);
}

}  // namespace afem
