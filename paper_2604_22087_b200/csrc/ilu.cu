// ILU(0) on the device CSR (Ilu0Preconditioner, krylov.hpp:116-192): zero-fill incomplete LU in
// the reference's IKJ order, L unit lower and U sharing the pattern, z = U^-1 L^-1 r.
//
// Row i of the factorisation and of the forward solve depends only on rows k < i that appear in
// row i, so rows are grouped into dependency levels (level(i) = 1 + max level(k), computed once per
// pattern on the host) and one launch per level processes every row of the level, one thread per
// row, in the reference's per-row operation order. The backward solve uses the mirrored levels.
// Inherently sequential across levels (≈ 3 (nx + ny + nz) · dim levels on a grid): this is the
// parity path of the reference's solver menu, not a throughput path.
#include <algorithm>
#include <memory>
#include <vector>

#include "afem_impl.hpp"

namespace afem {

struct IluLevels {
  std::vector<int64_t> lptr, uptr;  // rows of level l: [lptr[l], lptr[l + 1]) in lrows (same for U)
  DevArray<int32_t> lrows, urows;
  DevArray<int64_t> diag;  // value index of each row's diagonal entry
};

namespace {

// Row layout of the pattern-ordered values (afem_impl.hpp): row i = D n + a spans D deg(n) entries
// starting at D^2 adj_ptr[n] + a D deg(n); entry jj has column D adj[adj_ptr[n] + jj / D] + jj % D.
__device__ __forceinline__ void row_span(const SysView& s, int64_t i, int64_t& base, int& len, int64_t& a0) {
  const int D = s.dim;
  const int64_t n = i / D;
  const int a = static_cast<int>(i % D);
  a0 = s.adj_ptr[n];
  const int deg = static_cast<int>(s.adj_ptr[n + 1] - a0);
  len = D * deg;
  base = (int64_t)D * D * a0 + (int64_t)a * len;
}

__device__ __forceinline__ int64_t col_of(const SysView& s, int64_t a0, int jj) {
  return (int64_t)s.dim * s.adj[a0 + jj / s.dim] + jj % s.dim;
}

// IKJ elimination of the rows of one level (krylov.hpp:133-148).
__global__ void k_ilu_factor(SysView s, double* f, const int32_t* rows, int64_t nrows, const int64_t* diag,
                             unsigned long long* bad) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nrows; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = rows[t];
    int64_t base, a0;
    int len;
    row_span(s, i, base, len, a0);
    for (int kk = 0; kk < len; ++kk) {
      const int64_t k = col_of(s, a0, kk);
      if (k >= i) break;
      const double ukk = f[diag[k]];
      if (ukk == 0.0) {
        atomicMin(bad, static_cast<unsigned long long>(k));
        return;
      }
      const double lik = f[base + kk] / ukk;
      f[base + kk] = lik;
      int64_t kbase, ka0;
      int klen;
      row_span(s, k, kbase, klen, ka0);
      const int kd = static_cast<int>(diag[k] - kbase);
      int pos = kk + 1;  // both rows are column-sorted: merge instead of a search per entry
      for (int uk = kd + 1; uk < klen; ++uk) {
        const int64_t j = col_of(s, ka0, uk);
        while (pos < len && col_of(s, a0, pos) < j) ++pos;
        if (pos < len && col_of(s, a0, pos) == j) f[base + pos] -= lik * f[kbase + uk];
      }
    }
    if (f[diag[i]] == 0.0) atomicMin(bad, static_cast<unsigned long long>(i));
  }
}

// Forward substitution with the unit lower factor (krylov.hpp:159-164).
__global__ void k_ilu_lower(SysView s, const double* f, const int32_t* rows, int64_t nrows, const double* r, double* z) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nrows; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = rows[t];
    int64_t base, a0;
    int len;
    row_span(s, i, base, len, a0);
    double sum = r[i];
    for (int k = 0; k < len; ++k) {
      const int64_t c = col_of(s, a0, k);
      if (c >= i) break;
      sum -= f[base + k] * z[c];
    }
    z[i] = sum;
  }
}

// Backward substitution with U (krylov.hpp:165-170).
__global__ void k_ilu_upper(SysView s, const double* f, const int32_t* rows, int64_t nrows, const int64_t* diag,
                            double* z) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nrows; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = rows[t];
    int64_t base, a0;
    int len;
    row_span(s, i, base, len, a0);
    const int dk = static_cast<int>(diag[i] - base);
    double sum = z[i];
    for (int k = dk + 1; k < len; ++k) sum -= f[base + k] * z[col_of(s, a0, k)];
    z[i] = sum / f[base + dk];
  }
}

std::shared_ptr<IluLevels> build_levels(System& s) {
  Ctx& c = *s.ctx;
  const int D = s.dim;
  std::vector<int64_t> ap(s.n_nodes + 1);
  std::vector<int32_t> adj(s.adj.n);
  AFEM_CK(cudaMemcpyAsync(ap.data(), s.adj_ptr.p, ap.size() * 8, cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaMemcpyAsync(adj.data(), s.adj.p, adj.size() * 4, cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  const int64_t n = s.n_dof;
  std::vector<int32_t> lv(n, 0), uv(n, 0);
  std::vector<int64_t> diag(n, -1);
  auto walk = [&](int64_t i, auto&& fn) {
    const int64_t nd = i / D;
    const int a = static_cast<int>(i % D);
    const int deg = static_cast<int>(ap[nd + 1] - ap[nd]);
    const int64_t base = (int64_t)D * D * ap[nd] + (int64_t)a * D * deg;
    for (int jj = 0; jj < D * deg; ++jj) fn(base + jj, (int64_t)D * adj[ap[nd] + jj / D] + jj % D);
  };
  for (int64_t i = 0; i < n; ++i) {
    int l = 0;
    walk(i, [&](int64_t k, int64_t col) {
      if (col < i) l = std::max(l, lv[col] + 1);
      if (col == i) diag[i] = k;
    });
    if (diag[i] < 0) throw FactorizationError("ilu0: structurally missing diagonal at row " + std::to_string(i));
    lv[i] = l;
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    int l = 0;
    walk(i, [&](int64_t, int64_t col) {
      if (col > i) l = std::max(l, uv[col] + 1);
    });
    uv[i] = l;
  }
  auto bucket = [&](const std::vector<int32_t>& lev, std::vector<int64_t>& ptr, DevArray<int32_t>& out) {
    const int nl = lev.empty() ? 0 : *std::max_element(lev.begin(), lev.end()) + 1;
    ptr.assign(nl + 1, 0);
    for (int32_t l : lev) ++ptr[l + 1];
    for (int l = 0; l < nl; ++l) ptr[l + 1] += ptr[l];
    std::vector<int32_t> rows(n);
    std::vector<int64_t> fillp(ptr.begin(), ptr.end() - 1);
    for (int64_t i = 0; i < n; ++i) rows[fillp[lev[i]]++] = static_cast<int32_t>(i);
    out.alloc(std::max<int64_t>(n, 1));
    AFEM_CK(cudaMemcpyAsync(out.p, rows.data(), n * 4, cudaMemcpyHostToDevice, c.stream));
  };
  auto L = std::make_shared<IluLevels>();
  bucket(lv, L->lptr, L->lrows);
  bucket(uv, L->uptr, L->urows);
  L->diag.alloc(n);
  AFEM_CK(cudaMemcpyAsync(L->diag.p, diag.data(), n * 8, cudaMemcpyHostToDevice, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  return L;
}

unsigned grid_rows(int64_t nrows) { return grid_for(nrows, 128, 148 * 16); }

}  // namespace

void Ilu0::setup(System& sys, const double* values) {
  s = &sys;
  if (!sys.ilu_levels) sys.ilu_levels = build_levels(sys);
  const IluLevels& L = *sys.ilu_levels;
  Ctx& c = *sys.ctx;
  f.alloc(sys.nnz);
  AFEM_CK(cudaMemcpyAsync(f.p, values, sys.nnz * 8, cudaMemcpyDeviceToDevice, c.stream));
  DevArray<unsigned long long> bad(1);
  const unsigned long long init = ~0ull;
  AFEM_CK(cudaMemcpyAsync(bad.p, &init, 8, cudaMemcpyHostToDevice, c.stream));
  for (size_t l = 0; l + 1 < L.lptr.size(); ++l) {
    const int64_t nr = L.lptr[l + 1] - L.lptr[l];
    launch(c, k_ilu_factor, grid_rows(nr), 128, 0, sys.view(), f.p, L.lrows.p + L.lptr[l], nr, L.diag.p, bad.p);
  }
  unsigned long long b = 0;
  AFEM_CK(cudaMemcpyAsync(&b, bad.p, 8, cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  if (b != ~0ull) throw FactorizationError("ilu0: zero pivot at row " + std::to_string(b));
}

void Ilu0::apply(const double* r, double* z) const {
  const IluLevels& L = *s->ilu_levels;
  Ctx& c = *s->ctx;
  for (size_t l = 0; l + 1 < L.lptr.size(); ++l) {
    const int64_t nr = L.lptr[l + 1] - L.lptr[l];
    launch(c, k_ilu_lower, grid_rows(nr), 128, 0, s->view(), f.p, L.lrows.p + L.lptr[l], nr, r, z);
  }
  for (size_t l = 0; l + 1 < L.uptr.size(); ++l) {
    const int64_t nr = L.uptr[l + 1] - L.uptr[l];
    launch(c, k_ilu_upper, grid_rows(nr), 128, 0, s->view(), f.p, L.urows.p + L.uptr[l], nr, L.diag.p, z);
  }
}

}  // namespace afem
