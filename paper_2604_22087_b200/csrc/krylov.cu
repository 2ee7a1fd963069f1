// Krylov solvers on the device: Jacobi-preconditioned CG (krylov.hpp:350-408) and restarted,
// left-preconditioned GMRES(m) (krylov.hpp:415-530). The reference orthogonalises with modified
// Gram-Schmidt; here each Arnoldi step is CGS2 (classical Gram-Schmidt twice) in three fused
// kernels — Jacobi + normalisation of the previous basis vector + all first-pass inner products,
// update + all second-pass inner products, update + the new vector's exact norm — with one host
// sync per step (the Givens rotations stay on the host, as in the reference).
//
// CG keeps every scalar (rz, pAp, alpha, beta, the residual history) in device memory. One
// iteration is four launches — operator apply, pAp reduction, the fused x/r/z update with the
// (r.r, r.z) reduction, and the p update — each of which becomes a no-op once the device-side
// `done` flag is set, so the host enqueues chunks of iterations and synchronises once per chunk
// while the iteration count and history stay exact. Observable semantics follow the reference:
// convergence on the recurrence residual, then re-verification with a fresh apply and a restart
// from the true residual if the recurrence drifted; pAp <= 0 reports a failure string;
// b = 0 uses an absolute test.
// Small assembled systems (config 1 is 8 450 dofs) are launch-latency bound: there the whole
// iteration loop runs in ONE persistent cooperative kernel (CSR SpMV warp-per-node, the x/r/z
// update and the p update, three grid syncs per iteration; every block reduces the per-block
// partials in the same fixed order, so the scalars are identical everywhere and deterministic).
#include <cooperative_groups.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <string>

#include "afem_impl.hpp"
#include "reduce.cuh"

namespace afem {

unsigned red_grid(int64_t n);

namespace {

struct CgDev {
  double rz, pap, alpha, beta, denom, rtol;
  int it, max_iter, done, fail, conv, pad;
};

__global__ void k_residual_vec(const double* b, const double* ax, double* r, int64_t n, double* partials,
                               unsigned int* counter, double* out) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = b[i] - ax[i];
    if (r) r[i] = d;
    s += d * d;
  }
  double v[1] = {s};
  if (grid_reduce<1>(v, partials, counter))
    if (threadIdx.x == 0) out[0] = sqrt(v[0]);
}

// p = z = M r; rz = r.z
__global__ void k_cg_start(const double* r, const double* inv, double* p, int64_t n, double* partials,
                           unsigned int* counter, CgDev* st) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double zi = inv ? r[i] * inv[i] : r[i];
    p[i] = zi;
    s += r[i] * zi;
  }
  double v[1] = {s};
  if (grid_reduce<1>(v, partials, counter))
    if (threadIdx.x == 0) {
      st->rz = v[0];
      st->done = 0;
    }
}

__global__ void k_cg_pap(const double* p, const double* ap, int64_t n, double* partials, unsigned int* counter,
                         CgDev* st) {
  if (st->done) return;
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += p[i] * ap[i];
  double v[1] = {s};
  if (grid_reduce<1>(v, partials, counter))
    if (threadIdx.x == 0) st->pap = v[0];
}

// x += alpha p; r -= alpha Ap; (r.r, r.z) with z = M r formed on the fly (never stored). alpha =
// rz / pAp, where pAp was produced by k_cg_pap or fused into the operator apply.
__global__ void k_cg_update(double* x, const double* p, double* r, const double* ap, const double* inv, int64_t n,
                            double* partials, unsigned int* counter, CgDev* st, double* hist) {
  // r -= alpha Ap and (r.r, r.z) with z = M r on the fly; x += alpha p is deferred to k_cg_p, which
  // reads p anyway (the converging iteration's x update is applied by the host loop's epilogue)
  if (st->done) return;
  const double pap = st->pap;
  if (!(pap > 0.0)) {  // krylov.hpp:377-381
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->alpha = 0.0;
      st->fail = 1;
      st->done = 1;
    }
    return;
  }
  const double a = st->rz / pap;
  double rr = 0.0, rz = 0.0;
  // 16-byte vector body (device allocations are 256-byte aligned) + scalar tail
  const int64_t n2 = n / 2;
  double2* r2 = reinterpret_cast<double2*>(r);
  const double2* ap2 = reinterpret_cast<const double2*>(ap);
  const double2* inv2 = reinterpret_cast<const double2*>(inv);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 av = __ldcs(&ap2[i]);
    double2 rv = r2[i];
    rv.x -= a * av.x;
    rv.y -= a * av.y;
    r2[i] = rv;
    double zx = rv.x, zy = rv.y;
    if (inv) {
      const double2 iv = __ldg(&inv2[i]);
      zx *= iv.x;
      zy *= iv.y;
    }
    rr += rv.x * rv.x + rv.y * rv.y;
    rz += rv.x * zx + rv.y * zy;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) {
    const int64_t i = n - 1;
    const double ri = r[i] - a * ap[i];
    r[i] = ri;
    const double zi = inv ? ri * inv[i] : ri;
    rr += ri * ri;
    rz += ri * zi;
  }
  double v[2] = {rr, rz};
  if (grid_reduce<2>(v, partials, counter))
    if (threadIdx.x == 0) {
      const int it = st->it + 1;
      st->it = it;
      st->alpha = a;
      const double h = sqrt(v[0]) / st->denom;
      hist[it] = h;
      if (h <= st->rtol) {
        st->done = 1;
        st->conv = 1;
      } else {
        st->beta = v[1] / st->rz;
        st->rz = v[1];
        if (it >= st->max_iter) st->done = 1;
      }
    }
  (void)x;
  (void)p;
}

// x += alpha p (the deferred update of k_cg_update), then p = M r + beta p
__global__ void k_cg_p(const double* __restrict__ r, const double* __restrict__ inv, double* __restrict__ p,
                       double* __restrict__ x, int64_t n, const CgDev* st) {
  if (st->done) return;
  const double a = st->alpha, b = st->beta;
  const int64_t n2 = n / 2;
  const double2* r2 = reinterpret_cast<const double2*>(r);
  const double2* inv2 = reinterpret_cast<const double2*>(inv);
  double2* p2 = reinterpret_cast<double2*>(p);
  double2* x2 = reinterpret_cast<double2*>(x);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    double2 z = __ldcs(&r2[i]);
    if (inv) {
      const double2 iv = __ldg(&inv2[i]);
      z.x *= iv.x;
      z.y *= iv.y;
    }
    double2 pv = p2[i];
    double2 xv = __ldcs(&x2[i]);
    xv.x += a * pv.x;
    xv.y += a * pv.y;
    __stcs(&x2[i], xv);
    pv.x = z.x + b * pv.x;
    pv.y = z.y + b * pv.y;
    p2[i] = pv;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) {
    const int64_t i = n - 1;
    x[i] += a * p[i];
    p[i] = (inv ? r[i] * inv[i] : r[i]) + b * p[i];
  }
}

// the converging (or last) iteration's deferred x += alpha p (alpha = 0 after a pAp failure)
__global__ void k_cg_x_epilogue(double* __restrict__ x, const double* __restrict__ p, int64_t n, const CgDev* st) {
  const double a = st->alpha;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += a * p[i];
}

__global__ void k_inv_diag(const double* d, double* inv, int64_t n, unsigned long long* first_zero) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = d[i];
    if (v == 0.0) atomicMin(first_zero, static_cast<unsigned long long>(i));
    inv[i] = 1.0 / v;
  }
}

__global__ void k_precond(const double* r, const double* inv, double* z, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = inv ? r[i] * inv[i] : r[i];
}

__global__ void k_scale_into(const double* w, double inv_s, double* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = w[i] / inv_s;
}


// Block sum of NV values (all threads get the result).
template <int NV>
__device__ __forceinline__ void block_allsum(double (&v)[NV], double* sh /* NV * 32 */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double t = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) sh[k * 32 + w] = t;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double t = lane < nw ? sh[k * 32 + lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    v[k] = t;
  }
  __syncthreads();
}

// Fixed-order sum of gridDim.x partials (stride NV), identical in every block.
template <int NV>
__device__ __forceinline__ void grid_partials_sum(const double* part, double (&v)[NV], double* sh) {
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __ldcg(&part[b * NV + k]);
  block_allsum<NV>(v, sh);
}

// The whole Jacobi-PCG iteration loop for an assembled (CSR) operator; st holds rz etc. from
// k_cg_start. Writes hist[it] per iteration and the final state back to st.
template <int D>
__global__ void __launch_bounds__(256) k_cg_persistent(SysView s, const double* __restrict__ vals, double* x,
                                                       double* r, double* p, double* ap, const double* inv,
                                                       int64_t n, CgDev* st, double* hist, double* part_a,
                                                       double* part_b) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[2 * 32];
  const int lane = threadIdx.x & 31;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t warp = tid >> 5, nwarps = nth >> 5;
  double rz = st->rz;
  const double denom = st->denom, rtol = st->rtol;
  const int max_iter = st->max_iter;
  int it = st->it, fail = 0, conv = 0;
  while (true) {
    // (1) ap = A p, one warp per node (its D rows are contiguous), and p.ap
    double pap_loc = 0.0;
    for (int64_t nd = warp; nd < s.n_nodes; nd += nwarps) {
      const int64_t a0 = s.adj_ptr[nd];
      const int deg = static_cast<int>(s.adj_ptr[nd + 1] - a0);
      const int len = D * deg;
      double acc[D];
#pragma unroll
      for (int a = 0; a < D; ++a) acc[a] = 0.0;
      for (int jj = lane; jj < len; jj += 32) {
        const double xv = __ldcg(&p[(int64_t)D * s.adj[a0 + jj / D] + jj % D]);
#pragma unroll
        for (int a = 0; a < D; ++a) acc[a] += vals[(int64_t)D * D * a0 + (int64_t)a * len + jj] * xv;
      }
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double v = acc[a];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {
          ap[D * nd + a] = v;
          pap_loc += __ldcg(&p[D * nd + a]) * v;
        }
      }
    }
    double t1[1] = {pap_loc};
    block_allsum<1>(t1, sh);
    if (threadIdx.x == 0) part_a[blockIdx.x] = t1[0];
    grid.sync();
    grid_partials_sum<1>(part_a, t1, sh);
    const double pap = t1[0];
    if (!(pap > 0.0)) {  // krylov.hpp:377-381
      fail = 1;
      break;
    }
    const double alpha = rz / pap;
    // (2) x += alpha p; r -= alpha ap; (r.r, r.z)
    double rr = 0.0, rzn = 0.0;
    for (int64_t i = tid; i < n; i += nth) {
      const double pi = __ldcg(&p[i]);
      x[i] += alpha * pi;
      const double ri = r[i] - alpha * __ldcg(&ap[i]);
      r[i] = ri;
      const double zi = inv ? ri * inv[i] : ri;
      rr += ri * ri;
      rzn += ri * zi;
    }
    double t2[2] = {rr, rzn};
    block_allsum<2>(t2, sh);
    if (threadIdx.x == 0) {
      part_b[2 * blockIdx.x] = t2[0];
      part_b[2 * blockIdx.x + 1] = t2[1];
    }
    grid.sync();
    grid_partials_sum<2>(part_b, t2, sh);
    ++it;
    const double h = sqrt(t2[0]) / denom;
    if (blockIdx.x == 0 && threadIdx.x == 0) hist[it] = h;
    if (h <= rtol) {
      conv = 1;
      break;
    }
    const double beta = t2[1] / rz;
    rz = t2[1];
    if (it >= max_iter) break;
    // (3) p = z + beta p (same element mapping as (2): own elements only)
    for (int64_t i = tid; i < n; i += nth) {
      const double zi = inv ? r[i] * inv[i] : r[i];
      p[i] = zi + beta * __ldcg(&p[i]);
    }
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->it = it;
    st->rz = rz;
    st->fail = fail;
    st->conv = conv;
    st->done = 1;
  }
}

// Cooperative launch of k_cg_persistent (false when the device / size does not qualify).
bool cg_persistent(Operator& op, double* x, double* r, double* p, double* ap, const double* inv, CgDev* st,
                   double* hist) {
  static const bool off = std::getenv("AFEM_NO_PERSISTENT_CG") != nullptr;
  const double* vals = op.csr_values();
  System& s = *op.sys;
  Ctx& c = *s.ctx;
  // grid-wide syncs beat kernel launches only while an iteration is short: measured crossover between
  // 3.8 M nonzeros (22 vs 30 us per iteration) and 8.7 M (41 vs 38 us); 348 vs 146 us at 67 M
  if (off || !vals || s.nnz > 6000000) return false;
  int coop = 0;
  AFEM_CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c.device));
  if (!coop) return false;
  auto kern = s.dim == 2 ? k_cg_persistent<2> : k_cg_persistent<3>;
  int per_sm = 0;
  AFEM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
  if (per_sm < 1) return false;
  // one warp per node, at most two blocks per SM (measured best on config 1: 10.4 us per iteration)
  static const int cap = std::getenv("AFEM_PCG_BLOCKS") ? std::atoi(std::getenv("AFEM_PCG_BLOCKS")) : 2 * c.num_sms;
  const int64_t want = (s.n_nodes * 32 + 255) / 256;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(want, cap),
                                                                               (int64_t)per_sm * c.num_sms)));
  DevArray<double>& parts = c.pcg_parts;
  if (parts.n < (size_t)3 * blocks) parts.alloc(3 * (size_t)blocks);
  SysView v = s.view();
  int64_t n = op.n;
  double* part_a = parts.p;
  double* part_b = parts.p + blocks;
  void* args[] = {&v, (void*)&vals, &x, &r, &p, &ap, (void*)&inv, &n, &st, &hist, &part_a, &part_b};
  AFEM_CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), blocks, 256, args, 0, c.stream));
  ++c.launches;
  return true;
}


// BiCGStab vector steps (krylov.hpp:557-598)
__global__ void k_bicg_p(const double* __restrict__ r, double* __restrict__ p, const double* __restrict__ v, double beta,
                         double omega, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = r[i] + beta * (p[i] - omega * v[i]);
}

__global__ void k_bicg_s(const double* __restrict__ r, const double* __restrict__ v, double alpha, double* __restrict__ s,
                         int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s[i] = r[i] - alpha * v[i];
}

__global__ void k_bicg_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ phat,
                          const double* __restrict__ shat, const double* __restrict__ s, const double* __restrict__ t,
                          double alpha, double omega, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * phat[i] + omega * shat[i];
    r[i] = s[i] - omega * t[i];
  }
}

struct Timer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double seconds() const { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
};

template <class T>
T fetch(Ctx& c, const T* d) {
  T h{};
  AFEM_CK(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  return h;
}

// ||b - A x|| via a fresh apply; optionally keeps r = b - A x.
double residual_norm(Operator& op, const double* b, const double* x, double* scratch, double* r) {
  Ctx& c = *op.sys->ctx;
  op.apply(x, scratch);
  launch(c, k_residual_vec, red_grid(op.n), kRedThreads, 0, b, scratch, r, op.n, c.red_partials.p,
         c.red_counter.p, c.red_out.p);
  return fetch(c, c.red_out.p);
}

}  // namespace

double Operator::inner(const double* a, const double* b) { return dot(*sys->ctx, a, b, n); }
void Operator::inner_dev(const double* a, const double* b, double* out_dev) { dot_dev(*sys->ctx, a, b, n, out_dev); }
double Operator::resid(const double* b, const double* x, double* scratch, double* r) {
  return residual_norm(*this, b, x, scratch, r);
}

namespace {

// JacobiPreconditioner::from_diagonal (krylov.hpp:83-92).
void jacobi_inverse(Operator& op, DevArray<double>& inv) {
  Ctx& c = *op.sys->ctx;
  DevArray<double> d(op.n);
  op.diagonal(d.p);
  inv.alloc(op.n);
  DevArray<unsigned long long> fz(1);
  const unsigned long long init = ~0ull;
  AFEM_CK(cudaMemcpyAsync(fz.p, &init, 8, cudaMemcpyHostToDevice, c.stream));
  launch(c, k_inv_diag, grid_for(op.n, 256, 148 * 16), 256, 0, d.p, inv.p, op.n, fz.p);
  const unsigned long long z = fetch(c, fz.p);
  if (z != ~0ull) throw FactorizationError("jacobi: zero diagonal at row " + std::to_string(z));
}

void cg(Operator& op, const SolverCfg& cfg, const double* b, double* x, const double* inv, SolveReport& rep) {
  Ctx& c = *op.sys->ctx;
  const int64_t n = op.n;
  DevArray<double> r(n), p(n), ap(n), scratch(n), hist(cfg.max_iter + 2);
  DevArray<CgDev> st(1);
  const double bnorm = std::sqrt(dot(c, b, b, n));
  const double denom = bnorm > 0.0 ? bnorm : 1.0;
  double h0 = residual_norm(op, b, x, ap.p, r.p) / denom;
  rep.history.assign(1, h0);
  CgDev hs{};
  hs.denom = denom;
  hs.rtol = cfg.rtol;
  hs.max_iter = cfg.max_iter;
  hs.done = 1;
  AFEM_CK(cudaMemcpyAsync(st.p, &hs, sizeof hs, cudaMemcpyHostToDevice, c.stream));
  const unsigned rg = red_grid(n), eg = grid_for(n, 256, 148 * 16);
  while (true) {
    if (rep.history.back() > cfg.rtol && rep.iterations < cfg.max_iter) {
      launch(c, k_cg_start, rg, kRedThreads, 0, r.p, inv, p.p, n, c.red_partials.p, c.red_counter.p, st.p);
      int chunk = 4;
      const bool persistent = cg_persistent(op, x, r.p, p.p, ap.p, inv, st.p, hist.p);
      if (persistent) {
        hs = fetch(c, st.p);
      } else {
        auto enqueue = [&](int cnt) {
          for (int k = 0; k < cnt; ++k) {
            // fused operators write p^T A p straight into st->pap; others get the reduction kernel
            double* pap_dev = reinterpret_cast<double*>(reinterpret_cast<char*>(st.p) + offsetof(CgDev, pap));
            if (!op.apply_dot(p.p, ap.p, pap_dev)) {
              op.apply(p.p, ap.p);
              launch(c, k_cg_pap, rg, kRedThreads, 0, p.p, ap.p, n, c.red_partials.p, c.red_counter.p, st.p);
            }
            launch(c, k_cg_update, rg, kRedThreads, 0, x, p.p, r.p, ap.p, inv, n, c.red_partials.p,
                   c.red_counter.p, st.p, hist.p);
            launch(c, k_cg_p, eg, 256, 0, r.p, inv, p.p, x, n, st.p);
          }
        };
        // Operators that can skip on the device-side done flag get one chunk enqueued ahead of the
        // host's check of the previous one, so the GPU never drains at a chunk boundary; the
        // speculative iterations after convergence are no-ops (every kernel tests the flag).
        const int* done_dev = reinterpret_cast<const int*>(reinterpret_cast<const char*>(st.p) + offsetof(CgDev, done));
        const bool spec = op.set_skip(done_dev);
        if (!spec) {
          while (true) {
            enqueue(chunk);
            hs = fetch(c, st.p);
            if (hs.done) break;
            chunk = std::min(chunk * 2, 64);
          }
        } else {
          // the iteration loop as a CUDA graph of kGraphIters iterations (captured once per solve):
          // one launch per chunk instead of four per iteration, so host hiccups cannot drain the GPU
          constexpr int kGraphIters = 16;
          CgDev* hst = static_cast<CgDev*>(c.pinned_snap(2 * sizeof(CgDev)));  // snapshots of chunks k, k + 1
          cudaEvent_t* ev = c.snap_ev;
          cudaGraph_t graph = nullptr;
          cudaGraphExec_t exec = nullptr;
          // on every exit (exceptions included): the speculative skip flag points into this solve's
          // CgDev, so it is detached before st is freed; graph objects are released
          ScopeExit cleanup([&] {
            op.set_skip(nullptr);
            if (exec) cudaGraphExecDestroy(exec);
            if (graph) cudaGraphDestroy(graph);
          });
          int64_t per_graph = 0;
          {
            CaptureGuard cap(c);  // instantiated graph is launched on the context stream
            enqueue(kGraphIters);
            graph = cap.end(&per_graph);
          }
          AFEM_CK(cudaGraphInstantiate(&exec, graph, 0));
          auto run = [&] {
            AFEM_CK(cudaGraphLaunch(exec, c.stream));
            c.launches += per_graph;
          };
          // two chunks queued ahead of the host's check: a host stall shorter than two chunks
          // (about 5 ms at 128^3) never drains the GPU; chunks past convergence are no-ops
          auto run_snap = [&](int slot) {
            run();
            AFEM_CK(cudaMemcpyAsync(hst + slot, st.p, sizeof(CgDev), cudaMemcpyDeviceToHost, c.stream));
            AFEM_CK(cudaEventRecord(ev[slot], c.stream));
          };
          run_snap(0);
          run_snap(1);
          for (int k = 0;; ++k) {
            AFEM_CK(cudaEventSynchronize(ev[k & 1]));
            hs = hst[k & 1];
            if (hs.done) break;
            run_snap(k & 1);
          }
          AFEM_CK(cudaStreamSynchronize(c.stream));
          hs = fetch(c, st.p);
        }
      }
      if (!persistent) launch(c, k_cg_x_epilogue, eg, 256, 0, x, p.p, n, st.p);
      const int it0 = rep.iterations;
      rep.iterations = hs.it;
      if (hs.it > it0) {
        rep.history.resize(hs.it + 1);
        AFEM_CK(cudaMemcpyAsync(rep.history.data() + it0 + 1, hist.p + it0 + 1, (hs.it - it0) * sizeof(double),
                                cudaMemcpyDeviceToHost, c.stream));
        AFEM_CK(cudaStreamSynchronize(c.stream));
      }
      if (hs.fail)
        rep.failure = "cg: operator not positive definite (p^T A p <= 0 at iteration " +
                      std::to_string(rep.iterations + 1) + ")";
    }
    const double true_rres = residual_norm(op, b, x, scratch.p, nullptr) / denom;
    rep.history.back() = true_rres;
    if (true_rres <= cfg.rtol) {
      rep.converged = rep.failure.empty();
      break;
    }
    if (!rep.failure.empty() || rep.iterations >= cfg.max_iter) break;
    // recurrence drifted: restart from the fresh residual (krylov.hpp:402-404)
    residual_norm(op, b, x, ap.p, r.p);
    hs.done = 1;
    hs.conv = 0;
    AFEM_CK(cudaMemcpyAsync(&reinterpret_cast<CgDev*>(st.p)->conv, &hs.conv, sizeof(int), cudaMemcpyHostToDevice,
                            c.stream));
  }
}


// ---- fused Arnoldi step (GMRES): classical Gram-Schmidt with one re-orthogonalisation (CGS2)
// in three passes over the basis instead of 2(j+1) modified-Gram-Schmidt kernels. Every pass
// reads the j+1 basis vectors once and reduces all its inner products in the same launch
// (per-block partials, then the last block sums them in a fixed order: deterministic).
constexpr int kGmMax = 32;  // inner products one pass carries (basis vectors + the norm)

// Block sums of acc[0..nv) -> part[k * gridDim.x + block]; the last block to finish writes the
// fixed-order grid sums to out[0..nv).
// WithExtra: one more value (extra) in slot nv.
template <bool WithExtra>
__device__ __forceinline__ void gm_reduce(const double (&acc)[kGmMax], int nv, double extra, double* part,
                                          unsigned int* counter, double* out) {
  __shared__ double sh[kGmMax + 1][kRedThreads / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < kGmMax; ++k) {
    if (k < nv) {
      double t = acc[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) sh[k][w] = t;
    }
  }
  if (WithExtra) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) extra += __shfl_xor_sync(0xffffffffu, extra, o);
    if (lane == 0) sh[nv][w] = extra;
    ++nv;
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double t = 0.0;
    for (int q = 0; q < nw; ++q) t += sh[threadIdx.x][q];
    part[threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int k = w; k < nv; k += nw) {  // one warp per inner product, fixed lane assignment
    double t = 0.0;
    for (unsigned b = lane; b < gridDim.x; b += 32) t += __ldcg(&part[k * gridDim.x + b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) out[k] = t;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// Passes 1 and 2: one row per thread; the row's products with the (up to 32) basis vectors are
// reduced across the warp by a transpose-reduction (5 halving exchange steps, 31 shuffles in all),
// after which lane k holds the warp's sum for vector k and keeps ONE running partial sum. Every
// load of a row is independent (all 32 in flight) and no per-vector accumulators live across the
// row loop — the per-thread form with 32 accumulators ran at 1.9-3.4 TB/s. Fixed shuffle order and
// fixed per-CTA / cross-CTA reduction order: deterministic.
__device__ __forceinline__ double warp_transpose_reduce(double (&p)[kGmMax]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < o; ++k) {
      const double send = upper ? p[k] : p[k + o];
      const double keep = upper ? p[k + o] : p[k];
      p[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return p[0];  // lane L: the sum over the warp's lanes of p[L]
}

// Block sum of every lane's single partial (lane k = vector k) -> part[k * gridDim.x + block]; the
// last block sums the partials of each vector in block order.
__device__ __forceinline__ void gm_lane_reduce(double acc, int nv, double* part, unsigned int* counter,
                                               double* out) {
  __shared__ double sh[kRedThreads / 32][32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  sh[w][lane] = acc;
  __syncthreads();
  if (threadIdx.x < nv) {
    double t = 0.0;
    for (int q = 0; q < nw; ++q) t += sh[q][threadIdx.x];
    part[threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int k = w; k < nv; k += nw) {
    double t = 0.0;
    for (unsigned b = lane; b < gridDim.x; b += 32) t += __ldcg(&part[k * gridDim.x + b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) out[k] = t;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// Step j's basis vector V_{nv-1} arrives unnormalised (pass 3 of the previous step writes
// w - V h2 and its exact norm s): A V_{nv-1} was applied to it, so w = M^-1 src / s, and V_{nv-1} is
// normalised in place here (s = 1 for the restart vector). Then h1[k] = V_k . w over the owned rows
// [off, n), k < nv. Jacobi: inv; else src is already preconditioned and w == src.
__global__ void __launch_bounds__(kRedThreads) k_gm_pass1(const double* __restrict__ src, const double* __restrict__ inv,
                                                          double* w, double* V, int64_t ld, int nv, double s_last,
                                                          int64_t n, int64_t off, double* part, unsigned int* counter,
                                                          double* h1) {
  const int lane = threadIdx.x & 31;
  const double rs = 1.0 / s_last;  // one division per thread, not two per row (fp64 division is slow)
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // whole warps iterate (rows past n contribute zeros) so the shuffles always see 32 lanes
  const int64_t n_up = (n + 31) / 32 * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i - lane < n_up; i += stride) {
    const bool in = i < n;
    double wi = 0.0;
    if (in) {
      wi = src[i];
      if (inv) wi *= inv[i];
      if (s_last != 1.0) wi *= rs;
      if (inv || s_last != 1.0) w[i] = wi;
    }
    const double wd = in && i >= off ? wi : 0.0;
    double p[kGmMax];
#pragma unroll
    for (int k = 0; k < kGmMax; ++k) p[k] = (k < nv && in) ? __ldcs(&V[k * ld + i]) : 0.0;  // all loads first
    if (s_last != 1.0 && in) {  // normalise the last vector in place (after the loads: no aliasing barrier)
#pragma unroll
      for (int k = 0; k < kGmMax; ++k)
        if (k == nv - 1) {
          p[k] *= rs;
          V[k * ld + i] = p[k];
        }
    }
#pragma unroll
    for (int k = 0; k < kGmMax; ++k) p[k] *= wd;
    acc += warp_transpose_reduce(p);
  }
  gm_lane_reduce(lane < nv ? acc : 0.0, nv, part, counter, h1);
}

// w -= V h1 (in place); h2[k] = V_k . w (k < nv), owned rows. The row's basis values stay in
// registers between the update and the products (V is read once).
__global__ void __launch_bounds__(kRedThreads) k_gm_pass2(double* w, const double* __restrict__ V, int64_t ld, int nv,
                                                          const double* __restrict__ h1, int64_t n, int64_t off,
                                                          double* part, unsigned int* counter, double* h2) {
  __shared__ double hs[kGmMax];
  if (threadIdx.x < kGmMax) hs[threadIdx.x] = threadIdx.x < nv ? h1[threadIdx.x] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n_up = (n + 31) / 32 * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i - lane < n_up; i += stride) {
    const bool in = i < n;
    double p[kGmMax];
#pragma unroll
    for (int k = 0; k < kGmMax; ++k) p[k] = (k < nv && in) ? __ldcs(&V[k * ld + i]) : 0.0;
    double wi = in ? w[i] : 0.0;
#pragma unroll
    for (int k = 0; k < kGmMax; ++k) wi -= hs[k] * p[k];
    if (in) w[i] = wi;
    const double wd = in && i >= off ? wi : 0.0;
#pragma unroll
    for (int k = 0; k < kGmMax; ++k) p[k] *= wd;
    acc += warp_transpose_reduce(p);
  }
  gm_lane_reduce(lane < nv ? acc : 0.0, nv, part, counter, h2);
}

// vnext = w - V h2 (left unnormalised: pass 1 of the next step divides by its norm) and
// vn2[0] = |vnext|^2 over the owned rows, reduced exactly (the H subdiagonal is the true norm of
// the twice-orthogonalised vector, as in the reference's MGS); block 0 writes hcol = h1 + h2.
__global__ void __launch_bounds__(kRedThreads) k_gm_pass3(const double* __restrict__ w, double* __restrict__ vnext,
                                                          const double* __restrict__ V, int64_t ld, int nv,
                                                          const double* __restrict__ h1, const double* __restrict__ h2,
                                                          double* hcol, int64_t n, int64_t off, double* part,
                                                          unsigned int* counter, double* vn2) {
  __shared__ double hs[kGmMax];
  if (threadIdx.x < nv) hs[threadIdx.x] = h2[threadIdx.x];
  if (blockIdx.x == 0 && threadIdx.x < nv) hcol[threadIdx.x] = h1[threadIdx.x] + h2[threadIdx.x];
  __syncthreads();
  double acc[kGmMax];
  acc[0] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double wi = w[i];
#pragma unroll
    for (int k = 0; k < kGmMax; ++k)
      if (k < nv) wi -= hs[k] * __ldcs(&V[k * ld + i]);
    vnext[i] = wi;
    if (i >= off) acc[0] += wi * wi;
  }
  gm_reduce<false>(acc, 1, 0.0, part, counter, vn2);
}

// x += sum_k y_k V_k in the order of the reference's sequential axpys (krylov.hpp:517-519)
__global__ void k_gm_update_x(double* x, const double* __restrict__ V, int64_t ld, const double* __restrict__ y,
                              int cols, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = x[i];
    for (int k = 0; k < cols; ++k) s += y[k] * V[k * ld + i];
    x[i] = s;
  }
}

// The preconditioner of a solve: Jacobi (inverse diagonal, fused into the CG kernels), ILU(0), or none.
struct Pc {
  const double* inv = nullptr;
  const Ilu0* ilu = nullptr;
  void apply(Ctx& c, const double* in, double* out, int64_t n) const {
    if (ilu) ilu->apply(in, out);
    else launch(c, k_precond, grid_for(n, 256, 148 * 16), 256, 0, in, inv, out, n);
  }
};

// cg (krylov.hpp:350-408) with a general preconditioner (ILU(0)): host scalars, one sync per dot.
void cg_generic(Operator& op, const SolverCfg& cfg, const double* b, double* x, const Pc& pc, SolveReport& rep) {
  Ctx& c = *op.sys->ctx;
  const int64_t n = op.n;
  DevArray<double> r(n), z(n), p(n), ap(n), scratch(n);
  const double bnorm = std::sqrt(dot(c, b, b, n));
  const double denom = bnorm > 0.0 ? bnorm : 1.0;
  rep.history.push_back(residual_norm(op, b, x, ap.p, r.p) / denom);
  while (true) {
    if (rep.history.back() > cfg.rtol && rep.iterations < cfg.max_iter) {
      pc.apply(c, r.p, z.p, n);
      copy(c, z.p, p.p, n);
      double rz = dot(c, r.p, z.p, n);
      while (rep.iterations < cfg.max_iter && rep.history.back() > cfg.rtol) {
        op.apply(p.p, ap.p);
        const double pap = dot(c, p.p, ap.p, n);
        if (!(pap > 0.0)) {
          rep.failure = "cg: operator not positive definite (p^T A p <= 0 at iteration " +
                        std::to_string(rep.iterations + 1) + ")";
          break;
        }
        const double alpha = rz / pap;
        axpy(c, alpha, p.p, x, n);
        axpy(c, -alpha, ap.p, r.p, n);
        ++rep.iterations;
        rep.history.push_back(std::sqrt(dot(c, r.p, r.p, n)) / denom);
        if (rep.history.back() <= cfg.rtol) break;
        pc.apply(c, r.p, z.p, n);
        const double rz_new = dot(c, r.p, z.p, n);
        const double beta = rz_new / rz;
        rz = rz_new;
        launch(c, k_bicg_p, grid_for(n, 256, 148 * 16), 256, 0, z.p, p.p, z.p, beta, 0.0, n);  // p = z + beta p
      }
    }
    const double true_rres = residual_norm(op, b, x, scratch.p, nullptr) / denom;
    rep.history.back() = true_rres;
    if (true_rres <= cfg.rtol) {
      rep.converged = rep.failure.empty();
      break;
    }
    if (!rep.failure.empty() || rep.iterations >= cfg.max_iter) break;
    residual_norm(op, b, x, ap.p, r.p);  // krylov.hpp:402-404
  }
}

void gmres(Operator& op, const SolverCfg& cfg, const double* b, double* x, const Pc& pc, SolveReport& rep) {
  Ctx& c = *op.sys->ctx;
  const int64_t n = op.n;
  const int restart = static_cast<int>(std::min<int64_t>(cfg.restart, n));
  const unsigned eg = grid_for(n, 256, 148 * 16);
  DevArray<double> tmp(n), r(n), w(n), scratch(n), V(static_cast<size_t>(restart + 1) * n);
  DevArray<double> hcol(restart + 2);
  auto vec = [&](int k) { return V.p + static_cast<int64_t>(k) * n; };
  // fused CGS2 Arnoldi (one pass carries at most kGmMax inner products); AFEM_GMRES_MGS=1 keeps the
  // reference's modified Gram-Schmidt kernel by kernel (A/B measurements)
  static const bool force_mgs = std::getenv("AFEM_GMRES_MGS") != nullptr;
  const bool fused = !force_mgs && restart + 1 <= kGmMax;
  const unsigned rg = red_grid(n);
  const int64_t off = op.dot_begin();
  DevArray<double> part(fused ? static_cast<size_t>(rg) * kGmMax : 0), h1(kGmMax), h2(kGmMax), yd(restart);
  double s_last = 1.0;  // norm of the unnormalised last basis vector (fused path)
  DevArray<unsigned int> ctr(1);
  AFEM_CK(cudaMemsetAsync(ctr.p, 0, sizeof(unsigned int), c.stream));
  const double bnorm = std::sqrt(op.inner(b, b));
  const double denom = bnorm > 0.0 ? bnorm : 1.0;
  pc.apply(c, b, tmp.p, n);
  const double pnorm = std::sqrt(op.inner(tmp.p, tmp.p));
  const double pdenom = pnorm > 0.0 ? pnorm : 1.0;
  std::vector<double> h(static_cast<size_t>(restart + 1) * restart, 0.0), cs(restart), sn(restart), g(restart + 1);
  auto H = [&](int i, int j) -> double& { return h[static_cast<size_t>(i) * restart + j]; };

  double true_rres = op.resid(b, x, tmp.p, r.p) / denom;
  pc.apply(c, r.p, w.p, n);
  rep.history.push_back(std::sqrt(op.inner(w.p, w.p)) / pdenom);

  while (true_rres > cfg.rtol && rep.iterations < cfg.max_iter && rep.failure.empty()) {
    pc.apply(c, r.p, w.p, n);
    const double beta = std::sqrt(op.inner(w.p, w.p));
    if (beta == 0.0) break;
    const double target_est = beta * std::min(1.0, 0.5 * cfg.rtol / true_rres);  // krylov.hpp:454
    launch(c, k_scale_into, eg, 256, 0, w.p, beta, vec(0), n);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int j = 0, cols = 0;
    for (; j < restart && rep.iterations < cfg.max_iter; ++j) {
      op.apply(vec(j), tmp.p);
      std::vector<double> hc(j + 2);
      double hnext;
      if (fused) {
        // CGS2 Arnoldi step: three passes over V, allreduced per-pass scalars, one host sync
        const int nv = j + 1;
        if (!pc.inv) pc.apply(c, tmp.p, w.p, n);
        launch(c, k_gm_pass1, rg, kRedThreads, 0, pc.inv ? tmp.p : w.p, pc.inv, w.p, V.p, n, nv,
               j == 0 ? 1.0 : s_last, n, off, part.p, ctr.p, h1.p);
        op.allreduce_dev(h1.p, nv);
        launch(c, k_gm_pass2, rg, kRedThreads, 0, w.p, V.p, n, nv, h1.p, n, off, part.p, ctr.p, h2.p);
        op.allreduce_dev(h2.p, nv);
        launch(c, k_gm_pass3, rg, kRedThreads, 0, w.p, vec(j + 1), V.p, n, nv, h1.p, h2.p, hcol.p, n, off, part.p,
               ctr.p, hcol.p + nv);
        op.allreduce_dev(hcol.p + nv, 1);
        AFEM_CK(cudaMemcpyAsync(hc.data(), hcol.p, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        AFEM_CK(cudaStreamSynchronize(c.stream));
        hnext = std::sqrt(hc[j + 1]);
        s_last = hnext;
      } else {
        pc.apply(c, tmp.p, w.p, n);
        for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt, scalars stay on the device
          op.inner_dev(vec(i), w.p, hcol.p + i);
          add_scaled_dev(c, hcol.p + i, -1.0, vec(i), w.p, n);
        }
        op.inner_dev(w.p, w.p, hcol.p + j + 1);
        AFEM_CK(cudaMemcpyAsync(hc.data(), hcol.p, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        AFEM_CK(cudaStreamSynchronize(c.stream));
        hnext = std::sqrt(hc[j + 1]);
      }
      for (int i = 0; i <= j; ++i) H(i, j) = hc[i];
      H(j + 1, j) = hnext;
      const bool happy = hnext <= beta * 1e-16;
      if (!happy && !fused) launch(c, k_scale_into, eg, 256, 0, w.p, hnext, vec(j + 1), n);
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * H(i, j) + sn[i] * H(i + 1, j);
        H(i + 1, j) = -sn[i] * H(i, j) + cs[i] * H(i + 1, j);
        H(i, j) = t;
      }
      const double rr = std::hypot(H(j, j), H(j + 1, j));
      if (rr == 0.0) {
        cs[j] = 1.0;
        sn[j] = 0.0;
      } else {
        cs[j] = H(j, j) / rr;
        sn[j] = H(j + 1, j) / rr;
      }
      H(j, j) = rr;
      H(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] *= cs[j];
      ++rep.iterations;
      cols = j + 1;
      const double est = std::abs(g[j + 1]);
      rep.history.push_back(est / pdenom);
      if (est <= target_est || happy) {
        ++j;
        break;
      }
    }
    std::vector<double> y(cols, 0.0);
    for (int i = cols - 1; i >= 0; --i) {
      double s = g[i];
      for (int k = i + 1; k < cols; ++k) s -= H(i, k) * y[k];
      if (H(i, i) == 0.0) {
        rep.failure = "gmres: singular least-squares system in restart cycle";
        break;
      }
      y[i] = s / H(i, i);
    }
    if (!rep.failure.empty()) break;
    if (cols > 0) {
      AFEM_CK(cudaMemcpyAsync(yd.p, y.data(), cols * sizeof(double), cudaMemcpyHostToDevice, c.stream));
      launch(c, k_gm_update_x, eg, 256, 0, x, V.p, n, yd.p, cols, n);
      AFEM_CK(cudaStreamSynchronize(c.stream));  // y is a host temporary
    }
    true_rres = op.resid(b, x, tmp.p, r.p) / denom;
  }
  true_rres = op.resid(b, x, scratch.p, nullptr) / denom;
  rep.history.push_back(true_rres);
  rep.converged = rep.failure.empty() && true_rres <= cfg.rtol;
}

// bicgstab (krylov.hpp:535-620): scalars on the host (one sync per dot); same breakdown messages,
// early exit on a small s, true-residual re-verification and restart from the fresh residual.
void bicgstab(Operator& op, const SolverCfg& cfg, const double* b, double* x, const Pc& pc, SolveReport& rep) {
  Ctx& c = *op.sys->ctx;
  const int64_t n = op.n;
  const unsigned eg = grid_for(n, 256, 148 * 16);
  DevArray<double> r(n), rhat(n), p(n), v(n), sv(n), t(n), phat(n), shat(n);
  fill(c, 0.0, p.p, n);
  fill(c, 0.0, v.p, n);
  const double bnorm = std::sqrt(op.inner(b, b));
  const double denom = bnorm > 0.0 ? bnorm : 1.0;
  rep.history.push_back(op.resid(b, x, t.p, r.p) / denom);
  copy(c, r.p, rhat.p, n);
  auto precond = [&](const double* in, double* out) { pc.apply(c, in, out, n); };
  while (true) {
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    while (rep.history.back() > cfg.rtol && rep.iterations < cfg.max_iter) {
      const double rho_new = op.inner(rhat.p, r.p);
      if (rho_new == 0.0) {
        rep.failure = "bicgstab: rho breakdown at iteration " + std::to_string(rep.iterations + 1);
        break;
      }
      const double beta = (rho_new / rho) * (alpha / omega);
      rho = rho_new;
      launch(c, k_bicg_p, eg, 256, 0, r.p, p.p, v.p, beta, omega, n);
      precond(p.p, phat.p);
      op.apply(phat.p, v.p);
      const double rhat_v = op.inner(rhat.p, v.p);
      if (rhat_v == 0.0) {
        rep.failure = "bicgstab: rhat^T v breakdown at iteration " + std::to_string(rep.iterations + 1);
        break;
      }
      alpha = rho / rhat_v;
      launch(c, k_bicg_s, eg, 256, 0, r.p, v.p, alpha, sv.p, n);
      if (std::sqrt(op.inner(sv.p, sv.p)) / denom <= cfg.rtol) {
        axpy(c, alpha, phat.p, x, n);
        copy(c, sv.p, r.p, n);
        ++rep.iterations;
        rep.history.push_back(std::sqrt(op.inner(r.p, r.p)) / denom);
        break;
      }
      precond(sv.p, shat.p);
      op.apply(shat.p, t.p);
      const double tt = op.inner(t.p, t.p);
      if (tt == 0.0) {
        rep.failure = "bicgstab: omega breakdown (t = 0) at iteration " + std::to_string(rep.iterations + 1);
        break;
      }
      omega = op.inner(t.p, sv.p) / tt;
      if (omega == 0.0) {
        rep.failure = "bicgstab: omega breakdown at iteration " + std::to_string(rep.iterations + 1);
        break;
      }
      launch(c, k_bicg_xr, eg, 256, 0, x, r.p, phat.p, shat.p, sv.p, t.p, alpha, omega, n);
      ++rep.iterations;
      rep.history.push_back(std::sqrt(op.inner(r.p, r.p)) / denom);
    }
    const double true_rres = op.resid(b, x, t.p, nullptr) / denom;
    rep.history.back() = true_rres;
    if (true_rres <= cfg.rtol) {
      rep.converged = rep.failure.empty();
      break;
    }
    if (!rep.failure.empty() || rep.iterations >= cfg.max_iter) break;
    op.resid(b, x, t.p, r.p);  // restart from the fresh residual (krylov.hpp:611-616)
    copy(c, r.p, rhat.p, n);
    fill(c, 0.0, p.p, n);
    fill(c, 0.0, v.p, n);
  }
}

}  // namespace

void validate_cfg(const SolverCfg& c) {  // SolverConfig::validate (krylov.hpp:50-54)
  if (!(c.rtol > 0.0)) throw std::invalid_argument("solver config: rtol must be > 0");
  if (c.max_iter < 1) throw std::invalid_argument("solver config: max_iter must be >= 1");
  if (c.restart < 1) throw std::invalid_argument("solver config: gmres_restart must be >= 1");
}

// run_solver (backend.hpp:241-286), iterative methods. x0 may alias x.
void solve(Operator& op, const SolverCfg& cfg, const double* b, const double* x0, double* x, SolveReport& rep) {
  validate_cfg(cfg);
  if (cfg.method < 0 || cfg.method > 4) throw std::invalid_argument("run_solver: unknown method");
  if (cfg.method >= 3) {  // DIRECT_CHOL / DIRECT_LU (backend.hpp:245-269)
    if (!op.csr_values()) throw CapabilityError("assembled matrix required, but the operator is matrix-free");
    op.validate();
    Timer timer;
    Ctx& c = *op.sys->ctx;
    const double bnorm = std::sqrt(dot(c, b, b, op.n));
    const double denom = bnorm > 0.0 ? bnorm : 1.0;
    rep.history.push_back(bnorm / denom);
    if (direct_solve(*op.sys, op.csr_values(), cfg.method == 3, b, x, rep.failure)) {
      rep.iterations = 1;
      DevArray<double> scratch(op.n);
      const double rres = residual_norm(op, b, x, scratch.p, nullptr) / denom;
      rep.history.push_back(rres);
      rep.converged = rres <= 1e-10;  // kDirectResidualContract (krylov.hpp:59)
    } else {
      fill(c, 0.0, x, op.n);
    }
    AFEM_CK(cudaStreamSynchronize(c.stream));
    rep.wall_time = timer.seconds();
    return;
  }
  if (cfg.precond < 0 || cfg.precond > 2) throw std::invalid_argument("run_solver: unknown preconditioner");
  if (cfg.precond == 2 && !op.csr_values())  // backend.hpp:151-156, 282
    throw CapabilityError("assembled matrix required, but the operator is matrix-free");
  op.validate();
  Timer timer;
  Ctx& c = *op.sys->ctx;
  DevArray<double> inv;
  if (cfg.precond == 1) jacobi_inverse(op, inv);
  Ilu0 ilu;
  if (cfg.precond == 2) ilu.setup(*op.sys, op.csr_values());  // ilu0_setup(op.csr()), krylov.hpp:192
  Pc pc;
  pc.inv = inv.p;
  pc.ilu = cfg.precond == 2 ? &ilu : nullptr;
  // the vector kernels use 16-byte accesses: iterate in an aligned buffer if the caller's is not
  DevArray<double> xa;
  double* xw = x;
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0) {
    xa.alloc(op.n);
    xw = xa.p;
  }
  if (x0) copy(c, x0, xw, op.n);
  else fill(c, 0.0, xw, op.n);
  if (cfg.method == 0 && pc.ilu) cg_generic(op, cfg, b, xw, pc, rep);
  else if (cfg.method == 0) cg(op, cfg, b, xw, inv.p, rep);
  else if (cfg.method == 1) gmres(op, cfg, b, xw, pc, rep);
  else bicgstab(op, cfg, b, xw, pc, rep);
  if (xw != x) copy(c, xw, x, op.n);
  AFEM_CK(cudaStreamSynchronize(c.stream));
  rep.wall_time = timer.seconds();
}

}  // namespace afem
