// Structured-grid fast path for the linear matrix-free operator y = K x (backend.hpp:130-147) on
// hex8 grid systems (afem_system_create_grid, dim 3) whose phases are all linear elastic with a
// common Poisson ratio. Then every element stiffness is K_e = E_phase * Khat (Khat: the uniform
// brick at E = 1), and
//     y_n = E_base(n) * (S x)_n  +  sum_{octants o of n with E_o != E_base} (E_o - E_base) Khat_rows(o) x_e(o)
// where S (27 blocks of 3x3) is the assembled homogeneous stencil and E_base(n) the majority
// modulus of the node's eight octant elements (octants outside the domain count as E = 0).
//
// Kernels:
//  k_stencil_main   32x8 node tile per CTA, marching in z over a chunk of planes; each x-plane
//                   (with a one-node halo, Dirichlet-masked) is staged once in shared memory
//                   (double-buffered, register prefetch) and each thread keeps the partial sums of
//                   the three nodes of its column the plane touches (z-1, z, z+1). 153 DFMA per
//                   node (the 243-entry stencil minus the 90 entries that vanish by symmetry), no
//                   atomics, every y entry written exactly once.
//  k_stencil_edge   the x columns a 32-wide tile cannot cover (NX mod 32), node per thread.
//  k_stencil_fix    interface nodes only (a precomputed list): adds the octant corrections.
// Algorithmic traffic: x (8 B/dof) + y (8 B/dof) + one info byte per node (Dirichlet bits +
// base phase) — no connectivity is read.
#include <cmath>
#include <vector>

#include "afem_impl.hpp"

namespace afem {

constexpr int kVoid = 31;  // phase code for octants outside the domain (E = 0)

struct StencilParams {
  double S[27][3][3];  // homogeneous stencil at E = 1: S[d][a][b], d = (dx+1) + 3(dy+1) + 9(dz+1)
  double K[24][24];    // uniform-brick element stiffness at E = 1
  double E[32];        // modulus per phase code (E[kVoid] = 0)
  int NX, NY, NZ;      // node counts per axis
  int NXm;             // columns covered by 32-wide tiles
};

struct StencilPlan {
  StencilParams p;
  DevArray<uint8_t> info;       // per node: bits 0-2 Dirichlet mask, bits 3-7 base phase code
  DevArray<int32_t> fix_nodes;  // interface nodes
  DevArray<uint8_t> fix_mask;   // per interface node: octants needing a correction
  int64_t n_fix = 0;
  int kchunk = 16;
};

namespace {

constexpr int TX = 32, TY = 8, NT = TX * TY;
constexpr int RW = 3 * (TX + 2);          // doubles per staged row (x-interleaved dofs)
constexpr int ITEMS = (TY + 2) * RW;      // doubles per staged plane
constexpr int PER = (ITEMS + NT - 1) / NT;

// Is S[d][a][b] structurally zero? Off-diagonal (a != b) entries vanish by reflection symmetry of
// the brick unless the offset is non-zero along both axes a and b.
__host__ __device__ constexpr bool szero(int dx, int dy, int dz, int a, int b) {
  if (a == b) return false;
  const int da = a == 0 ? dx : (a == 1 ? dy : dz);
  const int db = b == 0 ? dx : (b == 1 ? dy : dz);
  return da == 0 || db == 0;
}

template <int DX, int DY, int DZ>
__device__ __forceinline__ void sblock(const StencilParams& P, const double (&xv)[3], double (&acc)[3]) {
  constexpr int d = (DX + 1) + 3 * (DY + 1) + 9 * (DZ + 1);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      if (!szero(DX, DY, DZ, a, b)) acc[a] = fma(P.S[d][a][b], xv[b], acc[a]);
}

// Contributions of one staged plane (neighbour (DI, DJ) in-plane) to the three column nodes.
template <int DI, int DJ>
__device__ __forceinline__ void plane_neighbour(const StencilParams& P, const double (&xv)[3], bool dprev, bool dcur,
                                                bool dnext, double (&ap)[3], double (&ac)[3], double (&an)[3]) {
  if (dnext) sblock<DI, DJ, -1>(P, xv, an);  // node above sees this plane at dz = -1
  if (dcur) sblock<DI, DJ, 0>(P, xv, ac);
  if (dprev) sblock<DI, DJ, 1>(P, xv, ap);   // node below sees this plane at dz = +1
}

__global__ void __launch_bounds__(NT, 3) k_stencil_main(const __grid_constant__ StencilParams P,
                                                        const double* __restrict__ x,
                                                        const uint8_t* __restrict__ info, double* __restrict__ y,
                                                        int kchunk) {
  __shared__ double sm[2][3][TY + 2][TX + 2];
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int NX = P.NX, NY = P.NY, NZ = P.NZ;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int k0 = blockIdx.z * kchunk, k1 = min(k0 + kchunk, NZ);
  const int i = i0 + tx, j = j0 + ty;
  const bool active = j < NY;
  const int64_t plane = (int64_t)NX * NY;

  double pf[PER];
  auto fetch = [&](int p) {
#pragma unroll
    for (int it = 0; it < PER; ++it) {
      const int idx = threadIdx.x + it * NT;
      double v = 0.0;
      if (idx < ITEMS && p >= 0 && p < NZ) {
        const int r = idx / RW, c = idx - r * RW;
        const int ii = i0 - 1 + c / 3, jj = j0 - 1 + r, comp = c % 3;
        if (ii >= 0 && ii < NX && jj >= 0 && jj < NY) {
          const int64_t node = ii + (int64_t)NX * jj + plane * p;
          const uint8_t inf = __ldg(&info[node]);
          v = ((inf >> comp) & 1) ? 0.0 : __ldg(&x[3 * node + comp]);
        }
      }
      pf[it] = v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int it = 0; it < PER; ++it) {
      const int idx = threadIdx.x + it * NT;
      if (idx < ITEMS) {
        const int r = idx / RW, c = idx - r * RW;
        sm[buf][c % 3][r][c / 3] = pf[it];
      }
    }
  };

  double ap[3] = {0.0, 0.0, 0.0}, ac[3] = {0.0, 0.0, 0.0}, an[3] = {0.0, 0.0, 0.0};
  fetch(k0 - 1);
  store(0);
  __syncthreads();
  for (int p = k0 - 1; p <= k1; ++p) {
    const int buf = (p - (k0 - 1)) & 1;
    if (p < k1) fetch(p + 1);
    if (active && p >= 0 && p < NZ) {
      const bool dprev = p - 1 >= k0, dcur = p >= k0 && p < k1, dnext = p + 1 < k1;
#define AFEM_NB(DI, DJ)                                                                      \
  {                                                                                          \
    const double xv[3] = {sm[buf][0][ty + 1 + DJ][tx + 1 + DI], sm[buf][1][ty + 1 + DJ][tx + 1 + DI], \
                          sm[buf][2][ty + 1 + DJ][tx + 1 + DI]};                             \
    plane_neighbour<DI, DJ>(P, xv, dprev, dcur, dnext, ap, ac, an);                          \
  }
      AFEM_NB(-1, -1) AFEM_NB(0, -1) AFEM_NB(1, -1)
      AFEM_NB(-1, 0) AFEM_NB(0, 0) AFEM_NB(1, 0)
      AFEM_NB(-1, 1) AFEM_NB(0, 1) AFEM_NB(1, 1)
#undef AFEM_NB
    }
    if (active && p - 1 >= k0) {  // node (i, j, p-1) is complete
      const int64_t node = i + (int64_t)NX * j + plane * (p - 1);
      const uint8_t inf = __ldg(&info[node]);
      const double E = P.E[inf >> 3];
#pragma unroll
      for (int a = 0; a < 3; ++a) y[3 * node + a] = ((inf >> a) & 1) ? __ldg(&x[3 * node + a]) : E * ap[a];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      ap[a] = ac[a];
      ac[a] = an[a];
      an[a] = 0.0;
    }
    if (p < k1) store(buf ^ 1);
    __syncthreads();
  }
}

__device__ __forceinline__ double xm_at(const double* __restrict__ x, const uint8_t* __restrict__ info, int NX,
                                        int NY, int NZ, int ii, int jj, int kk, int comp) {
  if (ii < 0 || ii >= NX || jj < 0 || jj >= NY || kk < 0 || kk >= NZ) return 0.0;
  const int64_t node = ii + (int64_t)NX * (jj + (int64_t)NY * kk);
  return ((__ldg(&info[node]) >> comp) & 1) ? 0.0 : __ldg(&x[3 * node + comp]);
}

// Columns i >= NXm: full 27-point stencil per node with direct (cached) loads.
__global__ void k_stencil_edge(const __grid_constant__ StencilParams P, const double* __restrict__ x,
                               const uint8_t* __restrict__ info, double* __restrict__ y) {
  const int NX = P.NX, NY = P.NY, NZ = P.NZ, W = NX - P.NXm;
  const int64_t total = (int64_t)W * NY * NZ;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = P.NXm + static_cast<int>(t % W);
    const int64_t r = t / W;
    const int j = static_cast<int>(r % NY), k = static_cast<int>(r / NY);
    double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int d = 0; d < 27; ++d) {
      const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
      double xv[3];
#pragma unroll
      for (int b = 0; b < 3; ++b) xv[b] = xm_at(x, info, NX, NY, NZ, i + dx, j + dy, k + dz, b);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          if (!szero(dx, dy, dz, a, b)) acc[a] = fma(P.S[d][a][b], xv[b], acc[a]);
    }
    const int64_t node = i + (int64_t)NX * (j + (int64_t)NY * k);
    const uint8_t inf = info[node];
    const double E = P.E[inf >> 3];
#pragma unroll
    for (int a = 0; a < 3; ++a) y[3 * node + a] = ((inf >> a) & 1) ? x[3 * node + a] : E * acc[a];
  }
}

// hex8 local node index of corner (lx, ly, lz) (element.hpp:22-23 ring, then z = +1).
__host__ __device__ __forceinline__ int local_node(int lx, int ly, int lz) {
  const int ring = lx ? (ly ? 2 : 1) : (ly ? 3 : 0);
  return ring + 4 * lz;
}

// Interface corrections: y_n += sum_o (E_o - E_base) Khat_rows(ln(o)) x_e(o), free rows only.
__global__ void k_stencil_fix(const __grid_constant__ StencilParams P, const double* __restrict__ x,
                              const uint8_t* __restrict__ info, const uint8_t* __restrict__ phase,
                              const int32_t* __restrict__ nodes, const uint8_t* __restrict__ omask, int64_t n_fix,
                              double* __restrict__ y) {
  const int NX = P.NX, NY = P.NY, NZ = P.NZ;
  const int ex = NX - 1, ey = NY - 1, ez = NZ - 1;  // element counts
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_fix; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = nodes[t];
    const int i = static_cast<int>(node % NX);
    const int64_t r = node / NX;
    const int j = static_cast<int>(r % NY), k = static_cast<int>(r / NY);
    const uint8_t inf = info[node];
    const double Eb = P.E[inf >> 3];
    const uint8_t om = omask[t];
    double acc[3] = {0.0, 0.0, 0.0};
    for (int o = 0; o < 8; ++o) {
      if (!((om >> o) & 1)) continue;
      const int ox = o & 1, oy = (o >> 1) & 1, oz = o >> 2;
      const int ei = i - 1 + ox, ej = j - 1 + oy, ek = k - 1 + oz;
      const bool inside = ei >= 0 && ei < ex && ej >= 0 && ej < ey && ek >= 0 && ek < ez;
      const int ph = inside ? phase[ei + (int64_t)ex * (ej + (int64_t)ey * ek)] : kVoid;
      const double dE = P.E[ph] - Eb;
      const int ln = local_node(1 - ox, 1 - oy, 1 - oz);
      double t3[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int mx = ((m & 3) == 1 || (m & 3) == 2) ? 1 : 0, my = (m & 3) >= 2 ? 1 : 0, mz = m >> 2;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const double xv = xm_at(x, info, NX, NY, NZ, ei + mx, ej + my, ek + mz, b);
#pragma unroll
          for (int a = 0; a < 3; ++a) t3[a] = fma(P.K[3 * ln + a][3 * m + b], xv, t3[a]);
        }
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) acc[a] = fma(dE, t3[a], acc[a]);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (!((inf >> a) & 1)) y[3 * node + a] += acc[a];
  }
}

// Node info byte + interface list. Base phase = most frequent octant phase (void counted), ties to
// the smaller code.
__global__ void k_stencil_classify(int NX, int NY, int NZ, const uint8_t* __restrict__ phase,
                                   const uint8_t* __restrict__ dof_mask, uint8_t* __restrict__ info,
                                   int32_t* __restrict__ fix_nodes, uint8_t* __restrict__ fix_mask,
                                   unsigned long long* __restrict__ n_fix) {
  const int ex = NX - 1, ey = NY - 1, ez = NZ - 1;
  const int64_t total = (int64_t)NX * NY * NZ;
  for (int64_t node = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; node < total;
       node += (int64_t)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(node % NX);
    const int64_t r = node / NX;
    const int j = static_cast<int>(r % NY), k = static_cast<int>(r / NY);
    int ph[8];
    for (int o = 0; o < 8; ++o) {
      const int ei = i - 1 + (o & 1), ej = j - 1 + ((o >> 1) & 1), ek = k - 1 + (o >> 2);
      const bool inside = ei >= 0 && ei < ex && ej >= 0 && ej < ey && ek >= 0 && ek < ez;
      ph[o] = inside ? phase[ei + (int64_t)ex * (ej + (int64_t)ey * ek)] : kVoid;
    }
    int best = ph[0], bestc = 0;
    for (int o = 0; o < 8; ++o) {
      int c = 0;
      for (int q = 0; q < 8; ++q) c += ph[q] == ph[o];
      if (c > bestc || (c == bestc && ph[o] < best)) {
        best = ph[o];
        bestc = c;
      }
    }
    uint8_t om = 0;
    for (int o = 0; o < 8; ++o)
      if (ph[o] != best) om |= static_cast<uint8_t>(1u << o);
    const uint8_t m = (dof_mask[3 * node] ? 1 : 0) | (dof_mask[3 * node + 1] ? 2 : 0) | (dof_mask[3 * node + 2] ? 4 : 0);
    info[node] = static_cast<uint8_t>(m | (best << 3));
    if (om && m != 7) {
      const unsigned long long slot = atomicAdd(n_fix, 1ull);
      fix_nodes[slot] = static_cast<int32_t>(node);
      fix_mask[slot] = om;
    }
  }
}

// Uniform-brick element stiffness at E = 1 (same device math as the general tangent kernel).
__global__ void k_brick_stiffness(const double* coords, const int32_t* conn, DMat m, double* K) {
  const int a_node = threadIdx.x;  // 8 threads: one per row node
  if (a_node >= 8) return;
  double xc[8][3];
  for (int k = 0; k < 8; ++k)
    for (int c = 0; c < 3; ++c) xc[k][c] = coords[3 * conn[k] + c];
  double rows[3][24];
  for (int a = 0; a < 3; ++a)
    for (int j = 0; j < 24; ++j) rows[a][j] = 0.0;
  for (int q = 0; q < 8; ++q) {
    double g[8][3], wdet;
    qp_geometry<3>(xc, q, g, wdet);
    double H[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    TangentQP<3> t;
    int err = 0;
    tangent_qp<3>(m, H, t, err);
    double gn[3] = {g[a_node][0], g[a_node][1], g[a_node][2]};
    for (int lm = 0; lm < 8; ++lm) {
      double gm[3] = {g[lm][0], g[lm][1], g[lm][2]}, blk[3][3];
      tangent_block<3>(t, gn, gm, blk);
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) rows[a][3 * lm + b] += wdet * blk[a][b];
    }
  }
  for (int a = 0; a < 3; ++a)
    for (int j = 0; j < 24; ++j) K[(3 * a_node + a) * 24 + j] = rows[a][j];
}

}  // namespace

StencilPlan* make_stencil_plan(System& s, const MfOp& op) {
  if (!s.grid || s.dim != 3) return nullptr;
  if (s.mats.empty() || s.mats.size() >= kVoid) return nullptr;
  const double nu = s.mats[0].nu;
  for (const DMat& m : s.mats)
    if (m.model != MODEL_LINEAR || m.nu != nu) return nullptr;
  if (s.n_nodes > (int64_t)INT32_MAX) return nullptr;
  Ctx& c = *s.ctx;
  auto plan = std::make_unique<StencilPlan>();
  StencilParams& P = plan->p;
  P.NX = s.nx + 1;
  P.NY = s.ny + 1;
  P.NZ = s.nz + 1;
  P.NXm = (P.NX / TX) * TX;
  for (int k = 0; k < 32; ++k) P.E[k] = 0.0;
  for (size_t k = 0; k < s.mats.size(); ++k) P.E[k] = s.mats[k].E;

  // Khat from element 0 at E = 1 (K_e = E * Khat for a common nu: c11, c12, c33 scale with E).
  DevArray<double> dK(576);
  DMat unit = make_dmat(MODEL_LINEAR, 1.0, nu);
  launch(c, k_brick_stiffness, 1, 32, 0, s.coords.p, s.conn.p, unit, dK.p);
  std::vector<double> K(576);
  AFEM_CK(cudaMemcpyAsync(K.data(), dK.p, 576 * 8, cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  for (int r = 0; r < 24; ++r)
    for (int q = 0; q < 24; ++q) P.K[r][q] = K[r * 24 + q];
  // S(d) = sum over octants o containing n and n + d of Khat[ln(o), lm(o, d)]
  double smax = 0.0;
  for (int d = 0; d < 27; ++d)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) P.S[d][a][b] = 0.0;
  for (int o = 0; o < 8; ++o) {
    const int ox = o & 1, oy = (o >> 1) & 1, oz = o >> 2;
    const int lx = 1 - ox, ly = 1 - oy, lz = 1 - oz;
    const int ln = local_node(lx, ly, lz);
    for (int mz = 0; mz < 2; ++mz)
      for (int my = 0; my < 2; ++my)
        for (int mx = 0; mx < 2; ++mx) {
          const int lm = local_node(mx, my, mz);
          const int d = (mx - lx + 1) + 3 * (my - ly + 1) + 9 * (mz - lz + 1);
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) P.S[d][a][b] += K[(3 * ln + a) * 24 + 3 * lm + b];
        }
  }
  for (int d = 0; d < 27; ++d)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) smax = std::max(smax, std::abs(P.S[d][a][b]));
  for (int d = 0; d < 27; ++d)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        if (szero(d % 3 - 1, (d / 3) % 3 - 1, d / 9 - 1, a, b)) {
          if (std::abs(P.S[d][a][b]) > 1e-12 * smax) return nullptr;  // not a symmetric brick grid
          P.S[d][a][b] = 0.0;
        }

  const int64_t nn = s.n_nodes;
  plan->info.alloc(nn);
  plan->fix_nodes.alloc(nn);
  plan->fix_mask.alloc(nn);
  DevArray<unsigned long long> cnt(1);
  AFEM_CK(cudaMemsetAsync(cnt.p, 0, 8, c.stream));
  launch(c, k_stencil_classify, grid_for(nn, 256, 148 * 32), 256, 0, P.NX, P.NY, P.NZ, s.phase.p, op.mask.p,
         plan->info.p, plan->fix_nodes.p, plan->fix_mask.p, cnt.p);
  unsigned long long nf = 0;
  AFEM_CK(cudaMemcpyAsync(&nf, cnt.p, 8, cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  plan->n_fix = static_cast<int64_t>(nf);
  // z chunk: enough CTAs for ~3 per SM, at least 8 planes per chunk
  const int64_t tiles = (int64_t)(P.NXm / TX) * ((P.NY + TY - 1) / TY);
  int chunks = tiles > 0 ? static_cast<int>((3 * c.num_sms + tiles - 1) / tiles) : 1;
  chunks = std::max(1, std::min(chunks, (P.NZ + 7) / 8));
  plan->kchunk = (P.NZ + chunks - 1) / chunks;
  return plan.release();
}

void stencil_apply(StencilPlan& pl, const MfOp& op, const double* x, double* y) {
  Ctx& c = *op.sys->ctx;
  const StencilParams& P = pl.p;
  if (P.NXm > 0) {
    dim3 grid(P.NXm / TX, (P.NY + TY - 1) / TY, (P.NZ + pl.kchunk - 1) / pl.kchunk);
    launch(c, k_stencil_main, grid, NT, 0, P, x, pl.info.p, y, pl.kchunk);
  }
  const int64_t edge = (int64_t)(P.NX - P.NXm) * P.NY * P.NZ;
  if (edge > 0) launch(c, k_stencil_edge, grid_for(edge, 128, 148 * 16), 128, 0, P, x, pl.info.p, y);
  if (pl.n_fix > 0)
    launch(c, k_stencil_fix, grid_for(pl.n_fix, 128, 148 * 32), 128, 0, P, x, pl.info.p, op.sys->phase.p,
           pl.fix_nodes.p, pl.fix_mask.p, pl.n_fix, y);
}

void destroy_stencil_plan(StencilPlan* p) { delete p; }

}  // namespace afem
