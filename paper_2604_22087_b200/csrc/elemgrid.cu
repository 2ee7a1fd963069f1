// Element-centric kernels for structured grid systems (afem_system_create_grid): residual,
// matrix-free JVP and Jacobi diagonal of ANY constitutive law (linear, SVK, Neo-Hookean, J2).
//
// The general node-centric kernels (assembly.cu) re-evaluate an element's quadrature loop once per
// incident node (8x in 3D). On a uniform grid every element is the same brick, so the shape-function
// gradients g_i(q) and w detJ(q) are computed once per system (GridGeo, passed as a __grid_constant__
// parameter: uniform broadcast reads, no per-element geometry) and the element kernel evaluates the
// constitutive update once per Gauss point, writing the element's nd-vector to a scratch array:
//     k_grid_elem<MODE>  thread per element: gather u_e (and x_e), qp loop, ev[corner][e] = f_e
//                        (corner-major scratch: a warp's stores of one corner, and the gather's
//                        loads of one incidence slot over consecutive nodes, are contiguous)
//     k_gather           thread per node: y_n = sum over the node's incident (element, corner) pairs
//                        in the reference's (batch, element) order (assembly.hpp:130-137)
// The reduction order is the node-centric kernels' (and the reference's), so results stay
// deterministic run to run with no atomics. Algorithmic traffic per element: u_e/x_e gathers
// (L2-resident neighbours), J2 history (nq*64 B), 2*nd*8 B of scratch.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cuda_pipeline.h>

#include "afem_impl.hpp"
#include "reduce.cuh"

namespace afem {

namespace {

template <int D>
struct GeoT {
  double g[EL<D>::nq][EL<D>::npe][D];
  double wdet[EL<D>::nq];
};

// Uniform-brick geometry from element 0 (the same device math as the general kernels).
template <int D>
__global__ void k_grid_geometry(const double* coords, const int32_t* conn, double* out, int* err) {
  constexpr int npe = EL<D>::npe, nq = EL<D>::nq;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double xc[npe][D];
  for (int k = 0; k < npe; ++k)
    for (int c = 0; c < D; ++c) xc[k][c] = coords[(int64_t)conn[k] * D + c];
  for (int q = 0; q < nq; ++q) {
    double g[npe][D], wdet;
    if (!qp_geometry<D>(xc, q, g, wdet)) atomicOr(err, ERR_DETJ);
    for (int i = 0; i < npe; ++i)
      for (int b = 0; b < D; ++b) out[(q * npe + i) * D + b] = g[i][b];
    out[nq * npe * D + q] = wdet;
  }
}

enum : int { EV_RESIDUAL = 0, EV_JVP = 1, EV_DIAG = 2 };

__device__ __forceinline__ int grid_find_pos(const int32_t* adj, int deg, int64_t m) {
  int lo = 0, hi = deg;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (adj[mid] < m) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <int D>
__device__ __forceinline__ void elem_nodes(int64_t e, int nx, int ny, int64_t (&nd)[EL<D>::npe]);

// J2 history commit on grids: thread per (element, Gauss point) — consecutive threads own
// consecutive 64-byte history slots (coalesced read-modify-write), uniform-brick gradients.
template <int D>
__global__ void __launch_bounds__(128) k_grid_history_commit(const __grid_constant__ GeoT<D> G, SysView s, int nx,
                                                             int ny, const double* __restrict__ u, double* hist) {
  constexpr int npe = EL<D>::npe, nq = EL<D>::nq;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < s.n_elem * nq; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / nq;
    const int q = static_cast<int>(t % nq);
    const DMat m = s.mats[s.phase[e]];
    if (m.model != MODEL_J2) continue;
    int64_t nodes[npe];
    elem_nodes<D>(e, nx, ny, nodes);
    double H[D][D];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) H[a][b] = 0.0;
#pragma unroll
    for (int k = 0; k < npe; ++k)
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double ua = __ldg(&u[nodes[k] * D + a]);
#pragma unroll
        for (int b = 0; b < D; ++b) H[a][b] += ua * G.g[q][k][b];
      }
    double* hq = hist + t * kHist;
    j2_commit<D>(m, H, hq, hq);
  }
}

// Element-centric tangent (3D grids), two passes per z slab of node planes:
//   k_grid_kelem    warp per element: lanes 0-7 evaluate the 8 Gauss-point tangents once (shared
//                   memory), lane (corner ln, corner pair g) accumulates the blocks (ln, 2g), (ln, 2g+1)
//                   over the Gauss points in order -> scratch [e][ln][a][24]
//   k_grid_kgather  warp per node: the node's 9 deg row entries accumulated in shared memory over its
//                   incident elements in (batch, element) order, then written once, coalesced
// Per entry the sums run in the node-centric kernel's order (Gauss points within an element, then
// elements in incidence order), so the values are the same; each Gauss point's constitutive
// tangent is evaluated once instead of once per incident node, and every CSR value is written once.
constexpr int kKelemWarps = 4;
constexpr int kKe = 8 * 3 * 24;  // doubles of one element's scratch block

__global__ void __launch_bounds__(32 * kKelemWarps) k_grid_kelem(const __grid_constant__ GeoT<3> G, SysView s, int nx,
                                                                 int ny, const double* __restrict__ u, int64_t e0,
                                                                 int64_t e1, double* __restrict__ scr) {
  __shared__ TangentQP<3> ts[kKelemWarps][2][8];
  __shared__ double us[kKelemWarps][2][24];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int err = 0;
  // two elements per warp trip: lanes 0-15 evaluate both elements' 16 Gauss-point tangents at once
  for (int64_t ep = e0 + 2 * (blockIdx.x * (int64_t)kKelemWarps + w); ep < e1;
       ep += 2 * (int64_t)gridDim.x * kKelemWarps) {
    const int ne = ep + 1 < e1 ? 2 : 1;
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (h < ne && lane < 24) {
        int64_t nodes[8];
        elem_nodes<3>(ep + h, nx, ny, nodes);
        us[w][h][lane] = __ldg(&u[nodes[lane / 3] * 3 + lane % 3]);
      }
    __syncwarp();
    if (lane < 8 * ne) {
      const int h = lane >> 3, q = lane & 7;
      const int64_t e = ep + h;
      const DMat m = s.mats[s.phase[e]];
      double H[3][3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          double hh = 0.0;
#pragma unroll
          for (int k = 0; k < 8; ++k) hh += us[w][h][k * 3 + a] * G.g[q][k][b];
          H[a][b] = hh;
        }
      TangentQP<3> t;
      tangent_qp<3>(m, H, t, err, s.hist ? s.hist + (e * 8 + q) * kHist : nullptr);
      ts[w][h][q] = t;
    }
    __syncwarp();
    for (int he = 0; he < ne; ++he) {  // lane = (corner ln, corner pair g): blocks (ln, 2g), (ln, 2g + 1)
      const int64_t e = ep + he;
      const int ln = lane >> 2, g = lane & 3;
      double K[2][3][3];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) K[h][a][b] = 0.0;
      for (int q = 0; q < 8; ++q) {
        const TangentQP<3>& t = ts[w][he][q];
        double gn[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) gn[c] = G.g[q][ln][c];
        const double wdet = G.wdet[q];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int lm = 2 * g + h;
          double gm[3], blk[3][3];
#pragma unroll
          for (int c = 0; c < 3; ++c) gm[c] = G.g[q][lm][c];
          tangent_block<3>(t, gn, gm, blk);
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) K[h][a][b] += wdet * blk[a][b];
        }
      }
      double* o = scr + (e - e0) * kKe + ln * 72 + 6 * g;  // [ln][a][lm * 3 + b]
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int b = 0; b < 3; ++b) o[a * 24 + h * 3 + b] = K[h][a][b];
    }
    __syncwarp();
  }
  if (err) atomicOr(s.err, err);
}

constexpr int kGatherWarps = 4;

// hex8 corner m's position bits (element.hpp:22-23 ring, then z)
__device__ __forceinline__ int corner_bit_x(int m) { return ((m & 3) == 1 || (m & 3) == 2) ? 1 : 0; }
__device__ __forceinline__ int corner_bit_y(int m) { return (m & 3) >= 2 ? 1 : 0; }

__global__ void __launch_bounds__(32 * kGatherWarps) k_grid_kgather(SysView s, int nx, int ny, int nz, int64_t n0, int64_t n1,
                                                                    int64_t e0, const double* __restrict__ scr,
                                                                    double* __restrict__ values) {
  __shared__ double row[kGatherWarps][243];
  __shared__ int pos[kGatherWarps][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t n = n0 + blockIdx.x * (int64_t)kGatherWarps + w; n < n1; n += (int64_t)gridDim.x * kGatherWarps) {
    const int64_t a0 = s.adj_ptr[n];
    // the grid node's neighbours sorted by id = (dz, dy, dx) lexicographic over the offsets that
    // stay inside the grid: slot of offset (dx, dy, dz) in closed form
    const int NXn = nx + 1, NYn = ny + 1;
    const int i = static_cast<int>(n % NXn);
    const int64_t rr = n / NXn;
    const int j = static_cast<int>(rr % NYn), kz = static_cast<int>(rr / NYn);
    const int xlo = i > 0, ylo = j > 0, zlo = kz > 0;
    const int cx = 1 + xlo + (i < nx), cy = 1 + ylo + (j < ny), cz = 1 + zlo + (kz < nz);
    const int deg = cx * cy * cz;
    const int len = 9 * deg;
    for (int jj = lane; jj < len; jj += 32) row[w][jj] = 0.0;
    // all (<= 8) incident elements' 72-value rows are loaded up front (24 independent loads per
    // lane), then added element by element in incidence order
    const int64_t p0 = s.inc_ptr[n];
    const int cnt = static_cast<int>(s.inc_ptr[n + 1] - p0);
    double vals[8][3];
#pragma unroll
    for (int pe = 0; pe < 8; ++pe) {
      if (pe < cnt) {
        const uint32_t v = s.inc[p0 + pe];
        const double* src = scr + (static_cast<int64_t>(v / 8) - e0) * kKe + (v % 8) * 72;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const int k = lane + 32 * r;
          vals[pe][r] = k < 72 ? __ldg(&src[k]) : 0.0;
        }
      }
    }
    for (int h = lane; h < 8 * cnt; h += 32) {  // slot of corner (h % 8) of incident element h / 8
      const int ln = static_cast<int>(s.inc[p0 + h / 8] % 8), cm = h % 8;
      const int dx = corner_bit_x(cm) - corner_bit_x(ln), dy = corner_bit_y(cm) - corner_bit_y(ln);
      const int dz = (cm >> 2) - (ln >> 2);
      pos[w][h] = ((dz + zlo) * cy + (dy + ylo)) * cx + (dx + xlo);
    }
    __syncwarp();
#pragma unroll
    for (int pe = 0; pe < 8; ++pe) {
      if (pe < cnt) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {  // k = a * 24 + lm * 3 + b: distinct targets within an element
          const int k = lane + 32 * r;
          if (k < 72) {
            const int a = k / 24, q = k % 24;
            row[w][a * 3 * deg + pos[w][pe * 8 + q / 3] * 3 + q % 3] += vals[pe][r];
          }
        }
      }
      __syncwarp();
    }
    double* out = values + 9 * a0;
    for (int jj = lane; jj < len; jj += 32) out[jj] = row[w][jj];
    __syncwarp();
  }
}

// K(u) rows of node n into pattern-ordered CSR values: assembly.cu's k_jacobian (assembly.hpp:144-173)
// with the uniform-brick gradients instead of a per-(node, element, qp) Jacobian inverse and
// implicit connectivity. Same per-entry summation order (elements in (batch, element) order, Gauss
// points in order), so the result is deterministic.
template <int D>
__global__ void __launch_bounds__(128) k_grid_jacobian(const __grid_constant__ GeoT<D> G, SysView s, int nx, int ny,
                                                       const double* __restrict__ u, double* __restrict__ values) {
  constexpr int npe = EL<D>::npe, nq = EL<D>::nq, nd = EL<D>::nd;
  int err = 0;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < s.n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a0 = s.adj_ptr[n];
    const int deg = static_cast<int>(s.adj_ptr[n + 1] - a0);
    const int64_t base = (int64_t)D * D * a0;
    for (int j = 0; j < D * D * deg; ++j) values[base + j] = 0.0;
    for (int64_t p = s.inc_ptr[n]; p < s.inc_ptr[n + 1]; ++p) {
      const uint32_t v = s.inc[p];
      const int64_t e = v / npe;
      const int ln = v % npe;
      int64_t nodes[npe];
      elem_nodes<D>(e, nx, ny, nodes);
      double ue[nd];
#pragma unroll
      for (int k = 0; k < npe; ++k)
#pragma unroll
        for (int c = 0; c < D; ++c) ue[k * D + c] = __ldg(&u[nodes[k] * D + c]);
      const DMat m = s.mats[s.phase[e]];
      int pos[npe];
#pragma unroll
      for (int k = 0; k < npe; ++k) pos[k] = grid_find_pos(s.adj + a0, deg, nodes[k]);
      double K[D][nd];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int j = 0; j < nd; ++j) K[a][j] = 0.0;
      for (int q = 0; q < nq; ++q) {
        double H[D][D];
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b < D; ++b) {
            double h = 0.0;
#pragma unroll
            for (int k = 0; k < npe; ++k) h += ue[k * D + a] * G.g[q][k][b];
            H[a][b] = h;
          }
        TangentQP<D> t;
        tangent_qp<D>(m, H, t, err, s.hist ? s.hist + (e * nq + q) * kHist : nullptr);
        double gn[D];
#pragma unroll
        for (int c = 0; c < D; ++c) gn[c] = G.g[q][ln][c];
        const double wdet = G.wdet[q];
#pragma unroll
        for (int lm = 0; lm < npe; ++lm) {
          double gm[D], blk[D][D];
#pragma unroll
          for (int c = 0; c < D; ++c) gm[c] = G.g[q][lm][c];
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
  }
  if (err) atomicOr(s.err, err);
}


template <int D>
__device__ __forceinline__ void elem_nodes(int64_t e, int nx, int ny, int64_t (&nd)[EL<D>::npe]) {
  const int ex = static_cast<int>(e % nx);
  const int64_t r = e / nx;
  const int ey = static_cast<int>(r % ny);
  const int64_t ez = r / ny;
  const int64_t NX = nx + 1, NXY = NX * (ny + 1);
  const int64_t n0 = ex + NX * ey + NXY * ez;
  nd[0] = n0; nd[1] = n0 + 1; nd[2] = n0 + 1 + NX; nd[3] = n0 + NX;
  if constexpr (D == 3) {
    nd[4] = n0 + NXY; nd[5] = n0 + 1 + NXY; nd[6] = n0 + 1 + NX + NXY; nd[7] = n0 + NX + NXY;
  }
}

// Element vector f_e into the corner-major scratch ev[corner][element][D]
template <int D>
__device__ __forceinline__ void ev_store(double* ev, int64_t n_elem, int64_t e, const double (&f)[EL<D>::nd]) {
#pragma unroll
  for (int k = 0; k < EL<D>::npe; ++k)
#pragma unroll
    for (int a = 0; a < D; ++a) ev[((int64_t)k * n_elem + e) * D + a] = f[k * D + a];
}

template <int D, int MODE>
__global__ void __launch_bounds__(128) k_grid_elem(const __grid_constant__ GeoT<D> G, SysView s, int nx, int ny,
                                                   const double* __restrict__ u, const uint8_t* __restrict__ mask,
                                                   const double* __restrict__ x, double* __restrict__ ev) {
  constexpr int npe = EL<D>::npe, nq = EL<D>::nq, nd = EL<D>::nd;
  int err = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s.n_elem; e += (int64_t)gridDim.x * blockDim.x) {
    const DMat m = s.mats[s.phase[e]];
    const bool lin = m.model == MODEL_LINEAR;
    int64_t nodes[npe];
    elem_nodes<D>(e, nx, ny, nodes);
    double ue[nd], xe[nd];
#pragma unroll
    for (int k = 0; k < npe; ++k)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const int64_t d = nodes[k] * D + c;
        ue[k * D + c] = (MODE == EV_JVP && lin) ? 0.0 : __ldg(&u[d]);
        if constexpr (MODE == EV_JVP) xe[k * D + c] = mask[d] ? 0.0 : __ldg(&x[d]);
      }
    double f[nd];
#pragma unroll
    for (int k = 0; k < nd; ++k) f[k] = 0.0;
    const double* hbase = s.hist ? s.hist + e * nq * kHist : nullptr;
#pragma unroll 1
    for (int q = 0; q < nq; ++q) {
      const double wdet = G.wdet[q];
      const double* hq = hbase ? hbase + q * kHist : nullptr;
      double H[D][D];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) {
          double t = 0.0;
#pragma unroll
          for (int i = 0; i < npe; ++i) t += ue[D * i + a] * G.g[q][i][b];
          H[a][b] = t;
        }
      if constexpr (MODE == EV_DIAG) {
        TangentQP<D> t;
        tangent_qp<D>(m, H, t, err, hq);
#pragma unroll
        for (int i = 0; i < npe; ++i) {
          double gi[D], blk[D][D];
#pragma unroll
          for (int c = 0; c < D; ++c) gi[c] = G.g[q][i][c];
          tangent_block<D>(t, gi, gi, blk);
#pragma unroll
          for (int a = 0; a < D; ++a) f[D * i + a] += wdet * blk[a][a];
        }
      } else {
        double P[D][D];
        if constexpr (MODE == EV_RESIDUAL) {
          piola<D>(m, H, P, err, hq);
        } else {
          double dH[D][D];
#pragma unroll
          for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = 0; b < D; ++b) {
              double t = 0.0;
#pragma unroll
              for (int i = 0; i < npe; ++i) t += xe[D * i + a] * G.g[q][i][b];
              dH[a][b] = t;
            }
          piola_jvp<D>(m, H, dH, P, hq);
        }
#pragma unroll
        for (int i = 0; i < npe; ++i)
#pragma unroll
          for (int a = 0; a < D; ++a) {
            double t = 0.0;
#pragma unroll
            for (int b = 0; b < D; ++b) t += P[a][b] * G.g[q][i][b];
            f[D * i + a] += wdet * t;
          }
      }
    }
    ev_store<D>(ev, s.n_elem, e, f);
  }
  if (err) atomicOr(s.err, err);
}

// y_n = sum of the node's element contributions in (batch, element) order; JVP: unit rows on
// constrained dofs (backend.hpp:146-147).
template <int D>
// dot_out (JVP only): also x.y over every row, into dot_out[0] (fixed-order grid reduction over
// <= kRedBlocks * 4 blocks): the CG's p.Ap fused into the apply, so the loop does not re-read p, Ap.
__global__ void __launch_bounds__(256) k_gather(SysView s, const double* __restrict__ ev, const uint8_t* __restrict__ mask,
                                                const double* __restrict__ x, double* __restrict__ y,
                                                const int* skip, double* partials, unsigned* counter,
                                                double* dot_out) {
  if (skip && *skip) return;
  double dsum = 0.0;
  constexpr int npe = EL<D>::npe, nd = EL<D>::nd;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < s.n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    double acc[D];
#pragma unroll
    for (int a = 0; a < D; ++a) acc[a] = 0.0;
    for (int64_t p = s.inc_ptr[n]; p < s.inc_ptr[n + 1]; ++p) {
      const uint32_t v = __ldg(&s.inc[p]);
      const double* src = ev + ((int64_t)(v % npe) * s.n_elem + v / npe) * D;
#pragma unroll
      for (int a = 0; a < D; ++a) acc[a] += __ldg(&src[a]);
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int64_t d = D * n + a;
      const double yv = (mask && mask[d]) ? x[d] : acc[a];
      y[d] = yv;
      if (dot_out) dsum += x[d] * yv;
    }
  }
  if (!dot_out) return;
  double v[1] = {dsum};
  if (grid_reduce<1>(v, partials, counter) && threadIdx.x == 0) dot_out[0] = v[0];
}


// ---- cached consistent tangents (J2 + linear grids): the matrix-free operator's state is fixed, so
// the return map of every J2 Gauss point is evaluated once at operator creation and its consistent
// tangent stored as (lam_eff, mu_eff, g2, n[6]) (kQpt doubles per Gauss point, structure of arrays
// [q][k][element] so a warp's loads are coalesced); each apply then costs
// one gather, dH, the cached isotropic-plus-rank-one tangent and the projection per Gauss point.
constexpr int kQpt = 9;

template <int D>
__global__ void __launch_bounds__(128) k_grid_qp_tangent(const __grid_constant__ GeoT<D> G, SysView s, int nx, int ny,
                                                         const double* __restrict__ u, double* __restrict__ qpt) {
  constexpr int npe = EL<D>::npe, nq = EL<D>::nq, nd = EL<D>::nd;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s.n_elem; e += (int64_t)gridDim.x * blockDim.x) {
    const DMat m = s.mats[s.phase[e]];
    if (m.model != MODEL_J2) continue;
    int64_t nodes[npe];
    elem_nodes<D>(e, nx, ny, nodes);
    double ue[nd];
#pragma unroll
    for (int k = 0; k < npe; ++k)
#pragma unroll
      for (int c = 0; c < D; ++c) ue[k * D + c] = __ldg(&u[nodes[k] * D + c]);
    for (int q = 0; q < nq; ++q) {
      double H[D][D];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) {
          double t = 0.0;
#pragma unroll
          for (int i = 0; i < npe; ++i) t += ue[D * i + a] * G.g[q][i][b];
          H[a][b] = t;
        }
      J2QP j;
      j2_state<D>(m, H, s.hist + (e * nq + q) * kHist, j);
      const int64_t ne = s.n_elem;
      double* o = qpt + (int64_t)q * kQpt * ne + e;
      const double mu_eff = m.mu * j.beta;
      o[0 * ne] = m.kappa - 2.0 * mu_eff / 3.0;
      o[1 * ne] = mu_eff;
      o[2 * ne] = 2.0 * m.mu * j.gbar;
      o[3 * ne] = j.n[0][0]; o[4 * ne] = j.n[1][1]; o[5 * ne] = j.n[2][2];
      o[6 * ne] = j.n[1][2]; o[7 * ne] = j.n[0][2]; o[8 * ne] = j.n[0][1];
    }
  }
}

// The element's nq * kQpt cached values are copied into a thread-private shared-memory column with
// cp.async at the start of the element (all in flight together, beside the x gathers), then read per
// Gauss point: one HBM round trip per element instead of one per Gauss point (ncu at 128^3: 59 %
// long-scoreboard stalls on the per-Gauss-point loads at 8 warps per SM, 2.5 TB/s).
constexpr int kJvpThreads = 128;
template <int D>
constexpr size_t jvp_cached_smem() { return (size_t)EL<D>::nq * kQpt * kJvpThreads * sizeof(double); }

template <int D>
__global__ void __launch_bounds__(kJvpThreads) k_grid_jvp_cached(const __grid_constant__ GeoT<D> G, SysView s, int nx,
                                                                int ny, const double* __restrict__ qpt,
                                                                const uint8_t* __restrict__ mask,
                                                                const double* __restrict__ x, double* __restrict__ ev,
                                                                const int* skip) {
  if (skip && *skip) return;
  constexpr int npe = EL<D>::npe, nq = EL<D>::nq, nd = EL<D>::nd;
  extern __shared__ double qsh[];  // [q * kQpt + k][thread]
  double* col = qsh + threadIdx.x;
  const int64_t ne = s.n_elem;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s.n_elem; e += (int64_t)gridDim.x * blockDim.x) {
    const DMat m = s.mats[s.phase[e]];
    const bool j2 = m.model == MODEL_J2;
    if (j2) {
#pragma unroll
      for (int k = 0; k < nq * kQpt; ++k) __pipeline_memcpy_async(col + k * kJvpThreads, qpt + (int64_t)k * ne + e, 8);
      __pipeline_commit();
    }
    int64_t nodes[npe];
    elem_nodes<D>(e, nx, ny, nodes);
    double xe[nd];
#pragma unroll
    for (int k = 0; k < npe; ++k)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const int64_t d = nodes[k] * D + c;
        xe[k * D + c] = mask[d] ? 0.0 : __ldg(&x[d]);
      }
    double f[nd];
#pragma unroll
    for (int k = 0; k < nd; ++k) f[k] = 0.0;
#pragma unroll 1
    for (int q = 0; q < nq; ++q) {
      double dH[D][D];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) {
          double t = 0.0;
#pragma unroll
          for (int i = 0; i < npe; ++i) t += xe[D * i + a] * G.g[q][i][b];
          dH[a][b] = t;
        }
      double P[D][D];
      if (j2) {  // lam tr(de) I + 2 mu de - g2 (n : de) n with the cached tangent
        if (q == 0) __pipeline_wait_prior(0);
        const double* t = col + q * kQpt * kJvpThreads;
        constexpr int T = kJvpThreads;
        const double lam = t[0], mu = t[T], g2 = t[2 * T];
        const double n00 = t[3 * T], n11 = t[4 * T], n22 = t[5 * T];
        const double n12 = t[6 * T], n02 = t[7 * T], n01 = t[8 * T];
        const double n3[3][3] = {{n00, n01, n02}, {n01, n11, n12}, {n02, n12, n22}};
        double tr = 0.0, nde = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          tr += dH[a][a];
#pragma unroll
          for (int b = 0; b < D; ++b) nde += n3[a][b] * 0.5 * (dH[a][b] + dH[b][a]);
        }
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b < D; ++b)
            P[a][b] = (a == b ? lam * tr : 0.0) + mu * (dH[a][b] + dH[b][a]) - g2 * nde * n3[a][b];
      } else {
        stress_linear<D>(m, dH, P);
      }
      const double wdet = G.wdet[q];
#pragma unroll
      for (int i = 0; i < npe; ++i)
#pragma unroll
        for (int a = 0; a < D; ++a) {
          double t = 0.0;
#pragma unroll
          for (int b = 0; b < D; ++b) t += P[a][b] * G.g[q][i][b];
          f[D * i + a] += wdet * t;
        }
    }
    ev_store<D>(ev, s.n_elem, e, f);
  }
}

template <int D>
void geo(const System& s, GeoT<D>& G) {
  std::memcpy(&G, s.grid_geo.data(), sizeof G);
}

template <int D, int MODE>
void run(System& s, const double* u, const uint8_t* mask, const double* x, double* y, double* dot_out = nullptr) {
  GeoT<D> G;
  static_assert(sizeof(GeoT<D>) == sizeof(double) * (EL<D>::nq * EL<D>::npe * D + EL<D>::nq), "layout");
  std::memcpy(&G, s.grid_geo.data(), sizeof G);
  if (!s.ev.p) s.ev.alloc((size_t)s.n_elem * EL<D>::nd);
  launch(*s.ctx, k_grid_elem<D, MODE>, grid_for(s.n_elem, 128, 148 * 64), 128, 0, G, s.view(), s.nx, s.ny, u, mask, x,
         s.ev.p);
  Ctx& c = *s.ctx;
  launch(c, k_gather<D>, std::min<unsigned>(grid_for(s.n_nodes, 256, 148 * 32), kRedBlocks * 4), 256, 0, s.view(),
         s.ev.p, MODE == EV_JVP ? mask : nullptr, x, y, nullptr, c.red_partials.p, c.red_counter.p,
         MODE == EV_JVP ? dot_out : nullptr);
}

template <int D>
void cached_tangent(System& s, const double* u, DevArray<double>& qpt) {
  GeoT<D> G;
  geo<D>(s, G);
  qpt.alloc((size_t)s.n_elem * EL<D>::nq * kQpt);
  launch(*s.ctx, k_grid_qp_tangent<D>, grid_for(s.n_elem, 128, 148 * 64), 128, 0, G, s.view(), s.nx, s.ny, u, qpt.p);
}

template <int D>
void cached_apply(System& s, const double* qpt, const uint8_t* mask, const double* x, double* y, const int* skip,
                  double* dot_out) {
  GeoT<D> G;
  geo<D>(s, G);
  if (!s.ev.p) s.ev.alloc((size_t)s.n_elem * EL<D>::nd);
  static const bool attr = [] {
    AFEM_CK(cudaFuncSetAttribute(k_grid_jvp_cached<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)jvp_cached_smem<D>()));
    return true;
  }();
  (void)attr;
  launch(*s.ctx, k_grid_jvp_cached<D>, grid_for(s.n_elem, kJvpThreads, 148 * 64), kJvpThreads, jvp_cached_smem<D>(),
         G, s.view(), s.nx, s.ny, qpt, mask, x, s.ev.p, skip);
  Ctx& c = *s.ctx;
  launch(c, k_gather<D>, std::min<unsigned>(grid_for(s.n_nodes, 256, 148 * 32), kRedBlocks * 4), 256, 0, s.view(),
         s.ev.p, mask, x, y, skip, c.red_partials.p, c.red_counter.p, dot_out);
}

}  // namespace

// J2 (+ linear) grid systems: the operator's Gauss-point tangents can be cached.
bool grid_tangent_cacheable(const System& s) {
  static const bool off = std::getenv("AFEM_NO_TANGENT_CACHE") != nullptr;
  if (off || !grid_elem_path(s) || !s.has_history()) return false;
  for (const DMat& m : s.mats)
    if (m.model != MODEL_LINEAR && m.model != MODEL_J2) return false;
  return true;
}

void grid_tangent_cache(System& s, const double* u, DevArray<double>& qpt) {
  if (s.dim == 2) cached_tangent<2>(s, u, qpt);
  else cached_tangent<3>(s, u, qpt);
}

void grid_mf_apply_cached(System& s, const double* qpt, const uint8_t* mask, const double* x, double* y,
                          const int* skip, double* dot_out) {
  if (s.dim == 2) cached_apply<2>(s, qpt, mask, x, y, skip, dot_out);
  else cached_apply<3>(s, qpt, mask, x, y, skip, dot_out);
}

void grid_geometry(System& s) {
  const size_t n = s.dim == 2 ? (4 * 4 * 2 + 4) : (8 * 8 * 3 + 8);
  DevArray<double> d(n);
  if (s.dim == 2) launch(*s.ctx, k_grid_geometry<2>, 1, 32, 0, s.coords.p, s.conn.p, d.p, s.err.p);
  else launch(*s.ctx, k_grid_geometry<3>, 1, 32, 0, s.coords.p, s.conn.p, d.p, s.err.p);
  s.grid_geo.resize(n);
  AFEM_CK(cudaMemcpyAsync(s.grid_geo.data(), d.p, n * 8, cudaMemcpyDeviceToHost, s.ctx->stream));
  AFEM_CK(cudaStreamSynchronize(s.ctx->stream));
}

bool grid_elem_path(const System& s) {
  static const bool off = std::getenv("AFEM_NO_GRID_ELEM") != nullptr;
  return s.grid && !s.grid_geo.empty() && !off;
}

void grid_residual(System& s, const double* u, double* r) {
  if (s.dim == 2) run<2, EV_RESIDUAL>(s, u, nullptr, nullptr, r);
  else run<3, EV_RESIDUAL>(s, u, nullptr, nullptr, r);
}

void grid_history_commit(System& s, const double* u) {
  GeoT<3> G;
  geo<3>(s, G);
  launch(*s.ctx, k_grid_history_commit<3>, grid_for(s.n_elem * 8, 128, 148 * 64), 128, 0, G, s.view(), s.nx, s.ny, u,
         s.hist.p);
}

void grid_jacobian(System& s, const double* u, double* values) {
  if (s.dim == 2) {
    GeoT<2> G;
    geo<2>(s, G);
    launch(*s.ctx, k_grid_jacobian<2>, grid_for(s.n_nodes, 128, 148 * 64), 128, 0, G, s.view(), s.nx, s.ny, u, values);
  } else {
    GeoT<3> G;
    geo<3>(s, G);
    static const bool node_centric = std::getenv("AFEM_NODE_JACOBIAN") != nullptr;
    const int64_t budget = (int64_t)1 << 31;  // element-block scratch bytes of the slab path
    const int64_t plane_bytes = (int64_t)s.nx * s.ny * kKe * 8;
    // the slab path holds at least two element planes of blocks (a slab plus its lower halo
    // plane); when that exceeds the budget (very wide xy grids) the node-centric kernel, which
    // needs no scratch, assembles instead
    if (node_centric || budget / plane_bytes < 2) {
      launch(*s.ctx, k_grid_jacobian<3>, grid_for(s.n_nodes, 128, 148 * 64), 128, 0, G, s.view(), s.nx, s.ny, u,
             values);
      return;
    }
    // z slabs of node planes; slab [k0, k1) needs element planes [k0 - 1, k1) (clamped)
    const int64_t epp = (int64_t)s.nx * s.ny, npp = (int64_t)(s.nx + 1) * (s.ny + 1);
    const int nzn = s.nz + 1;
    int S = static_cast<int>(std::max<int64_t>(1, budget / plane_bytes - 1));
    if (const char* e = std::getenv("AFEM_JAC_SLAB")) S = std::max(1, std::atoi(e));  // tests: force slabs
    if (!s.kscr.p || s.kscr.n < (size_t)std::min<int64_t>(S + 1, s.nz) * epp * kKe)
      s.kscr.alloc((size_t)std::min<int64_t>(S + 1, s.nz) * epp * kKe);
    for (int k0 = 0; k0 < nzn; k0 += S) {
      const int k1 = std::min(nzn, k0 + S);
      const int ea = std::max(0, k0 - 1), eb = std::min(s.nz, k1);
      const int64_t e0 = ea * epp, e1 = eb * epp;
      launch(*s.ctx, k_grid_kelem, grid_for((e1 - e0) * 32, 32 * kKelemWarps, 148 * 16), 32 * kKelemWarps, 0, G,
             s.view(), s.nx, s.ny, u, e0, e1, s.kscr.p);
      const int64_t n0 = k0 * npp, n1 = k1 * npp;
      launch(*s.ctx, k_grid_kgather, grid_for((n1 - n0) * 32, 32 * kGatherWarps, 148 * 16), 32 * kGatherWarps, 0,
             s.view(), s.nx, s.ny, s.nz, n0, n1, e0, s.kscr.p, values);
    }
  }
}

void grid_diagonal(System& s, const double* u, double* d) {
  if (s.dim == 2) run<2, EV_DIAG>(s, u, nullptr, nullptr, d);
  else run<3, EV_DIAG>(s, u, nullptr, nullptr, d);
}

void grid_mf_apply(System& s, const double* state, const uint8_t* mask, const double* x, double* y,
                   double* dot_out) {
  if (s.dim == 2) run<2, EV_JVP>(s, state, mask, x, y, dot_out);
  else run<3, EV_JVP>(s, state, mask, x, y, dot_out);
}

}  // namespace afem
