// Mesh ingestion / generation, batches, node incidence and the CSR sparsity pattern — all built on
// the device. Integer outputs are bit-exact with the reference:
//   generate_two_phase_mesh (mesh.hpp:47-85) and its hex8 twin: coordinates i*h and the strict
//     centroid test use __dmul_rn/__dadd_rn so no FMA contraction changes a phase label;
//   build_batches (assembly.hpp:36-67): batch order = phase order, element order preserved; here
//     the node incidence lists are sorted by (phase, element) so every gather sums in the
//     reference's (batch, element) scatter order;
//   precompute_sparsity (assembly.hpp:71-99): the sorted unique (row, col) set equals the dim x dim
//     expansion of the sorted node adjacency, which is what we build (no 64/576-pair sort).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>

#include "afem_impl.hpp"

namespace afem {

DMat make_dmat(int model, double E, double nu, double sigma_y, double hardening) {
  DMat m{};
  m.model = model;
  m.E = E;
  m.nu = nu;
  m.lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));  // material.hpp:20
  m.mu = E / (2.0 * (1.0 + nu));                     // material.hpp:21
  const double c = E / ((1.0 + nu) * (1.0 - 2.0 * nu));  // material.hpp:35-38
  m.c11 = c * (1.0 - nu);
  m.c12 = c * nu;
  m.c33 = c * (1.0 - 2.0 * nu) / 2.0;
  m.kappa = m.lam + 2.0 * m.mu / 3.0;
  m.sy = sigma_y;
  m.hh = hardening;
  return m;
}

void check_err(System& s) {
  int h = 0;
  AFEM_CK(cudaMemcpyAsync(&h, s.err.p, sizeof(int), cudaMemcpyDeviceToHost, s.ctx->stream));
  AFEM_CK(cudaStreamSynchronize(s.ctx->stream));
  if (h) {
    AFEM_CK(cudaMemsetAsync(s.err.p, 0, sizeof(int), s.ctx->stream));
    if (h & ERR_DETJ) throw std::invalid_argument("element_internal_force: non-positive element Jacobian");
    if (h & ERR_INVERTED) throw InvertedElementError("stress_svk: deformation gradient determinant <= 0");
    if (h & ERR_VALENCE) throw std::invalid_argument("mesh: node valence exceeds the supported maximum");
    throw std::runtime_error("device error flag set");
  }
}

namespace {

constexpr int kMaxAdj = 96;  // unique neighbours per node (structured hex8: 27)

__global__ void k_validate_mesh(const int32_t* conn, const int32_t* phase_in, int64_t n_elem, int npe,
                                int64_t n_nodes, int n_mat, uint8_t* phase_out, int* flags) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_elem; e += (int64_t)gridDim.x * blockDim.x) {
    const int p = phase_in[e];
    if (p < 0) atomicOr(flags, 1);
    else if (p >= n_mat) atomicOr(flags, 2);
    phase_out[e] = static_cast<uint8_t>(p < 0 ? 0 : (p > 255 ? 255 : p));
    for (int k = 0; k < npe; ++k) {
      const int32_t n = conn[e * npe + k];
      if (n < 0 || n >= n_nodes) atomicOr(flags, 4);
    }
  }
}

__global__ void k_iota(int32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = static_cast<int32_t>(i);
}

__global__ void k_widen(const unsigned int* a, int64_t* b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

__global__ void k_count_incidence(const int32_t* conn, int64_t total, unsigned int* cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[conn[i]], 1u);
}

__global__ void k_phase_hist(const uint8_t* phase, int64_t n_elem, unsigned long long* hist) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_elem; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[phase[e]], 1ull);
}

__global__ void k_fill_incidence(const int32_t* conn, int64_t n_elem, int npe, const int64_t* inc_ptr,
                                 unsigned int* cursor, uint32_t* inc) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_elem; e += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < npe; ++k) {
      const int32_t n = conn[e * npe + k];
      const unsigned int slot = atomicAdd(&cursor[n], 1u);
      inc[inc_ptr[n] + slot] = static_cast<uint32_t>(e * npe + k);
    }
}

// Sort each node's incidence list by (phase, element id): the reference's (batch, element) order.
__global__ void k_sort_incidence(const int64_t* inc_ptr, uint32_t* inc, const uint8_t* phase, int npe,
                                 int64_t n_nodes) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = inc_ptr[n], e = inc_ptr[n + 1];
    for (int64_t i = b + 1; i < e; ++i) {
      const uint32_t v = inc[i];
      const uint64_t kv = (static_cast<uint64_t>(phase[v / npe]) << 40) | (v / npe);
      int64_t j = i - 1;
      while (j >= b) {
        const uint32_t w = inc[j];
        const uint64_t kw = (static_cast<uint64_t>(phase[w / npe]) << 40) | (w / npe);
        if (kw <= kv) break;
        inc[j + 1] = w;
        --j;
      }
      inc[j + 1] = v;
    }
  }
}

// Unique sorted neighbour set of node n (including n) into nb[]; returns its size or -1 on overflow.
__device__ int node_neighbours(const int64_t* inc_ptr, const uint32_t* inc, const int32_t* conn, int npe, int64_t n,
                               int32_t* nb) {
  int cnt = 0;
  for (int64_t p = inc_ptr[n]; p < inc_ptr[n + 1]; ++p) {
    const uint32_t v = inc[p];
    const int64_t e = v / npe;
    for (int k = 0; k < npe; ++k) {
      const int32_t m = conn[e * npe + k];
      // insert m into sorted nb[0..cnt) if absent
      int lo = 0, hi = cnt;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (nb[mid] < m) lo = mid + 1; else hi = mid;
      }
      if (lo < cnt && nb[lo] == m) continue;
      if (cnt >= kMaxAdj) return -1;
      for (int t = cnt; t > lo; --t) nb[t] = nb[t - 1];
      nb[lo] = m;
      ++cnt;
    }
  }
  return cnt;
}

__global__ void k_count_adjacency(const int64_t* inc_ptr, const uint32_t* inc, const int32_t* conn, int npe,
                                  int64_t n_nodes, int64_t* deg, int* err) {
  int32_t nb[kMaxAdj];
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    const int c = node_neighbours(inc_ptr, inc, conn, npe, n, nb);
    if (c < 0) atomicOr(err, ERR_VALENCE);
    deg[n] = c < 0 ? 0 : c;
  }
}

__global__ void k_fill_adjacency(const int64_t* inc_ptr, const uint32_t* inc, const int32_t* conn, int npe,
                                 int64_t n_nodes, const int64_t* adj_ptr, int32_t* adj) {
  int32_t nb[kMaxAdj];
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    const int c = node_neighbours(inc_ptr, inc, conn, npe, n, nb);
    const int64_t b = adj_ptr[n];
    for (int i = 0; i < c; ++i) adj[b + i] = nb[i];
  }
}

// Dof-level CSR export (row_ptr closed-form from the node adjacency).
__global__ void k_export_pattern(const int64_t* adj_ptr, const int32_t* adj, int dim, int64_t n_nodes,
                                 int64_t* row_ptr, int32_t* rows, int32_t* cols) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a0 = adj_ptr[n];
    const int deg = static_cast<int>(adj_ptr[n + 1] - a0);
    for (int a = 0; a < dim; ++a) {
      const int64_t r = dim * n + a;
      const int64_t start = (int64_t)dim * dim * a0 + (int64_t)a * dim * deg;
      if (row_ptr) {
        row_ptr[r] = start;
        if (n == n_nodes - 1 && a == dim - 1) row_ptr[r + 1] = start + (int64_t)dim * deg;
      }
      for (int j = 0; j < deg; ++j)
        for (int b = 0; b < dim; ++b) {
          const int64_t k = start + (int64_t)j * dim + b;
          if (rows) rows[k] = static_cast<int32_t>(r);
          if (cols) cols[k] = dim * adj[a0 + j] + b;
        }
    }
  }
}

// ---- structured generators
__global__ void k_grid_coords(int dim, int nx, int ny, int nz, double hx, double hy, double hz, double* coords) {
  const int64_t nn = (int64_t)(nx + 1) * (ny + 1) * (dim == 3 ? nz + 1 : 1);
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nn; n += (int64_t)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(n % (nx + 1));
    const int64_t r = n / (nx + 1);
    const int j = static_cast<int>(r % (ny + 1));
    const int k = static_cast<int>(r / (ny + 1));
    coords[dim * n] = __dmul_rn(static_cast<double>(i), hx);
    coords[dim * n + 1] = __dmul_rn(static_cast<double>(j), hy);
    if (dim == 3) coords[dim * n + 2] = __dmul_rn(static_cast<double>(k), hz);
  }
}

__global__ void k_grid_elems(int dim, int nx, int ny, int nz, double hx, double hy, const double* incl, int n_incl,
                             double r2, int32_t* conn, int32_t* phase) {
  const int64_t ne = (int64_t)nx * ny * (dim == 3 ? nz : 1);
  const int npe = dim == 2 ? 4 : 8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const int ex = static_cast<int>(e % nx);
    const int64_t r = e / nx;
    const int ey = static_cast<int>(r % ny);
    const int ez = static_cast<int>(r / ny);
    auto node = [&](int i, int j, int k) -> int32_t {
      return static_cast<int32_t>(i + (int64_t)(nx + 1) * (j + (int64_t)(ny + 1) * k));
    };
    int32_t* c = conn + e * npe;
    c[0] = node(ex, ey, ez); c[1] = node(ex + 1, ey, ez); c[2] = node(ex + 1, ey + 1, ez); c[3] = node(ex, ey + 1, ez);
    if (dim == 3) {
      c[4] = node(ex, ey, ez + 1); c[5] = node(ex + 1, ey, ez + 1);
      c[6] = node(ex + 1, ey + 1, ez + 1); c[7] = node(ex, ey + 1, ez + 1);
    }
    int ph = 0;
    const double px = __dmul_rn(ex + 0.5, hx), py = __dmul_rn(ey + 0.5, hy);
    for (int f = 0; f < n_incl; ++f) {
      const double cx = __dsub_rn(px, incl[2 * f]);
      const double cy = __dsub_rn(py, incl[2 * f + 1]);
      if (__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)) < r2) { ph = 1; break; }
    }
    phase[e] = ph;
  }
}

template <class T>
void upload(Ctx& c, DevArray<T>& dst, const T* src, size_t n) {
  dst.alloc(n);
  if (n) AFEM_CK(cudaMemcpyAsync(dst.p, src, n * sizeof(T), cudaMemcpyHostToDevice, c.stream));
}

}  // namespace

// Incidence, batches and adjacency for a system whose coords/conn/phase are on the device.
static void build_topology(System& s, const int32_t* d_phase_in) {
  Ctx& c = *s.ctx;
  const int T = 256;
  const unsigned G = grid_for(std::max<int64_t>(s.n_elem, s.n_nodes), T, 148 * 32);
  s.err.alloc(1);
  AFEM_CK(cudaMemsetAsync(s.err.p, 0, sizeof(int), c.stream));
  s.phase.alloc(s.n_elem);
  DevArray<int> flags(1);
  AFEM_CK(cudaMemsetAsync(flags.p, 0, sizeof(int), c.stream));
  launch(c, k_validate_mesh, G, T, 0, s.conn.p, d_phase_in, s.n_elem, s.npe, s.n_nodes, (int)s.mats.size(),
         s.phase.p, flags.p);
  int hf = 0;
  AFEM_CK(cudaMemcpyAsync(&hf, flags.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  if (hf & 1) throw std::invalid_argument("build_batches: negative phase label");
  if (hf & 2) throw std::invalid_argument("build_batches: no material supplied for a mesh phase");
  if (hf & 4) throw std::out_of_range("precompute_sparsity: dof index outside system");

  // phase histogram -> batches (assembly.hpp:36-67: one per phase present, in phase order)
  DevArray<unsigned long long> hist(256);
  AFEM_CK(cudaMemsetAsync(hist.p, 0, hist.bytes(), c.stream));
  launch(c, k_phase_hist, G, T, 0, s.phase.p, s.n_elem, hist.p);
  std::vector<unsigned long long> hh(256);
  AFEM_CK(cudaMemcpyAsync(hh.data(), hist.p, hist.bytes(), cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  s.phase_count.assign(s.mats.size(), 0);
  for (size_t p = 0; p < s.mats.size(); ++p) s.phase_count[p] = static_cast<int64_t>(hh[p]);

  // element order (phase, id): stable radix sort of (phase key, id value)
  {
    DevArray<int32_t> ids(s.n_elem);
    launch(c, k_iota, G, T, 0, ids.p, s.n_elem);
    DevArray<uint8_t> kout(s.n_elem);
    s.elem_order.alloc(s.n_elem);
    size_t tmp = 0;
    AFEM_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, s.phase.p, kout.p, ids.p, s.elem_order.p, (int)s.n_elem, 0, 8,
                                            c.stream));
    DevArray<uint8_t> tbuf(tmp);
    AFEM_CK(cub::DeviceRadixSort::SortPairs(tbuf.p, tmp, s.phase.p, kout.p, ids.p, s.elem_order.p, (int)s.n_elem, 0, 8,
                                            c.stream));
    c.launches += 1;
    AFEM_CK(cudaStreamSynchronize(c.stream));
  }

  // node incidence
  DevArray<unsigned int> cnt(s.n_nodes + 1);
  AFEM_CK(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), c.stream));
  launch(c, k_count_incidence, G, T, 0, s.conn.p, s.n_elem * s.npe, cnt.p);
  {
    // widen counts and scan into inc_ptr (int64 offsets)
    DevArray<int64_t> cnt64(s.n_nodes);
    launch(c, k_widen, G, T, 0, cnt.p, cnt64.p, s.n_nodes);
    s.inc_ptr.alloc(s.n_nodes + 1);
    AFEM_CK(cudaMemsetAsync(s.inc_ptr.p, 0, sizeof(int64_t), c.stream));
    size_t tmp = 0;
    AFEM_CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt64.p, s.inc_ptr.p + 1, (int)s.n_nodes, c.stream));
    DevArray<uint8_t> tbuf(tmp);
    AFEM_CK(cub::DeviceScan::InclusiveSum(tbuf.p, tmp, cnt64.p, s.inc_ptr.p + 1, (int)s.n_nodes, c.stream));
    c.launches += 1;
    AFEM_CK(cudaStreamSynchronize(c.stream));
  }
  s.inc.alloc(s.n_elem * s.npe);
  AFEM_CK(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), c.stream));
  launch(c, k_fill_incidence, G, T, 0, s.conn.p, s.n_elem, s.npe, s.inc_ptr.p, cnt.p, s.inc.p);
  launch(c, k_sort_incidence, G, T, 0, s.inc_ptr.p, s.inc.p, s.phase.p, s.npe, s.n_nodes);

  // node adjacency (the pattern)
  DevArray<int64_t> deg(s.n_nodes + 1);
  launch(c, k_count_adjacency, grid_for(s.n_nodes, 128, 148 * 16), 128, 0, s.inc_ptr.p, s.inc.p, s.conn.p, s.npe,
         s.n_nodes, deg.p, s.err.p);
  check_err(s);
  s.adj_ptr.alloc(s.n_nodes + 1);
  AFEM_CK(cudaMemsetAsync(s.adj_ptr.p, 0, sizeof(int64_t), c.stream));
  {
    size_t tmp = 0;
    AFEM_CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, deg.p, s.adj_ptr.p + 1, (int)s.n_nodes, c.stream));
    DevArray<uint8_t> tbuf(tmp);
    AFEM_CK(cub::DeviceScan::InclusiveSum(tbuf.p, tmp, deg.p, s.adj_ptr.p + 1, (int)s.n_nodes, c.stream));
    c.launches += 1;
  }
  AFEM_CK(cudaMemcpyAsync(&s.adj_total, s.adj_ptr.p + s.n_nodes, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  s.adj.alloc(s.adj_total);
  launch(c, k_fill_adjacency, grid_for(s.n_nodes, 128, 148 * 16), 128, 0, s.inc_ptr.p, s.inc.p, s.conn.p, s.npe,
         s.n_nodes, s.adj_ptr.p, s.adj.p);
  s.nnz = static_cast<int64_t>(s.dim) * s.dim * s.adj_total;

  // empty Dirichlet table
  s.mask.alloc(s.n_dof);
  s.presc.alloc(s.n_dof);
  AFEM_CK(cudaMemsetAsync(s.mask.p, 0, s.mask.bytes(), c.stream));
  AFEM_CK(cudaMemsetAsync(s.presc.p, 0, s.presc.bytes(), c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
}

std::unique_ptr<System> make_system(Ctx& c, int dim, int64_t n_nodes, int64_t n_elem, const double* d_coords,
                                    const int32_t* d_conn, const int32_t* d_phase, const std::vector<DMat>& mats) {
  if (dim != 2 && dim != 3) throw std::invalid_argument("system: dim must be 2 (quad4) or 3 (hex8)");
  if (n_nodes < 1 || n_elem < 1) throw std::invalid_argument("system: empty mesh");
  if (mats.size() > (size_t)kMaxMat) throw std::invalid_argument("system: too many materials");
  for (const DMat& m : mats) {  // Material::validate (material.hpp:23-26)
    if (!(m.E > 0.0)) throw std::invalid_argument("material: E must be > 0");
    if (!(m.nu > -1.0 && m.nu < 0.5)) throw std::invalid_argument("material: nu must be in (-1, 0.5)");
    if (m.model < MODEL_LINEAR || m.model > MODEL_J2) throw std::invalid_argument("material: unsupported model");
    if (m.model == MODEL_J2 && !(m.sy > 0.0 && m.hh >= 0.0))
      throw std::invalid_argument("material: J2 needs sigma_y > 0 and hardening >= 0");
  }
  auto s = std::make_unique<System>();
  s->ctx = &c;
  s->dim = dim;
  s->npe = dim == 2 ? 4 : 8;
  s->n_nodes = n_nodes;
  s->n_elem = n_elem;
  s->n_dof = dim * n_nodes;
  if (n_elem * s->npe >= (int64_t)UINT32_MAX) throw std::invalid_argument("system: mesh too large");
  s->mats = mats;
  upload(c, s->d_mats, mats.data(), mats.size());
  s->coords.alloc(n_nodes * dim);
  s->conn.alloc(n_elem * s->npe);
  AFEM_CK(cudaMemcpyAsync(s->coords.p, d_coords, s->coords.bytes(), cudaMemcpyDeviceToDevice, c.stream));
  AFEM_CK(cudaMemcpyAsync(s->conn.p, d_conn, s->conn.bytes(), cudaMemcpyDeviceToDevice, c.stream));
  build_topology(*s, d_phase);
  bool j2 = false;
  for (const DMat& m : mats) j2 |= m.model == MODEL_J2;
  if (j2) {
    s->hist.alloc((size_t)n_elem * (dim == 2 ? 4 : 8) * kHist);
    history_reset(*s);
  }
  return s;
}

std::unique_ptr<System> make_grid_system(Ctx& c, int dim, int nx, int ny, int nz, double lx, double ly, double lz,
                                         const std::vector<double>& incl_xy, double radius,
                                         const std::vector<DMat>& mats) {
  if (nx < 1 || ny < 1 || (dim == 3 && nz < 1)) throw std::invalid_argument("mesh: cell counts must be >= 1");
  if (!(lx > 0.0) || !(ly > 0.0) || (dim == 3 && !(lz > 0.0)))
    throw std::invalid_argument("mesh: domain lengths must be > 0");
  if (radius < 0.0) throw std::invalid_argument("mesh: inclusion radius must be >= 0");
  if (dim != 2 && dim != 3) throw std::invalid_argument("system: dim must be 2 (quad4) or 3 (hex8)");
  const int64_t n_nodes = (int64_t)(nx + 1) * (ny + 1) * (dim == 3 ? nz + 1 : 1);
  const int64_t n_elem = (int64_t)nx * ny * (dim == 3 ? nz : 1);
  const int npe = dim == 2 ? 4 : 8;
  DevArray<double> coords(n_nodes * dim);
  DevArray<int32_t> conn(n_elem * npe), phase(n_elem);
  DevArray<double> incl;
  upload(c, incl, incl_xy.data(), incl_xy.size());
  const double hx = lx / nx, hy = ly / ny, hz = dim == 3 ? lz / nz : 1.0;
  launch(c, k_grid_coords, grid_for(n_nodes, 256, 148 * 32), 256, 0, dim, nx, ny, nz, hx, hy, hz, coords.p);
  launch(c, k_grid_elems, grid_for(n_elem, 256, 148 * 32), 256, 0, dim, nx, ny, nz, hx, hy, incl.p,
         (int)(incl_xy.size() / 2), radius * radius, conn.p, phase.p);
  auto s = make_system(c, dim, n_nodes, n_elem, coords.p, conn.p, phase.p, mats);
  s->grid = true;
  s->nx = nx; s->ny = ny; s->nz = dim == 3 ? nz : 0;
  s->lx = lx; s->ly = ly; s->lz = dim == 3 ? lz : 0.0;
  grid_geometry(*s);
  return s;
}

// validate_dirichlet (mesh.hpp:105-116) + constraint_table (assembly.hpp:197-211).
void set_dirichlet(System& s, const std::vector<Constraint>& cs) {
  std::vector<uint8_t> mask(s.n_dof, 0);
  std::vector<double> presc(s.n_dof, 0.0);
  for (const auto& c : cs) {
    if (c.node < 0 || c.node >= s.n_nodes) throw std::out_of_range("dirichlet: constrained node outside mesh");
    if (c.comp < 0 || c.comp >= s.dim)
      throw std::invalid_argument(s.dim == 2 ? "dirichlet: component must be 0 (x) or 1 (y)"
                                             : "dirichlet: component must be 0, 1 or 2");
    const int64_t d = (int64_t)s.dim * c.node + c.comp;
    if (mask[d]) throw std::invalid_argument("dirichlet: duplicate (node, component) pair");
    mask[d] = 1;
    presc[d] = c.value;
  }
  Ctx& c = *s.ctx;
  AFEM_CK(cudaMemcpyAsync(s.mask.p, mask.data(), s.mask.bytes(), cudaMemcpyHostToDevice, c.stream));
  AFEM_CK(cudaMemcpyAsync(s.presc.p, presc.data(), s.presc.bytes(), cudaMemcpyHostToDevice, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  s.constraints = cs;
}

// benchmark_bcs (mesh.hpp:89-101) and its 3D twin (SURVEY §8d C2 BCs).
std::vector<Constraint> benchmark_bcs(const System& s, double strain) {
  if (!s.grid) throw std::invalid_argument("benchmark_bcs: mesh lacks structured-grid metadata");
  std::vector<Constraint> c;
  const double u_right = strain * s.lx;
  const int nx = s.nx, ny = s.ny, nz = s.nz;
  if (s.dim == 2) {
    auto node = [&](int i, int j) { return i + j * (nx + 1); };
    for (int j = 0; j <= ny; ++j) c.push_back({node(0, j), 0, 0.0});
    c.push_back({node(0, 0), 1, 0.0});
    for (int j = 0; j <= ny; ++j) c.push_back({node(nx, j), 0, u_right});
  } else {
    auto node = [&](int i, int j, int k) { return i + (nx + 1) * (j + (ny + 1) * k); };
    for (int k = 0; k <= nz; ++k)
      for (int j = 0; j <= ny; ++j) c.push_back({node(0, j, k), 0, 0.0});
    c.push_back({node(0, 0, 0), 1, 0.0});
    c.push_back({node(0, 0, 0), 2, 0.0});
    c.push_back({node(0, 0, nz), 1, 0.0});
    for (int k = 0; k <= nz; ++k)
      for (int j = 0; j <= ny; ++j) c.push_back({node(nx, j, k), 0, u_right});
  }
  return c;
}

void pattern_export(System& s, int64_t* d_row_ptr, int32_t* d_rows, int32_t* d_cols) {
  launch(*s.ctx, k_export_pattern, grid_for(s.n_nodes, 128, 148 * 32), 128, 0, s.adj_ptr.p, s.adj.p, s.dim, s.n_nodes,
         d_row_ptr, d_rows, d_cols);
}

// ElementBatch b (assembly.hpp:22-31, 44-65): b indexes the non-empty phases in phase order.
void batch_export(System& s, int b, int64_t* size, int32_t* h_ids, int32_t* h_dof_map) {
  int64_t off = 0;
  int phase = -1, k = 0;
  for (size_t p = 0; p < s.phase_count.size(); ++p) {
    if (s.phase_count[p] == 0) continue;
    if (k == b) { phase = (int)p; break; }
    off += s.phase_count[p];
    ++k;
  }
  if (phase < 0) throw std::out_of_range("batch index outside the batch list");
  const int64_t sz = s.phase_count[phase];
  *size = sz;
  if (!h_ids && !h_dof_map) return;
  std::vector<int32_t> ids(sz), conn(sz * s.npe);
  AFEM_CK(cudaMemcpyAsync(ids.data(), s.elem_order.p + off, sz * 4, cudaMemcpyDeviceToHost, s.ctx->stream));
  std::vector<int32_t> all(s.n_elem * s.npe);
  AFEM_CK(cudaMemcpyAsync(all.data(), s.conn.p, all.size() * 4, cudaMemcpyDeviceToHost, s.ctx->stream));
  AFEM_CK(cudaStreamSynchronize(s.ctx->stream));
  if (h_ids) std::memcpy(h_ids, ids.data(), sz * 4);
  if (h_dof_map)
    for (int64_t i = 0; i < sz; ++i)
      for (int q = 0; q < s.npe; ++q)
        for (int c = 0; c < s.dim; ++c)
          h_dof_map[(i * s.npe + q) * s.dim + c] = s.dim * all[ids[i] * s.npe + q] + c;
}

}  // namespace afem
