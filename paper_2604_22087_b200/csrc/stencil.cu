// Structured-grid fast path for the linear matrix-free operator y = K x (backend.hpp:130-147) on
// hex8 grid systems (afem_system_create_grid, dim 3) whose phases are all linear elastic with a
// common Poisson ratio. Then every element stiffness is K_e = E_phase * Khat (Khat: the uniform
// brick at E = 1) and, with octant o of node n the element on side o of n,
//     y_n = sum_{o exists} E_o Khat_rows(o) x_e(o)
//         = E_base(n) (S_f x)_n + sum_{o in F(n), E_o != E_base} (E_o - E_base) Khat_rows(o) x_e(o)
// S_f is the assembled stencil of the octant family F(n): all 8 octants in the interior, the
// half / quarter families on y and z boundary faces (the void octants are dropped exactly by the
// coefficients), and E_base(n) the majority modulus over F(n) (octants void in x count as E = 0).
//
// Kernels:
//  k_stencil_tma    64x4 node tile per CTA (4 warps, one row per warp, 2 nodes per lane; one wave of
//                   4 CTAs per SM, each taking an equal contiguous range of (tile, plane) units),
//                   marching in z. Each plane's TY + 2 staged rows (one-node halo, interleaved dofs)
//                   and their info bytes arrive by TMA (rank-1 cp.async.bulk.tensor copies issued by
//                   lane 0 of every warp, one mbarrier per ring slot, a 4-slot ring); out-of-range
//                   columns and Dirichlet dofs are zeroed after landing from the staged info bytes.
//                   Each lane keeps the partial sums of the six column nodes a plane touches. 153
//                   DFMA per interior node (the 243-entry stencil minus the 90 symmetry zeros) over
//                   30 symmetry-unique coefficients in uniform registers; y / z faces switch to the
//                   half / quarter families (warp- or CTA-uniform). No atomics; every y entry of the
//                   covered columns is written exactly once; optional fused x.y partials (CG p.Ap).
//  k_stencil_items  one thread per (node, octant) correction: mixed-family nodes (fibre
//                   interfaces, the x = 0 face) add dE Khat_rows x_e; the NX mod 64 edge columns are
//                   written in exact octant form. Segmented, fixed-order shuffle sums per node.
// Algorithmic traffic of the main kernel: x (8 B/dof) + y (8 B/dof) + one info byte per node.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "afem_impl.hpp"
#include "reduce.cuh"
#include "tma.cuh"

namespace afem {

constexpr int kVoid = 31;  // phase code of an octant outside the domain (E = 0)

struct StencilParams {
  double HY[2][9][3][3];       // y face lo/hi, entries with dy = 0: index (dx+1) + 3(dz+1)
  double HZ[2][9][3][3];       // z face lo/hi, entries with dz = 0: index (dx+1) + 3(dy+1)
  double HYZ[2][2][3][3][3];   // y and z faces, entries with dy = dz = 0: index dx+1
  // Interior family by symmetry: S(d)_aa = Dg[a][|dx|][|dy|][|dz|];
  // S(d)_ab = sgn(d_a) sgn(d_b) Og[pair(a,b)][|d_c|] (a != b, c the third axis; zero if d_a d_b = 0).
  double Dg[3][2][2][2];
  double Og[3][2];             // pairs xy, xz, yz
  double E[32];                // modulus per phase code (E[kVoid] = 0)
  int NX, NY, NZ;              // node counts per axis
  int NXm;                     // node columns the main kernel covers (tiles of 64; the last may be partial)
};

// Rows of Khat for the element corner at bit position 0 (hex node local_node(0, 0, 0)), columns in
// bit-corner order: k[a][3 b + c] = Khat(node 0, corner with bits b)[a][c]. The brick is symmetric
// under the reflections of each axis, so every other corner's rows follow by reflecting the
// element (permuted corners, sign flips of the reflected components): the coefficients are the
// same for every lane and live in the constant bank.
struct RowsK0 {
  double k[3][24];
};

struct StencilPlan {
  StencilParams p;
  DevArray<uint8_t> info;       // per node: bits 0-2 Dirichlet mask, bits 3-7 base phase code
  // correction items (k_stencil_items): mixed-family nodes and the edge columns
  DevArray<uint64_t> it_rec;
  DevArray<uint32_t> it_zm;
  DevArray<double> Ed;   // modulus per phase code (32), device copy for the item kernel
  int item_blocks = 1;
  DevArray<double> part_main, part_items;  // fused p.Ap partials (main kernel, item kernel)
  DevArray<unsigned int> counter;
  DevArray<double> Kg;   // Khat (row-major 24 x 24)
  RowsK0 k0;             // the correction kernel's coefficients
  int64_t n_items = 0;   // tile correction items incl. padding
  int64_t n_fix_nodes = 0, n_edge_nodes = 0;
  int kchunk = 16;
  int nchunks = 1;
  int main_blocks = 1;  // balanced main-kernel grid
  // the plain apply (no fused dot, no skip flag) as instantiated two-kernel graphs keyed on (x, y):
  // a pair's graph is captured on its second use (a pointer pair seen once, e.g. one GMRES basis
  // vector, launches directly) and the kGraphSlots most recent pairs stay instantiated
  static constexpr int kGraphSlots = 8;
  struct GraphSlot {
    const double* x = nullptr;
    double* y = nullptr;
    cudaGraphExec_t exec = nullptr;
    uint64_t used = 0;
  } graphs[kGraphSlots];
  uint64_t graph_clock = 0;
  ~StencilPlan() {
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
  }
  // z pieces for the pipelined host-buffer apply (afem_op_apply with host x / y): items are
  // ordered piece-major, piece_items[p] = first item of piece p (multiple of 32)
  int zpiece = 16;
  int npieces = 1;
  std::vector<int64_t> piece_items;
  int iocc = 1;
  // TMA staging of the main kernel (k_stencil_tma): info map once per plan, x map per x pointer
  DevArray<uint8_t> info_pad;  // the TMA kernel's padded info rows (k_info_pad)
  int ipx = 0;
  CUtensorMap mi{}, mx{};
  const double* mx_ptr = nullptr;
  int xshift = 0;
};

namespace {

// Main-kernel tile: TY warps, one node row per warp, each lane owns 2 adjacent x nodes (64 per row).
// TY = 4 (4 CTAs / SM) measured 10 % faster than TY = 8 (2 CTAs / SM): the per-plane barrier spans
// fewer warps and the other CTAs on the SM keep the FP64 pipe busy meanwhile.
#ifndef AFEM_STENCIL_TY
#define AFEM_STENCIL_TY 4
#endif
constexpr int TX = 32, TXN = 2 * TX, TY = AFEM_STENCIL_TY, NT = TX * TY;
#ifndef AFEM_MAIN_MINB
#define AFEM_MAIN_MINB (16 / TY)  // 4 CTAs x 4 warps (5 CTAs at <= 96 registers measured 2 % slower)
#endif
constexpr int kMainBlocksPerSm = AFEM_MAIN_MINB;

// Structural zero of a family's entry (a, b) at offset d: the brick's reflection symmetry about
// an axis c that the family keeps intact makes every off-diagonal entry involving c vanish when
// d_c = 0. broken: bit 1 = y symmetry broken (y face), bit 2 = z symmetry broken (z face).
__host__ __device__ constexpr bool szero(int dx, int dy, int dz, int a, int b, int broken) {
  if (a == b) return false;
  for (int c = 0; c < 3; ++c) {
    if (c != a && c != b) continue;
    if ((broken >> c) & 1) continue;
    const int dc = c == 0 ? dx : (c == 1 ? dy : dz);
    if (dc == 0) return true;
  }
  return false;
}

template <int DX, int DY, int DZ, int A>
constexpr int dcomp() { return A == 0 ? DX : (A == 1 ? DY : DZ); }

// Coefficient of entry (d, a, b) for a node on y face YF / z face ZF (0 none, 1 lo, 2 hi). Interior
// entries come from the 30 symmetry-unique values (they stay resident in uniform registers).
template <int DX, int DY, int DZ, int YF, int ZF, int A, int B>
__device__ __forceinline__ double coef(const StencilParams& P) {
  constexpr bool yb = YF != 0 && DY == 0;
  constexpr bool zb = ZF != 0 && DZ == 0;
  if constexpr (yb && zb) return P.HYZ[YF - 1][ZF - 1][DX + 1][A][B];
  else if constexpr (yb) return P.HY[YF - 1][(DX + 1) + 3 * (DZ + 1)][A][B];
  else if constexpr (zb) return P.HZ[ZF - 1][(DX + 1) + 3 * (DY + 1)][A][B];
  else if constexpr (A == B) return P.Dg[A][DX != 0][DY != 0][DZ != 0];
  else {
    constexpr int C = 3 - A - B;
    constexpr int pair = (A + B == 1) ? 0 : (A + B == 2 ? 1 : 2);
    constexpr int sg = dcomp<DX, DY, DZ, A>() * dcomp<DX, DY, DZ, B>();
    const double v = P.Og[pair][dcomp<DX, DY, DZ, C>() != 0];
    return sg > 0 ? v : -v;
  }
}

template <int DX, int DY, int DZ, int YF, int ZF>
constexpr int broken_of() {
  return ((YF != 0 && DY == 0) ? 2 : 0) | ((ZF != 0 && DZ == 0) ? 4 : 0);
}

// acc[n][r][a]: node n (0, 1) of the lane, role r (0: node below the plane sees dz = +1, 1: node on
// the plane dz = 0, 2: node above dz = -1), component a. One neighbour column (DI, DJ), one input
// component B, the two nodes' inputs x0, x1. RM: the roles computed (bit r); a segment's first
// plane only feeds the node above it (RM 4) and its last plane only the node below (RM 1).
template <int DI, int DJ, int YF, int ZF, int B, int RM>
__device__ __forceinline__ void nb(const StencilParams& P, double x0, double x1, double (&acc)[2][3][3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if constexpr ((RM & 1) != 0) {
      if (!szero(DI, DJ, 1, a, B, broken_of<DI, DJ, 1, YF, 0>())) {
        const double c = a == 0 ? coef<DI, DJ, 1, YF, 0, 0, B>(P) : (a == 1 ? coef<DI, DJ, 1, YF, 0, 1, B>(P)
                                                                              : coef<DI, DJ, 1, YF, 0, 2, B>(P));
        acc[0][0][a] = fma(c, x0, acc[0][0][a]);
        acc[1][0][a] = fma(c, x1, acc[1][0][a]);
      }
    }
    if constexpr ((RM & 2) != 0) {
      if (!szero(DI, DJ, 0, a, B, broken_of<DI, DJ, 0, YF, ZF>())) {
        const double c = a == 0 ? coef<DI, DJ, 0, YF, ZF, 0, B>(P) : (a == 1 ? coef<DI, DJ, 0, YF, ZF, 1, B>(P)
                                                                               : coef<DI, DJ, 0, YF, ZF, 2, B>(P));
        acc[0][1][a] = fma(c, x0, acc[0][1][a]);
        acc[1][1][a] = fma(c, x1, acc[1][1][a]);
      }
    }
    if constexpr ((RM & 4) != 0) {
      if (!szero(DI, DJ, -1, a, B, broken_of<DI, DJ, -1, YF, 0>())) {
        const double c = a == 0 ? coef<DI, DJ, -1, YF, 0, 0, B>(P) : (a == 1 ? coef<DI, DJ, -1, YF, 0, 1, B>(P)
                                                                               : coef<DI, DJ, -1, YF, 0, 2, B>(P));
        acc[0][2][a] = fma(c, x0, acc[0][2][a]);
        acc[1][2][a] = fma(c, x1, acc[1][2][a]);
      }
    }
  }
}

// The 12 interleaved dofs of the lane's window in one staged row (left neighbour, node 0, node 1,
// right neighbour): 12 LDS.64 at the row's offset (TMA boxes start on 16-byte boundaries, so a row
// lands 0 or 1 double in). 48-byte lane stride: two-way conflicts per half-warp, the same shared
// wavefronts as 16-byte loads of an aligned row, and no per-row code variants.
#ifndef AFEM_STENCIL_LDS128
#define AFEM_STENCIL_LDS128 0
#endif
__device__ __forceinline__ void load_window(const double* __restrict__ srow, int tx, int off, double (&w)[12]) {
#if AFEM_STENCIL_LDS128
  // 16-byte loads (half the shared wavefronts of 8-byte loads at this 48-byte lane stride): the row
  // base and 6 tx doubles are 16-byte aligned, so offset 0 is 6 aligned pairs and offset 1 is 7
  // pairs shifted by one element (warp-uniform branch)
  const double2* r2 = reinterpret_cast<const double2*>(srow + 6 * tx);
  if (off == 0) {
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const double2 v = r2[k];
      w[2 * k] = v.x;
      w[2 * k + 1] = v.y;
    }
  } else {
    double2 v[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) v[k] = r2[k];
#pragma unroll
    for (int k = 0; k < 12; ++k) w[k] = ((k + 1) & 1) ? v[(k + 1) >> 1].y : v[(k + 1) >> 1].x;
  }
#else
  const double* r = srow + off + 6 * tx;
#pragma unroll
  for (int k = 0; k < 12; ++k) w[k] = r[k];
#endif
}

template <int DJ, int YF, int ZF, int RM>
__device__ __forceinline__ void row_step(const StencilParams& P, const double* __restrict__ srow, int tx, int off,
                                         double (&acc)[2][3][3]) {
  double w[12];
  load_window(srow, tx, off, w);
  nb<-1, DJ, YF, ZF, 0, RM>(P, w[0], w[3], acc);
  nb<-1, DJ, YF, ZF, 1, RM>(P, w[1], w[4], acc);
  nb<-1, DJ, YF, ZF, 2, RM>(P, w[2], w[5], acc);
  nb<0, DJ, YF, ZF, 0, RM>(P, w[3], w[6], acc);
  nb<0, DJ, YF, ZF, 1, RM>(P, w[4], w[7], acc);
  nb<0, DJ, YF, ZF, 2, RM>(P, w[5], w[8], acc);
  nb<1, DJ, YF, ZF, 0, RM>(P, w[6], w[9], acc);
  nb<1, DJ, YF, ZF, 1, RM>(P, w[7], w[10], acc);
  nb<1, DJ, YF, ZF, 2, RM>(P, w[8], w[11], acc);
}

// offs: bit r = the window offset of staged row ty + r
template <int YF, int ZF, int STRIDE, int RM>
__device__ __forceinline__ void plane_step(const StencilParams& P, const double* __restrict__ s, int tx, int ty,
                                           int offs, double (&acc)[2][3][3]) {
  row_step<-1, YF, ZF, RM>(P, s + (ty + 0) * STRIDE, tx, offs & 1, acc);
  row_step<0, YF, ZF, RM>(P, s + (ty + 1) * STRIDE, tx, (offs >> 1) & 1, acc);
  row_step<1, YF, ZF, RM>(P, s + (ty + 2) * STRIDE, tx, (offs >> 2) & 1, acc);
}

template <int YF, int STRIDE, int RM>
__device__ __forceinline__ void plane_dispatch(const StencilParams& P, const double* s, int tx, int ty, int zc,
                                               double (&acc)[2][3][3], int offs) {
  if (zc == 0) plane_step<YF, 0, STRIDE, RM>(P, s, tx, ty, offs, acc);
  else if (zc == 1) plane_step<YF, 1, STRIDE, RM>(P, s, tx, ty, offs, acc);
  else plane_step<YF, 2, STRIDE, RM>(P, s, tx, ty, offs, acc);
}

template <int STRIDE, int RM>
__device__ __forceinline__ void plane_any(const StencilParams& P, const double* s, int tx, int ty, int yf, int zc,
                                          double (&acc)[2][3][3], int offs) {
  if (yf == 0) plane_dispatch<0, STRIDE, RM>(P, s, tx, ty, zc, acc, offs);
  else if (yf == 1) plane_dispatch<1, STRIDE, RM>(P, s, tx, ty, zc, acc, offs);
  else plane_dispatch<2, STRIDE, RM>(P, s, tx, ty, zc, acc, offs);
}

__host__ __device__ __forceinline__ int local_node(int lx, int ly, int lz) {
  const int ring = lx ? (ly ? 2 : 1) : (ly ? 3 : 0);  // element.hpp:22-23 ring, then z = +1
  return ring + 4 * lz;
}
__host__ __device__ __forceinline__ int corner_x(int m) { return ((m & 3) == 1 || (m & 3) == 2) ? 1 : 0; }
__host__ __device__ __forceinline__ int corner_y(int m) { return (m & 3) >= 2 ? 1 : 0; }

// DOT: also accumulate x.y (the CG p^T A p) into per-block partials; when `finish`, the last block
// completes the fixed-order reduction into dot_out (otherwise k_stencil_items does).
struct DotArgs {
  double* part_main;
  double* part_items;
  unsigned int* counter;
  double* out;
  int finish;
  int n_main;  // number of main-kernel partials (read by the items kernel's last block)
  const int* skip;  // CG speculation: the apply is a no-op while *skip != 0
};

// Planes per CTA barrier (PPB) and ring slots: the output plane pb - 1, PPB computing, and the
// landed / in-flight planes (2 for PPB = 1, PPB otherwise). PPB = 2 halves the barriers but was
// measured slower (ncu 53.2 -> 56.8 us, profiles/r02_*): the barrier stall is the warps' skew, not
// the barrier count.
#ifndef AFEM_STENCIL_PPB
#define AFEM_STENCIL_PPB 1
#endif
constexpr int PPB = AFEM_STENCIL_PPB;
constexpr int RING = 2 * PPB + (PPB == 1 ? 2 : 1);

// k_stencil_tma: the main kernel with Blackwell bulk-async staging. Per CTA plane the (TY + 2)
// rows of the 64 + 2 node window (interleaved dofs) and their info bytes arrive by TMA: rank-1
// tensor copies (cp.async.bulk.tensor.1d; boxes start on 16-byte boundaries, zero fill outside
// [0, n)) issued by lane 0 of each warp and completed on one mbarrier per ring slot — no per-thread address
// arithmetic and no registers spent on staging. x rows: the box starts at the even element at or
// below the row's first dof, so a row lands 0 or 1 double in (its parity, known to every thread;
// load_window reads either). Info rows come from a padded copy of the info bytes (row pitch ipx, a
// multiple of 16, >= 16 pad bytes of value 7 = "all components masked" before every row start and
// after every tile's last column), so a row's box always starts 16-byte aligned, 15 bytes before
// the window. Rows outside the y range are never copied (their slot rows are zeroed once per
// segment); columns outside [0, NX) and Dirichlet dofs are zeroed by one masking pass per plane
// from the staged info bytes (one 4-byte word per thread, an early out when it holds no constrained
// dof). Ring of 4 slots: plane p is computed, p + 1 is landed and masked, p + 2 is in flight, and
// p + 3 is issued into p - 1's slot after the plane barrier (a proxy fence orders the threads'
// generic writes before the async-proxy overwrite). Arithmetic, output order and the fused dot are
// those of the round-1 cp.async kernel (k_stencil_main, removed), so results are bitwise unchanged.
constexpr int RSP = 208;             // staged row pitch (doubles): 200 landed, rows 128-byte aligned for TMA
constexpr int IRP = 128;             // staged info row pitch (bytes)
constexpr int XBOX = 3 * (TXN + 2) + 2;  // doubles per x box (the 198-dof window + alignment slack)
constexpr int IBOX = 96;             // info bytes per box (15 pad + 66 window, rounded to 16)
constexpr int IOFF = 15;             // window byte offset inside an info box
constexpr int IW0 = IOFF / 4, IW1 = (IOFF + TXN + 2 + 3) / 4;  // info words touching the window
constexpr int IWORDS = IW1 - IW0;
constexpr size_t kTmaSmem = 128 + sizeof(double) * RING * (TY + 2) * RSP + RING * (TY + 2) * IRP +
                            8 * RING + 8 * 32;
static_assert((TY + 2) * IWORDS <= NT, "one info word per thread");
static_assert(XBOX <= RSP && IBOX <= IRP && XBOX <= 256, "TMA box sizes");

template <bool DOT>
__global__ void __launch_bounds__(NT, kMainBlocksPerSm)
    k_stencil_tma(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mi,
                  const __grid_constant__ StencilParams P, int xshift, int ipx, const double* __restrict__ x,
                  double* __restrict__ y, int kchunk, int kbeg, int kend, DotArgs dot, int ntx, int nty) {
  if (dot.skip && *dot.skip) return;
  double dsum = 0.0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 128-byte aligned base, derived from smem_raw itself so the compiler keeps shared-space
  // accesses (LDS / STS, not generic loads)
  unsigned char* const base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  double (*xs)[TY + 2][RSP] = reinterpret_cast<double (*)[TY + 2][RSP]>(base);
  uint8_t (*is)[TY + 2][IRP] =
      reinterpret_cast<uint8_t (*)[TY + 2][IRP]>(base + sizeof(double) * RING * (TY + 2) * RSP);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + sizeof(double) * RING * (TY + 2) * RSP + RING * (TY + 2) * IRP);
  double* Es = reinterpret_cast<double*>(bars + RING);
  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int NX = P.NX, NY = P.NY, NZ = P.NZ;
  if (tid < 32) Es[tid] = P.E[tid];
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < RING; ++q) mbar_init(smem_u32(&bars[q]), 1);
    mbar_init_fence();
  }
  __syncthreads();
  uint32_t phase = 0;  // bit s: parity of slot s's next completion
  auto ring = [](int p) { return (p + 1) % RING; };  // p >= -1
  const int nzr = kend - kbeg;
  int64_t u = 0, ue = 1;
  if (kchunk <= 0) {
    const int64_t U = (int64_t)ntx * nty * nzr;
    u = U * blockIdx.x / gridDim.x;
    ue = U * (blockIdx.x + 1) / gridDim.x;
  }
  while (u < ue) {
    int bx, by, k0, k1;
    if (kchunk > 0) {
      bx = blockIdx.x;
      by = blockIdx.y;
      k0 = kbeg + blockIdx.z * kchunk;
      k1 = min(k0 + kchunk, kend);
      u = ue;
    } else {
      const int tile = static_cast<int>(u / nzr), kk = static_cast<int>(u % nzr);
      const int kl = static_cast<int>(min(static_cast<int64_t>(nzr), kk + (ue - u)));
      bx = tile % ntx;
      by = tile / ntx;
      k0 = kbeg + kk;
      k1 = kbeg + kl;
      u += kl - kk;
    }
    const int i0 = bx * TXN, j0 = by * TY;
    const int i = i0 + 2 * tx, j = j0 + ty;
    const bool active = j < NY;
    const bool v0 = i < P.NXm, v1 = i + 1 < P.NXm;
    const int yf = j == 0 ? 1 : (j == NY - 1 ? 2 : 0);
    // window offset (0 / 1 double) of staged row r of plane p: parity of its first dof's element
    auto roff = [&](int r, int p) -> int {
      return (1 + NX * ((j0 - 1 + r) + NY * p) + xshift) & 1;  // 3 (i0 - 1 + ...) = i0 - 1 + ... mod 2
    };

    // rows outside [0, NY) are never copied: zero them in every slot for this segment
    __syncthreads();
    for (int r = 0; r < TY + 2; ++r) {
      const int jj = j0 - 1 + r;
      if (jj >= 0 && jj < NY) continue;
      for (int q = tid; q < RING * RSP; q += NT) xs[q / RSP][r][q % RSP] = 0.0;
    }
    __syncthreads();
    // plane p into its slot, issued by lane 0 of every warp (warp w copies rows w, w + TY, ...; warp
    // 0 also posts the expected bytes — a copy may complete first, the phase still needs that
    // arrival), so no single warp carries the issue work into the next barrier
    auto issue = [&](int p) {
      if ((tid & 31) != 0) return;
      const int w = tid >> 5;
      const int sl = ring(p);
      const uint32_t bar = smem_u32(&bars[sl]);
      fence_proxy_async_smem();  // this thread's view of the slot's generic writes before the overwrite
      if (p < 0 || p >= NZ) {
        if (w == 0) mbar_arrive(bar);
        return;
      }
      if (w == 0) {
        int rows = 0;
#pragma unroll
        for (int r = 0; r < TY + 2; ++r) rows += (j0 - 1 + r >= 0 && j0 - 1 + r < NY) ? 1 : 0;
        mbar_arrive_expect_tx(bar, static_cast<uint32_t>(rows * (XBOX * 8 + IBOX)));
      }
      for (int r = w; r < TY + 2; r += TY) {
        const int jj = j0 - 1 + r;
        if (jj < 0 || jj >= NY) continue;
        const int row = jj + NY * p;
        const int c = 3 * (i0 - 1 + NX * row) + xshift;  // < 2^31 (make_stencil_plan)
        tma_load_1d(smem_u32(&xs[sl][r][0]), &mx, c & ~1, bar);
        tma_load_1d(smem_u32(&is[sl][r][0]), &mi, i0 + ipx * row, bar);
      }
    };
    auto wait = [&](int p) {
      const int sl = ring(p);
      mbar_wait(smem_u32(&bars[sl]), (phase >> sl) & 1u);
      phase ^= 1u << sl;
    };
    auto mask = [&](int p) {  // zero out-of-range columns and Dirichlet dofs of landed plane p
      if (p < 0 || p >= NZ || tid >= (TY + 2) * IWORDS) return;
      const int sl = ring(p);
      const int r = tid / IWORDS, wb = 4 * (IW0 + tid - IWORDS * r);  // the word's first byte
      const int jj = j0 - 1 + r;
      if (jj < 0 || jj >= NY) return;
      const uint32_t word = *reinterpret_cast<const uint32_t*>(&is[sl][r][wb]);
      if (!(word & 0x07070707u)) return;
      double* row = &xs[sl][r][roff(r, p)];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int col = wb + b - IOFF;
        if (col < 0 || col >= TXN + 2) continue;
        const uint32_t m = (word >> (8 * b)) & 7u;
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if ((m >> c) & 1u) row[3 * col + c] = 0.0;
      }
    };

    double acc[2][3][3];
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int a = 0; a < 3; ++a) acc[n][r][a] = 0.0;
    // one CTA barrier per PPB planes: planes pb .. pb + PPB - 1 are computed back to back (step p
    // also writes the nodes of plane p - 1), the next PPB are waited for and masked, then the
    // barrier frees the slots of planes pb - 1 .. pb + PPB - 2 for the planes RING - 1 ahead
#pragma unroll
    for (int q = 0; q < RING - 1; ++q)
      if (k0 - 1 + q <= k1) issue(k0 - 1 + q);
#pragma unroll
    for (int q = 0; q < PPB; ++q)
      if (k0 - 1 + q <= k1) {
        wait(k0 - 1 + q);
        mask(k0 - 1 + q);
      }
    __syncthreads();
    for (int pb = k0 - 1; pb <= k1; pb += PPB) {
#pragma unroll 1
      for (int p = pb; p < pb + PPB && p <= k1; ++p) {
        if (active && p >= 0 && p < NZ) {
          const int zc = p == 0 ? 1 : (p == NZ - 1 ? 2 : 0);
          const double* sp = &xs[ring(p)][0][0];
          const int offs = roff(ty, p) | (roff(ty + 1, p) << 1) | (roff(ty + 2, p) << 2);
          plane_any<RSP, 7>(P, sp, tx, ty, yf, zc, acc, offs);
        }
        if (active && p - 1 >= k0) {  // nodes (i, j, p-1) and (i+1, j, p-1) are complete
          const int so = ring(p - 1);
          const uint32_t oi0 = is[so][ty + 1][IOFF + 2 * tx + 1], oi1 = is[so][ty + 1][IOFF + 2 * tx + 2];
          const double E0 = Es[oi0 >> 3], E1 = Es[oi1 >> 3];
          const int64_t onode = i + (int64_t)NX * (j + (int64_t)NY * (p - 1));
          // own nodes' staged inputs (raw x unless constrained)
          const double* xrow = &xs[so][ty + 1][roff(ty + 1, p - 1) + 3 * (2 * tx + 1)];
          double* yo = y + 3 * onode;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const bool c0 = (oi0 >> a) & 1, c1 = (oi1 >> a) & 1;
            const double x0 = c0 ? (v0 ? __ldg(&x[3 * onode + a]) : 0.0) : xrow[a];
            const double x1 = c1 ? (v1 ? __ldg(&x[3 * onode + 3 + a]) : 0.0) : xrow[3 + a];
            const double y0 = c0 ? x0 : E0 * acc[0][0][a];
            const double y1 = c1 ? x1 : E1 * acc[1][0][a];
            if (v0) yo[a] = y0;
            if (v1) yo[3 + a] = y1;
            if constexpr (DOT) {
              dsum = fma(v0 ? x0 : 0.0, y0, dsum);
              dsum = fma(v1 ? x1 : 0.0, y1, dsum);
            }
          }
        }
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            acc[n][0][a] = acc[n][1][a];
            acc[n][1][a] = acc[n][2][a];
            acc[n][2][a] = 0.0;
          }
      }
#pragma unroll
      for (int q = 0; q < PPB; ++q)
        if (pb + PPB + q <= k1) {
          wait(pb + PPB + q);
          mask(pb + PPB + q);
        }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < PPB; ++q)
        if (pb + RING - 1 + q <= k1) issue(pb + RING - 1 + q);  // into the slots of planes pb - 1 + q
    }
  }
  if constexpr (DOT) {
    const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int nb = gridDim.x * gridDim.y * gridDim.z;
    if (dot.finish) {
      block_to_slot_and_finish(dsum, dot.part_main, bid, nb, nullptr, 0, dot.counter, dot.out);
    } else {
      double a[1] = {dsum};
      block_reduce<1>(a);
      if (threadIdx.x == 0) dot.part_main[bid] = a[0];
    }
  }
}

// Padded info copy for the TMA kernel: row (j, k) of NX bytes at 16 + ipx (j + NY k); every other
// byte is 7 (all three components masked = outside the domain).
__global__ void k_info_pad(const uint8_t* __restrict__ info, uint8_t* __restrict__ out, int NX, int NY, int NZ,
                           int ipx, int64_t total) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q - 16;
    uint8_t v = 7;
    if (r >= 0) {
      const int64_t row = r / ipx;
      const int i = static_cast<int>(r - row * ipx);
      if (i < NX && row < (int64_t)NY * NZ) v = info[i + (int64_t)NX * row];
    }
    out[q] = v;
  }
}

// Correction items: one thread per (node, octant) pair. y_n receives dE * Khat_rows(o) x_e(o) with
// dE = E[octant phase] - E[base phase] (the base of an edge-column node is void, E = 0, and its
// sum is written, not added). Items are ordered tile-major — (64 x 8 x-y tile, plane, node,
// octant) — and every CTA walks one contiguous range of 32-item batches, so the x gathers of a
// CTA stay inside a few planes of one tile and hit L1. Items of a node are contiguous and never
// straddle a batch; the head sums them with fixed-order shuffles and updates y directly.
// Deterministic (fixed batch -> CTA mapping, fixed shuffle order), no atomics, no barriers.
// rec: node (low 32 bits, -1 = padding) | oct << 32 | seg << 35 | edge << 39 | pho << 40 |
// phb << 45 | rem << 50 (items left in the segment, this one included); zm: bit 3b+c = input c of
// the element's bit corner b ^ rm (the item's reflected frame) is zero (Dirichlet or outside).
#ifndef AFEM_ITEM_THREADS
#define AFEM_ITEM_THREADS 256
#endif
#ifndef AFEM_ITEM_MINB
#define AFEM_ITEM_MINB 4  // 32 warps per SM at a 64-register cap: items 32.4 -> 27.6-28.1 us on the same box
#endif
constexpr int kItemThreads = AFEM_ITEM_THREADS;
constexpr uint64_t kPadRec = 0xffffffffull;

struct Items {
  const uint64_t* rec;
  const uint32_t* zm;
  int64_t n;  // multiple of 32
  int kmin = 0, kmax = 1 << 30;  // only the items of nodes on planes [kmin, kmax) (plane-range applies)
};

template <bool DOT>
__global__ void __launch_bounds__(kItemThreads, AFEM_ITEM_MINB) k_stencil_items(int NX, int NY, const __grid_constant__ RowsK0 K0,
                                                                 const double* __restrict__ Epar,
                                                                 const double* __restrict__ x,
                                                                 const uint8_t* __restrict__ info, Items it,
                                                                 double* __restrict__ y, DotArgs dot) {
  if (dot.skip && *dot.skip) return;
  __shared__ double Es[32];
  __shared__ __align__(16) double Ks[3][24];  // every lane reads the same word: broadcasts, 16-byte pairs
  if (threadIdx.x < 32) Es[threadIdx.x] = __ldg(&Epar[threadIdx.x]);
  if (threadIdx.x < 72) Ks[threadIdx.x / 24][threadIdx.x % 24] = K0.k[threadIdx.x / 24][threadIdx.x % 24];
  __syncthreads();
  double dsum = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t nb = it.n >> 5;
  const int64_t blo = nb * blockIdx.x / gridDim.x, bhi = nb * (blockIdx.x + 1) / gridDim.x;
  const int NXY = NX * NY;
  uint64_t nrec = kPadRec;
  uint32_t nzm = 0;
  if (blo + warp < bhi) {
    nrec = __ldg(&it.rec[(blo + warp) * 32 + lane]);
    nzm = __ldg(&it.zm[(blo + warp) * 32 + lane]);
  }
  for (int64_t bt = blo + warp; bt < bhi; bt += nw) {
    uint64_t rec = nrec;
    const uint32_t zm = nzm;
    if (bt + nw < bhi) {  // next batch's record, one batch ahead
      nrec = __ldg(&it.rec[(bt + nw) * 32 + lane]);
      nzm = __ldg(&it.zm[(bt + nw) * 32 + lane]);
    }
    {  // outside the plane range: a pad (a node's items share its plane, so segments stay whole)
      const int nd = static_cast<int>(static_cast<uint32_t>(rec));
      if (nd >= 0 && (nd / NXY < it.kmin || nd / NXY >= it.kmax)) rec = kPadRec;
    }
    const int node = static_cast<int>(static_cast<uint32_t>(rec));
    const uint32_t w = static_cast<uint32_t>(rec >> 32);
    double r0 = 0.0, r1 = 0.0, r2 = 0.0;
    const int L = node >= 0 ? (w >> 3) & 15 : 0;
    const bool edge = (w >> 7) & 1;
    // the head's own node: info, current y and x, loaded before the compute (no other thread of
    // this kernel writes this node's y)
    uint32_t inf = 0;
    double yn[3] = {0.0, 0.0, 0.0}, xn3[3] = {0.0, 0.0, 0.0};
    if (L > 0) {
      inf = __ldg(&info[node]);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (!edge) yn[a] = y[3 * (int64_t)node + a];
        if (DOT || edge) xn3[a] = __ldg(&x[3 * (int64_t)node + a]);
      }
    }
    if (node >= 0) {
      const int rm = (w & 7) ^ 7;  // the node's bit corner in the element (octant o = its mirror)
      // frame corner b lies at +-bit_c(b) along axis c from the node (minus where rm has bit c)
      const int SX = (rm & 1) ? -1 : 1, SY = (rm & 2) ? -NX : NX, SZ = (rm & 4) ? -NXY : NXY;
      // reflected frame: the node sits at bit corner 0; frame corner b is element corner b ^ rm, and
      // component c of x and row c of y flip sign with bit c of rm
      const double s0 = (rm & 1) ? -1.0 : 1.0, s1 = (rm & 2) ? -1.0 : 1.0, s2 = (rm & 4) ? -1.0 : 1.0;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int nd = node + ((b & 1) ? SX : 0) + ((b & 2) ? SY : 0) + ((b & 4) ? SZ : 0);
        const uint32_t zb = (zm >> (3 * b)) & 7;
        const int a0 = zb == 7 ? 0 : 3 * nd;  // all-zero corners (outside) read a safe address
        const int odd = static_cast<int>((reinterpret_cast<uintptr_t>(x + a0) >> 3) & 1);  // 16 B-aligned pair
        const double2 pr = __ldg(reinterpret_cast<const double2*>(x + a0 + odd));
        const double sg = __ldg(x + (odd ? a0 : a0 + 2));
        const double c0 = (zb & 1) ? 0.0 : s0 * (odd ? sg : pr.x);
        const double c1 = (zb & 2) ? 0.0 : s1 * (odd ? pr.x : pr.y);
        const double c2 = (zb & 4) ? 0.0 : s2 * (odd ? pr.y : sg);
        const double cv[3] = {c0, c1, c2};
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          r0 = fma(Ks[0][3 * b + cc], cv[cc], r0);
          r1 = fma(Ks[1][3 * b + cc], cv[cc], r1);
          r2 = fma(Ks[2][3 * b + cc], cv[cc], r2);
        }
      }
      const double dE = Es[(w >> 8) & 31] - Es[(w >> 13) & 31];
      r0 *= s0 * dE;
      r1 *= s1 * dE;
      r2 *= s2 * dE;
    }
    // segmented tree sum: rem = items from this lane to its segment's end (<= 8, never crossing the
    // batch); after the step with offset d every lane holds the sum of [lane, min(lane + 2d, end))
    const int rem = static_cast<int>((rec >> 50) & 15);
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) {
      const double v0 = __shfl_down_sync(0xffffffffu, r0, d);
      const double v1 = __shfl_down_sync(0xffffffffu, r1, d);
      const double v2 = __shfl_down_sync(0xffffffffu, r2, d);
      if (d < rem) {
        r0 += v0;
        r1 += v1;
        r2 += v2;
      }
    }
    if (L > 0) {
      const double rr3[3] = {r0, r1, r2};
      double* yo = y + 3 * (int64_t)node;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const bool con = (inf >> a) & 1;
        if (edge) {  // edge column: the whole row sum, written
          const double ya = con ? xn3[a] : rr3[a];
          yo[a] = ya;
          if constexpr (DOT) dsum = fma(xn3[a], ya, dsum);
        } else if (!con) {
          yo[a] = yn[a] + rr3[a];
          if constexpr (DOT) dsum = fma(xn3[a], rr3[a], dsum);
        }
      }
    }
  }
  if constexpr (DOT)
    block_to_slot_and_finish(dsum, dot.part_items, blockIdx.x, gridDim.x, dot.part_main, dot.n_main, dot.counter,
                             dot.out);
}

// Per node: info byte (Dirichlet bits | base phase << 3) and, for nodes of the main kernel whose
// octant family mixes moduli, a fix entry. Family F(n): octants not void in y or z (those are
// removed exactly by the face coefficients); x-void octants stay in F(n) with E = 0. Base = the
// most frequent phase code in F(n), ties to the smaller code.
__global__ void k_stencil_classify(int NX, int NY, int NZ, int NXm, const uint8_t* __restrict__ phase,
                                   const uint8_t* __restrict__ dof_mask, uint8_t* __restrict__ info,
                                   uint64_t* __restrict__ fix_keys, unsigned long long* __restrict__ n_fix) {
  const int ex = NX - 1, ey = NY - 1, ez = NZ - 1;
  const int64_t total = (int64_t)NX * NY * NZ;
  for (int64_t node = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; node < total;
       node += (int64_t)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(node % NX);
    const int64_t r = node / NX;
    const int j = static_cast<int>(r % NY), k = static_cast<int>(r / NY);
    int ph[8];
    bool fam[8];
    for (int o = 0; o < 8; ++o) {
      const int ei = i - 1 + (o & 1), ej = j - 1 + ((o >> 1) & 1), ek = k - 1 + (o >> 2);
      const bool yz_in = ej >= 0 && ej < ey && ek >= 0 && ek < ez;
      const bool inside = yz_in && ei >= 0 && ei < ex;
      fam[o] = yz_in;
      ph[o] = inside ? phase[ei + (int64_t)ex * (ej + (int64_t)ey * ek)] : kVoid;
    }
    int best = kVoid, bestc = 0;
    for (int o = 0; o < 8; ++o) {
      if (!fam[o] || ph[o] == kVoid) continue;  // base: most frequent existing phase (E_base > 0)
      int c = 0;
      for (int q = 0; q < 8; ++q) c += fam[q] && ph[q] == ph[o];
      if (c > bestc || (c == bestc && ph[o] < best)) {
        best = ph[o];
        bestc = c;
      }
    }
    uint8_t om = 0;
    for (int o = 0; o < 8; ++o)
      if (fam[o] && ph[o] != best) om |= static_cast<uint8_t>(1u << o);
    const uint8_t m = (dof_mask[3 * node] ? 1 : 0) | (dof_mask[3 * node + 1] ? 2 : 0) | (dof_mask[3 * node + 2] ? 4 : 0);
    info[node] = static_cast<uint8_t>(m | (best << 3));
    if (i < NXm && om && m != 7) {
      const unsigned long long slot = atomicAdd(n_fix, 1ull);
      fix_keys[slot] = (static_cast<uint64_t>(om) << 32) | static_cast<uint64_t>(node);
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

// Family stencil from Khat: sum over octants o in the family containing offset d.
void family_stencil(const std::vector<double>& K, int yf, int zf, double out[27][3][3]) {
  for (int d = 0; d < 27; ++d)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) out[d][a][b] = 0.0;
  for (int o = 0; o < 8; ++o) {
    const int ox = o & 1, oy = (o >> 1) & 1, oz = o >> 2;
    if (yf == 1 && oy == 0) continue;  // y lo face: octants below are void
    if (yf == 2 && oy == 1) continue;
    if (zf == 1 && oz == 0) continue;
    if (zf == 2 && oz == 1) continue;
    const int lx = 1 - ox, ly = 1 - oy, lz = 1 - oz;
    const int ln = local_node(lx, ly, lz);
    for (int m = 0; m < 8; ++m) {
      const int mx = corner_x(m), my = corner_y(m), mz = m >> 2;
      const int d = (mx - lx + 1) + 3 * (my - ly + 1) + 9 * (mz - lz + 1);
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) out[d][a][b] += K[(3 * ln + a) * 24 + 3 * m + b];
    }
  }
}

// Snap structural zeros; false if a snapped entry is not negligible (not a symmetric brick grid).
bool snap(double s[27][3][3], int broken) {
  double smax = 0.0;
  for (int d = 0; d < 27; ++d)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) smax = std::max(smax, std::abs(s[d][a][b]));
  for (int d = 0; d < 27; ++d)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        if (szero(d % 3 - 1, (d / 3) % 3 - 1, d / 9 - 1, a, b, broken)) {
          if (std::abs(s[d][a][b]) > 1e-12 * smax) return false;
          s[d][a][b] = 0.0;
        }
  return true;
}

}  // namespace

void encode_map_1d(CUtensorMap* map, const void* base, uint64_t n, CUtensorMapDataType type, uint32_t box) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    AFEM_CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  const cuuint64_t dims[1] = {n};
  const cuuint64_t unused_stride[1] = {16};  // rank 1 has no strides, but the driver rejects a null array
  const cuuint32_t boxd[1] = {box}, estr[1] = {1};
  const CUresult r = enc(map, type, 1, const_cast<void*>(base), dims, unused_stride, boxd, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

// x map of the main kernel for this x (8-byte aligned: the map starts at the 16-byte boundary at or
// below x and element coordinates are shifted by one when x sits 8 bytes above it)
static void stencil_x_map(StencilPlan& pl, const double* x) {
  if (pl.mx_ptr == x) return;
  const uintptr_t a = reinterpret_cast<uintptr_t>(x), b = a & ~uintptr_t(15);
  pl.xshift = static_cast<int>((a - b) / 8);
  const uint64_t n = 3ull * pl.p.NX * pl.p.NY * pl.p.NZ + pl.xshift;
  encode_map_1d(&pl.mx, reinterpret_cast<const void*>(b), n, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, XBOX);
  pl.mx_ptr = x;
}

StencilPlan* make_stencil_plan(System& s, const MfOp& op) {
  if (!s.grid || s.dim != 3) return nullptr;
  if (s.mats.empty() || s.mats.size() >= kVoid) return nullptr;
  const double nu = s.mats[0].nu;
  for (const DMat& m : s.mats)
    if (m.model != MODEL_LINEAR || m.nu != nu) return nullptr;
  if (s.n_nodes > (int64_t)INT32_MAX / 3) return nullptr;
  Ctx& c = *s.ctx;
  auto plan = std::make_unique<StencilPlan>();
  StencilParams& P = plan->p;
  P.NX = s.nx + 1;
  P.NY = s.ny + 1;
  P.NZ = s.nz + 1;
  // A ragged last tile of >= 8 columns runs in the main kernel (masked lanes); narrower remainders
  // go to the correction items as edge columns (a mostly idle 64-wide tile would cost more).
  P.NXm = (P.NX % TXN) >= 8 ? P.NX : (P.NX / TXN) * TXN;
  for (int k = 0; k < 32; ++k) P.E[k] = 0.0;
  for (size_t k = 0; k < s.mats.size(); ++k) P.E[k] = s.mats[k].E;

  // Khat from element 0 at E = 1 (K_e = E * Khat for a common nu: c11, c12, c33 scale with E).
  DevArray<double> dK(576);
  const DMat unit = make_dmat(MODEL_LINEAR, 1.0, nu);
  launch(c, k_brick_stiffness, 1, 32, 0, s.coords.p, s.conn.p, unit, dK.p);
  std::vector<double> K(576);
  AFEM_CK(cudaMemcpyAsync(K.data(), dK.p, 576 * 8, cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  plan->Kg = std::move(dK);
  {
    const int r0 = 3 * local_node(0, 0, 0);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 8; ++b)
        for (int cc = 0; cc < 3; ++cc)
          plan->k0.k[a][3 * b + cc] = K[(r0 + a) * 24 + 3 * local_node(b & 1, (b >> 1) & 1, b >> 2) + cc];
  }
  double fam[27][3][3];
  family_stencil(K, 0, 0, fam);
  if (!snap(fam, 0)) return nullptr;
  // Symmetry-unique interior values; every entry must agree with its representative.
  double smax = 0.0;
  for (int d = 0; d < 27; ++d)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) smax = std::max(smax, std::abs(fam[d][a][b]));
  for (int a = 0; a < 3; ++a)
    for (int ax = 0; ax < 2; ++ax)
      for (int ay = 0; ay < 2; ++ay)
        for (int az = 0; az < 2; ++az) P.Dg[a][ax][ay][az] = fam[(ax + 1) + 3 * (ay + 1) + 9 * (az + 1)][a][a];
  const int pa[3] = {0, 0, 1}, pb[3] = {1, 2, 2};
  for (int q = 0; q < 3; ++q)
    for (int acz = 0; acz < 2; ++acz) {
      int dd[3] = {0, 0, 0};
      dd[pa[q]] = 1;
      dd[pb[q]] = 1;
      dd[3 - pa[q] - pb[q]] = acz;
      P.Og[q][acz] = fam[(dd[0] + 1) + 3 * (dd[1] + 1) + 9 * (dd[2] + 1)][pa[q]][pb[q]];
    }
  for (int d = 0; d < 27; ++d) {
    const int dv[3] = {d % 3 - 1, (d / 3) % 3 - 1, d / 9 - 1};
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double rep;
        if (a == b) {
          rep = P.Dg[a][dv[0] != 0][dv[1] != 0][dv[2] != 0];
        } else if (dv[a] == 0 || dv[b] == 0) {
          rep = 0.0;
        } else {
          const int q = (a + b == 1) ? 0 : (a + b == 2 ? 1 : 2);
          rep = (dv[a] * dv[b] > 0 ? 1.0 : -1.0) * P.Og[q][dv[3 - a - b] != 0];
        }
        if (std::abs(rep - fam[d][a][b]) > 1e-12 * smax) return nullptr;  // not a symmetric brick
      }
  }
  for (int sy = 0; sy < 2; ++sy) {
    family_stencil(K, sy + 1, 0, fam);
    if (!snap(fam, 2)) return nullptr;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dz = -1; dz <= 1; ++dz)
        std::memcpy(P.HY[sy][(dx + 1) + 3 * (dz + 1)], fam[(dx + 1) + 3 * 1 + 9 * (dz + 1)], 9 * 8);
  }
  for (int sz = 0; sz < 2; ++sz) {
    family_stencil(K, 0, sz + 1, fam);
    if (!snap(fam, 4)) return nullptr;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        std::memcpy(P.HZ[sz][(dx + 1) + 3 * (dy + 1)], fam[(dx + 1) + 3 * (dy + 1) + 9 * 1], 9 * 8);
  }
  for (int sy = 0; sy < 2; ++sy)
    for (int sz = 0; sz < 2; ++sz) {
      family_stencil(K, sy + 1, sz + 1, fam);
      if (!snap(fam, 6)) return nullptr;
      for (int dx = -1; dx <= 1; ++dx) std::memcpy(P.HYZ[sy][sz][dx + 1], fam[(dx + 1) + 3 + 9], 9 * 8);
    }

  // z chunks: one full wave of resident CTAs when tiles allow it
  static bool attrs = false;
  if (!attrs) {
    AFEM_CK(cudaFuncSetAttribute(k_stencil_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem));
    AFEM_CK(cudaFuncSetAttribute(k_stencil_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem));
    attrs = true;
  }
  int occ = 1;
  AFEM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stencil_tma<true>, NT, kTmaSmem));
  // one wave of kMainBlocksPerSm CTAs per SM even where 5 would fit (88 registers): 4 measured
  // 2-3 % faster (72.7 vs 74.9 us per C2 apply)
  occ = std::min(occ, kMainBlocksPerSm);
  const int64_t slots = (int64_t)std::max(occ, 1) * c.num_sms;
  const int64_t tiles = (int64_t)((P.NXm + TXN - 1) / TXN) * ((P.NY + TY - 1) / TY);
  int chunks = tiles > 0 ? static_cast<int>(std::max<int64_t>(1, slots / tiles)) : 1;
  chunks = std::min(chunks, std::max(1, P.NZ / 8));
  plan->kchunk = (P.NZ + chunks - 1) / chunks;
  plan->nchunks = (P.NZ + plan->kchunk - 1) / plan->kchunk;
  plan->zpiece = std::max(8, (P.NZ + 7) / 8);  // about 8 pieces
  plan->npieces = (P.NZ + plan->zpiece - 1) / plan->zpiece;
  const int64_t nn = s.n_nodes;
  plan->info.alloc(nn + 4);  // +4: the main kernel copies the aligned 4-byte word holding a node's byte
  AFEM_CK(cudaMemsetAsync(plan->info.p, 0, nn + 4, c.stream));

  DevArray<uint64_t> keys(nn);
  DevArray<unsigned long long> cnt(1);
  AFEM_CK(cudaMemsetAsync(cnt.p, 0, 8, c.stream));
  launch(c, k_stencil_classify, grid_for(nn, 256, 148 * 32), 256, 0, P.NX, P.NY, P.NZ, P.NXm, s.phase.p, op.mask.p,
         plan->info.p, keys.p, cnt.p);
  {
    const int ntiles_x = (P.NXm + TXN - 1) / TXN;
    plan->ipx = ((std::max(ntiles_x * TXN + 1, P.NX + 1) + 15) / 16) * 16;  // >= 1 pad byte after each tile
    const int64_t tot = 16 + (int64_t)plan->ipx * P.NY * P.NZ + 128;       // + the last box's overhang
    plan->info_pad.alloc(tot);
    launch(c, k_info_pad, grid_for(tot, 256, 148 * 16), 256, 0, plan->info.p, plan->info_pad.p, P.NX, P.NY, P.NZ,
           plan->ipx, tot);
    encode_map_1d(&plan->mi, plan->info_pad.p, tot, CU_TENSOR_MAP_DATA_TYPE_UINT8, IBOX);
  }
  unsigned long long nf = 0;
  AFEM_CK(cudaMemcpyAsync(&nf, cnt.p, 8, cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  {
    // Correction items, built on the host once per operator: (node, octant, dE) for every octant of
    // a mixed-family node whose modulus differs from the node's base, and for every existing octant
    // of the edge-column nodes (base 0, written). Node order; a node's items never cross a warp.
    std::vector<uint64_t> hk(nf);
    if (nf) AFEM_CK(cudaMemcpyAsync(hk.data(), keys.p, nf * 8, cudaMemcpyDeviceToHost, c.stream));
    std::vector<uint8_t> hph(s.n_elem), hinfo(nn);
    AFEM_CK(cudaMemcpyAsync(hph.data(), s.phase.p, s.n_elem, cudaMemcpyDeviceToHost, c.stream));
    AFEM_CK(cudaMemcpyAsync(hinfo.data(), plan->info.p, nn, cudaMemcpyDeviceToHost, c.stream));
    AFEM_CK(cudaStreamSynchronize(c.stream));
    struct NodeMask { int64_t node; uint8_t mask; bool edge; };
    std::vector<NodeMask> list;
    list.reserve(nf + (size_t)(P.NX - P.NXm) * P.NY * P.NZ);
    for (uint64_t k : hk) list.push_back({static_cast<int64_t>(k & 0xffffffffu), static_cast<uint8_t>(k >> 32), false});
    const int ex = P.NX - 1, ey = P.NY - 1, ez = P.NZ - 1;
    auto oct_phase = [&](int64_t node, int o) -> int {
      const int i = static_cast<int>(node % P.NX);
      const int64_t r = node / P.NX;
      const int j = static_cast<int>(r % P.NY), k = static_cast<int>(r / P.NY);
      const int ei = i - 1 + (o & 1), ej = j - 1 + ((o >> 1) & 1), ek = k - 1 + (o >> 2);
      const bool inside = ei >= 0 && ei < ex && ej >= 0 && ej < ey && ek >= 0 && ek < ez;
      return inside ? hph[ei + (int64_t)ex * (ej + (int64_t)ey * ek)] : kVoid;
    };
    for (int k = 0; k < P.NZ; ++k)
      for (int j = 0; j < P.NY; ++j)
        for (int i = P.NXm; i < P.NX; ++i) {
          const int64_t node = i + (int64_t)P.NX * (j + (int64_t)P.NY * k);
          uint8_t m = 0;
          for (int o = 0; o < 8; ++o)
            if (oct_phase(node, o) != kVoid) m |= static_cast<uint8_t>(1u << o);
          list.push_back({node, m, true});
        }
    std::sort(list.begin(), list.end(), [](const NodeMask& a, const NodeMask& b) { return a.node < b.node; });

    for (const NodeMask& nm : list) (nm.edge ? plan->n_edge_nodes : plan->n_fix_nodes) += 1;

    // k_stencil_items: every item of a mixed-family node (and of the edge columns, unless the
    // in-tile variant writes them), ordered (x tile, y tile, plane, node, octant); padded so that no
    // node's items straddle a 32-item batch.
    const int ntyc = (P.NY + TY - 1) / TY;
    struct TItem { uint32_t piece; uint64_t key; uint64_t rec; uint32_t zm; };
    std::vector<TItem> ti;
    for (const NodeMask& nm : list) {
      const int ni = static_cast<int>(nm.node % P.NX);
      const int64_t nr = nm.node / P.NX;
      const int nj = static_cast<int>(nr % P.NY), nk = static_cast<int>(nr / P.NY);
      const uint64_t lid = ((uint64_t)(ni / TXN) * ntyc + nj / TY) * P.NZ + nk;
      const uint64_t phb = nm.edge ? static_cast<uint64_t>(kVoid) : static_cast<uint64_t>(hinfo[nm.node] >> 3);
      for (int o = 0; o < 8; ++o) {
        if (!((nm.mask >> o) & 1)) continue;
        const uint64_t pho = static_cast<uint64_t>(oct_phase(nm.node, o));
        const uint64_t rec = static_cast<uint64_t>(static_cast<uint32_t>(nm.node)) |
                             (static_cast<uint64_t>(o) << 32) | ((nm.edge ? 1ull : 0ull) << 39) | (pho << 40) |
                             (phb << 45);
        // zero inputs (Dirichlet, or outside the domain) in the item kernel's reflected frame: bits
        // 3b..3b+2 belong to frame corner b = element bit corner b ^ rm, rm = the node's bit corner
        uint32_t zm = 0;
        const int ei = ni - 1 + (o & 1), ej = nj - 1 + ((o >> 1) & 1), ek = nk - 1 + (o >> 2);
        const int rm = o ^ 7;
        for (int b = 0; b < 8; ++b) {
          const int pb = b ^ rm;
          const int ii = ei + (pb & 1), jj = ej + ((pb >> 1) & 1), kk = ek + (pb >> 2);
          const bool in = ii >= 0 && ii < P.NX && jj >= 0 && jj < P.NY && kk >= 0 && kk < P.NZ;
          zm |= (in ? (hinfo[ii + (int64_t)P.NX * (jj + (int64_t)P.NY * kk)] & 7u) : 7u) << (3 * b);
        }
        ti.push_back({static_cast<uint32_t>(nk / plan->zpiece),
                      (lid << 36) | ((uint64_t)(nj % TY) * TXN + ni % TXN) << 3 | static_cast<uint64_t>(o), rec, zm});
      }
    }
    std::sort(ti.begin(), ti.end(), [](const TItem& a, const TItem& b) {
      return a.piece != b.piece ? a.piece < b.piece : a.key < b.key;
    });
    std::vector<uint64_t> trec;
    std::vector<uint32_t> tzm;
    plan->piece_items.assign(1, 0);
    for (size_t q2 = 0; q2 < ti.size();) {
      while (static_cast<int>(plan->piece_items.size()) <= static_cast<int>(ti[q2].piece)) {
        while (trec.size() % 32) {  // a piece starts on a batch boundary
          trec.push_back(kPadRec);
          tzm.push_back(0);
        }
        plan->piece_items.push_back(static_cast<int64_t>(trec.size()));
      }
      size_t e = q2;  // segment: one target node
      while (e < ti.size() && static_cast<uint32_t>(ti[e].rec) == static_cast<uint32_t>(ti[q2].rec)) ++e;
      const uint64_t L = e - q2;
      if ((trec.size() % 32) + L > 32)
        while (trec.size() % 32) {
          trec.push_back(kPadRec);
          tzm.push_back(0);
        }
      for (size_t t = q2; t < e; ++t) {
        trec.push_back(ti[t].rec | (t == q2 ? (L << 35) : 0ull) | (static_cast<uint64_t>(e - t) << 50));
        tzm.push_back(ti[t].zm);
      }
      q2 = e;
    }
    while (trec.size() % 32) {
      trec.push_back(kPadRec);
      tzm.push_back(0);
    }
    plan->n_items = static_cast<int64_t>(trec.size());
    while (static_cast<int>(plan->piece_items.size()) <= plan->npieces) plan->piece_items.push_back(plan->n_items);
    plan->it_rec.alloc(std::max<size_t>(trec.size(), 1));
    plan->it_zm.alloc(std::max<size_t>(tzm.size(), 1));
    if (!trec.empty()) {
      AFEM_CK(cudaMemcpyAsync(plan->it_rec.p, trec.data(), trec.size() * 8, cudaMemcpyHostToDevice, c.stream));
      AFEM_CK(cudaMemcpyAsync(plan->it_zm.p, tzm.data(), tzm.size() * 4, cudaMemcpyHostToDevice, c.stream));
    }
    AFEM_CK(cudaStreamSynchronize(c.stream));
  }
  // balanced main grid: one resident wave, no more CTAs than (tile, plane) units
  const int64_t units = (int64_t)((P.NXm + TXN - 1) / TXN) * ((P.NY + TY - 1) / TY) * P.NZ;
  plan->main_blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(slots, units)));
  if (const char* e = std::getenv("AFEM_MAIN_BLOCKS")) plan->main_blocks = std::max(1, std::atoi(e));
  plan->part_main.alloc(std::max<int64_t>(plan->main_blocks, 1));
  int iocc = 1;  // one wave of resident item CTAs, each walking one contiguous range
  AFEM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&iocc, k_stencil_items<true>, kItemThreads, 0));
  plan->iocc = std::max(iocc, 1);
  plan->item_blocks = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(plan->n_items / 256, (int64_t)std::max(iocc, 1) * c.num_sms)));
  plan->part_items.alloc(plan->item_blocks);
  plan->Ed.alloc(32);
  AFEM_CK(cudaMemcpyAsync(plan->Ed.p, P.E, 32 * 8, cudaMemcpyHostToDevice, c.stream));
  plan->counter.alloc(1);
  AFEM_CK(cudaMemsetAsync(plan->counter.p, 0, sizeof(unsigned), c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  return plan.release();
}

static void stencil_apply_launch(StencilPlan& pl, const MfOp& op, const double* x, double* y, double* dot_out,
                                 const int* skip);

void stencil_apply(StencilPlan& pl, const MfOp& op, const double* x, double* y, double* dot_out, const int* skip) {
  Ctx& c = *op.sys->ctx;
  static const bool no_graph = std::getenv("AFEM_NO_APPLY_GRAPH") != nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (!dot_out && !skip && !no_graph) AFEM_CK(cudaStreamIsCapturing(c.stream, &cs));
  if (dot_out || skip || no_graph || cs != cudaStreamCaptureStatusNone) {
    stencil_apply_launch(pl, op, x, y, dot_out, skip);
    return;
  }
  StencilPlan::GraphSlot* slot = nullptr;
  for (auto& g : pl.graphs)
    if (g.used && g.x == x && g.y == y) slot = &g;
  if (!slot) {  // first use of this pair: direct launches, remember the pair (least recently used slot)
    slot = &pl.graphs[0];
    for (auto& g : pl.graphs)
      if (g.used < slot->used) slot = &g;
    if (slot->exec) cudaGraphExecDestroy(slot->exec);
    *slot = StencilPlan::GraphSlot{x, y, nullptr, ++pl.graph_clock};
    stencil_apply_launch(pl, op, x, y, nullptr, nullptr);
    return;
  }
  slot->used = ++pl.graph_clock;
  if (!slot->exec) {  // second use: capture on the context's private stream
    cudaGraph_t g = nullptr;
    {
      CaptureGuard cap(c);
      stencil_apply_launch(pl, op, x, y, nullptr, nullptr);
      g = cap.end();
    }
    ScopeExit free_graph([&] { cudaGraphDestroy(g); });
    AFEM_CK(cudaGraphInstantiate(&slot->exec, g, 0));
  }
  AFEM_CK(cudaGraphLaunch(slot->exec, c.stream));
  c.launches += (pl.p.NXm > 0 ? 1 : 0) + (pl.n_items > 0 ? 1 : 0);
}

static void stencil_apply_launch(StencilPlan& pl, const MfOp& op, const double* x, double* y, double* dot_out,
                                 const int* skip) {
  Ctx& c = *op.sys->ctx;
  const StencilParams& P = pl.p;
  const int ntx = (P.NXm + TXN - 1) / TXN, nty = (P.NY + TY - 1) / TY;
  const int nb_main = P.NXm > 0 ? pl.main_blocks : 0;
  const DotArgs dot{pl.part_main.p, pl.part_items.p, pl.counter.p, dot_out, pl.n_items == 0 ? 1 : 0, nb_main, skip};
  // measurement switch (scripts only): AFEM_STENCIL_ONLY=main|items launches one of the two kernels
  static const char* only = std::getenv("AFEM_STENCIL_ONLY");
  const bool run_main = !only || only[0] == 'm', run_items = !only || only[0] == 'i';
  if (P.NXm > 0 && run_main) {  // balanced single wave (kchunk 0)
    stencil_x_map(pl, x);
    if (dot_out)
      launch(c, k_stencil_tma<true>, nb_main, NT, kTmaSmem, pl.mx, pl.mi, P, pl.xshift, pl.ipx, x, y, 0, 0, P.NZ, dot,
             ntx, nty);
    else
      launch(c, k_stencil_tma<false>, nb_main, NT, kTmaSmem, pl.mx, pl.mi, P, pl.xshift, pl.ipx, x, y, 0, 0, P.NZ, dot,
             ntx, nty);
  }
  if (pl.n_items > 0 && run_items) {
    const Items it{pl.it_rec.p, pl.it_zm.p, pl.n_items};
    if (dot_out)
      launch(c, k_stencil_items<true>, pl.item_blocks, kItemThreads, 0, P.NX, P.NY, pl.k0, pl.Ed.p, x, pl.info.p,
             it, y, dot);
    else
      launch(c, k_stencil_items<false>, pl.item_blocks, kItemThreads, 0, P.NX, P.NY, pl.k0, pl.Ed.p, x, pl.info.p,
             it, y, dot);
  }
}

int stencil_pieces(const StencilPlan& pl) { return pl.npieces; }
int stencil_piece_planes(const StencilPlan& pl) { return pl.zpiece; }

// y over the node planes of z pieces [pa, pb): reads x planes [pa*zpiece - 1, pb*zpiece], writes
// only y of those planes (bitwise identical to the full apply: same per-node arithmetic order).
void stencil_apply_pieces(StencilPlan& pl, const MfOp& op, const double* x, double* y, int pa, int pb) {
  Ctx& c = *op.sys->ctx;
  const StencilParams& P = pl.p;
  const int kb = pa * pl.zpiece, ke = std::min(pb * pl.zpiece, P.NZ);
  if (kb >= ke) return;
  const DotArgs dot{nullptr, nullptr, nullptr, nullptr, 0, 0, nullptr};
  if (P.NXm > 0) {
    const int ntx = (P.NXm + TXN - 1) / TXN, nty = (P.NY + TY - 1) / TY;
    const int64_t units = (int64_t)ntx * nty * (ke - kb);
    stencil_x_map(pl, x);
    static const bool chunked = std::getenv("AFEM_PIECES_CHUNKED") != nullptr;  // A/B switch
    if (!chunked && units >= 8 * (int64_t)pl.main_blocks) {  // a long z range (the slab interior): one balanced wave
      launch(c, k_stencil_tma<false>, pl.main_blocks, NT, kTmaSmem, pl.mx, pl.mi, P, pl.xshift, pl.ipx, x, y, 0, kb,
             ke, dot, ntx, nty);
    } else {  // a piece is a few planes: smaller z chunks so the launch still fills the GPU
      const int tiles = ntx * nty;
      const int want = std::max(1, kMainBlocksPerSm * c.num_sms / std::max(tiles, 1));
      const int kc = std::max(4, (ke - kb + want - 1) / want);
      const dim3 grid(ntx, nty, (ke - kb + kc - 1) / kc);
      launch(c, k_stencil_tma<false>, grid, NT, kTmaSmem, pl.mx, pl.mi, P, pl.xshift, pl.ipx, x, y, kc, kb, ke, dot, 0,
             0);
    }
  }
  const int64_t i0 = pl.piece_items[pa], i1 = pl.piece_items[pb];
  if (i1 > i0) {
    const Items it{pl.it_rec.p + i0, pl.it_zm.p + i0, i1 - i0};
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((i1 - i0) / 256, (int64_t)pl.iocc * c.num_sms)));
    launch(c, k_stencil_items<false>, blocks, kItemThreads, 0, P.NX, P.NY, pl.k0, pl.Ed.p, x, pl.info.p, it, y, dot);
  }
}

// y over node planes [kb, ke) only (main kernel balanced over the range's units, the items of
// those planes), on the context's current stream: the slab operator's boundary / interior split.
// dot_out: also x.y over the range's rows (fixed-order, the plan's partials: one such launch in
// flight per plan); skip: the CG loop's device done flag.
void stencil_apply_planes(StencilPlan& pl, const MfOp& op, const double* x, double* y, int kb, int ke,
                          double* dot_out, const int* skip) {
  Ctx& c = *op.sys->ctx;
  const StencilParams& P = pl.p;
  ke = std::min(ke, P.NZ);
  const int pa = kb / pl.zpiece, pb = std::min(pl.npieces, (ke + pl.zpiece - 1) / pl.zpiece);
  const int64_t i0 = kb < ke ? pl.piece_items[pa] : 0, i1 = kb < ke ? pl.piece_items[pb] : 0;
  const int ntx = (P.NXm + TXN - 1) / TXN, nty = (P.NY + TY - 1) / TY;
  const int64_t units = (int64_t)ntx * nty * std::max(0, ke - kb);
  const int mblocks = P.NXm > 0 ? static_cast<int>(std::min<int64_t>(pl.main_blocks, units)) : 0;
  const bool items = i1 > i0;
  if (dot_out && mblocks == 0 && !items) AFEM_CK(cudaMemsetAsync(dot_out, 0, sizeof(double), c.stream));
  if (kb >= ke) return;
  const DotArgs dot{pl.part_main.p, pl.part_items.p, pl.counter.p, dot_out, items ? 0 : 1, mblocks, skip};
  if (mblocks > 0) {
    stencil_x_map(pl, x);
    if (dot_out)
      launch(c, k_stencil_tma<true>, mblocks, NT, kTmaSmem, pl.mx, pl.mi, P, pl.xshift, pl.ipx, x, y, 0, kb, ke, dot,
             ntx, nty);
    else
      launch(c, k_stencil_tma<false>, mblocks, NT, kTmaSmem, pl.mx, pl.mi, P, pl.xshift, pl.ipx, x, y, 0, kb, ke, dot,
             ntx, nty);
  }
  if (items) {
    Items it{pl.it_rec.p + i0, pl.it_zm.p + i0, i1 - i0};
    it.kmin = kb;
    it.kmax = ke;
    const int blocks =
        static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((i1 - i0) / 256, (int64_t)pl.iocc * c.num_sms)));
    if (dot_out)
      launch(c, k_stencil_items<true>, blocks, kItemThreads, 0, P.NX, P.NY, pl.k0, pl.Ed.p, x, pl.info.p, it, y, dot);
    else
      launch(c, k_stencil_items<false>, blocks, kItemThreads, 0, P.NX, P.NY, pl.k0, pl.Ed.p, x, pl.info.p, it, y, dot);
  }
}

void destroy_stencil_plan(StencilPlan* p) { delete p; }

}  // namespace afem
