// Internal object model of libafem_b200 (not part of the ABI).
//
// HBM layout of a system (DESIGN.md §Data layout):
//   coords   n_nodes*dim  f64   nodal coordinates (AoS, like the dofs)
//   conn     n_elem*npe   i32   element connectivity (mesh order)
//   phase    n_elem       u8    phase label -> material table (<= kMaxMat)
//   inc_ptr  n_nodes+1    i64   node -> incident (element, local node) pairs, in the reference's
//   inc      n_elem*npe   u32   (batch, element) order = (phase, element id)  (assembly.hpp:125)
//   adj_ptr  n_nodes+1    i64   node adjacency = the CSR pattern at node granularity; the dof-level
//   adj      sum deg      i32   pattern (sparse.hpp:68-75) is its dim x dim expansion (never stored)
//   mask     n_dof        u8    Dirichlet constraint table (assembly.hpp:192-211)
//   presc    n_dof        f64
// CSR values (pattern order) are n_dof rows of dim*deg(node) entries each; row_ptr is closed-form.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "element.cuh"

namespace afem {

struct Constraint {
  int node, comp;
  double value;
};

// Kernel-side view of a system (plain pointers).
struct SysView {
  int dim, npe;
  int64_t n_nodes, n_elem, n_dof;
  const double* coords;
  const int32_t* conn;
  const uint8_t* phase;
  const DMat* mats;
  const int64_t* inc_ptr;
  const uint32_t* inc;
  const int64_t* adj_ptr;
  const int32_t* adj;
  const uint8_t* mask;
  const double* presc;
  int* err;
  const double* hist;  // committed quadrature-point history (J2), n_elem*nq*kHist, or null
};

struct StencilPlan;  // structured fast path (stencil.cu)
struct IluLevels;    // ILU(0) dependency levels of a pattern (ilu.cu)

struct System {
  Ctx* ctx = nullptr;
  int dim = 2, npe = 4;
  int64_t n_nodes = 0, n_elem = 0, n_dof = 0, nnz = 0, adj_total = 0;
  DevArray<double> coords;
  DevArray<int32_t> conn;
  DevArray<uint8_t> phase;
  std::vector<DMat> mats;
  DevArray<DMat> d_mats;
  std::vector<int64_t> phase_count;  // elements per phase (batches = non-empty phases)
  DevArray<int32_t> elem_order;      // element ids in (phase, id) order
  DevArray<int64_t> inc_ptr;
  DevArray<uint32_t> inc;
  DevArray<int64_t> adj_ptr;
  DevArray<int32_t> adj;
  DevArray<uint8_t> mask;
  DevArray<double> presc;
  std::vector<Constraint> constraints;
  DevArray<int> err;
  // committed quadrature-point history (allocated, zeroed, when any phase is J2): element-major,
  // nq slots of kHist doubles (DESIGN.md §Data layout). Stays resident across Newton iterations
  // and load steps; history_commit advances it from a converged state.
  DevArray<double> hist;
  bool has_history() const { return hist.p != nullptr; }
  // structured grids: uniform-brick Gauss-point geometry (g_i(q), w detJ(q)) and the element-vector
  // scratch of the element-centric kernels (elemgrid.cu), allocated on first use
  std::vector<double> grid_geo;
  DevArray<double> ev;
  DevArray<double> kscr;  // element tangent blocks of one z slab (elemgrid.cu grid_jacobian)
  std::shared_ptr<IluLevels> ilu_levels;  // built on the first ILU(0) setup
  // structured grid metadata (afem_system_create_grid)
  bool grid = false;
  int nx = 0, ny = 0, nz = 0;
  double lx = 0, ly = 0, lz = 0;

  SysView view() const {
    return SysView{dim, npe, n_nodes, n_elem, n_dof, coords.p, conn.p, phase.p, d_mats.p, inc_ptr.p, inc.p,
                   adj_ptr.p, adj.p, mask.p, presc.p, err.p, hist.p};
  }
  int64_t device_bytes() const {
    return coords.bytes() + conn.bytes() + phase.bytes() + elem_order.bytes() + inc_ptr.bytes() + inc.bytes() +
           adj_ptr.bytes() + adj.bytes() + mask.bytes() + presc.bytes() + hist.bytes() + ev.bytes();
  }
};

struct Values {
  System* sys = nullptr;
  DevArray<double> v;
};

struct Buffer {
  System* sys = nullptr;
  DevArray<double> store;
  int state = 0;  // 0 OwnedByAssembly, 1 LeasedToSolver
  uint64_t epoch = 0;
};

struct Operator {
  virtual ~Operator() = default;
  System* sys = nullptr;
  int kind = 0;  // 0 EXPLICIT, 1 MATRIX_FREE
  int64_t n = 0;
  virtual void validate() const {}
  virtual void apply(const double* x, double* y) = 0;  // device pointers, ctx stream, async
  // y = A x and dot_out[0] = x.y in one pass (deterministic); false if the operator cannot fuse.
  virtual bool apply_dot(const double*, double*, double*) { return false; }
  virtual void diagonal(double* d) = 0;                 // device pointer
  virtual bool uses_stencil() const { return false; }
  // pattern-ordered CSR values when the operator is the assembled matrix (persistent small-n CG)
  virtual const double* csr_values() const { return nullptr; }
  // device flag: while *flag != 0 the apply returns at once (the CG loop's speculative chunk after
  // convergence); false when the operator cannot skip
  virtual bool set_skip(const int*) { return false; }
  // Inner products of the Krylov methods (GMRES, BiCGStab): the whole vector here; a distributed
  // operator sums its owned dofs and allreduces (dist.cu).
  virtual double inner(const double* a, const double* b);
  virtual void inner_dev(const double* a, const double* b, double* out_dev);
  // first row of the owned range the inner products run over, and the sum of device scalars
  // across ranks (the fused GMRES passes); a single-domain operator owns every row
  virtual int64_t dot_begin() const { return 0; }
  virtual void allreduce_dev(double*, int) {}
  // ||b - A x||; keeps r = b - A x when r is given
  virtual double resid(const double* b, const double* x, double* scratch, double* r);
};

struct ExplicitOp : Operator {
  const Buffer* buf = nullptr;
  uint64_t epoch = 0;
  void validate() const override;
  void apply(const double* x, double* y) override;
  void diagonal(double* d) override;
  const double* csr_values() const override { return buf->store.p; }
  const int* skip = nullptr;
  bool set_skip(const int* flag) override {
    skip = flag;
    return true;
  }
};

struct MfOp : Operator {
  DevArray<double> state, diag;
  DevArray<double> qpt;  // cached Gauss-point tangents (J2 grids), elemgrid.cu
  DevArray<uint8_t> mask;
  StencilPlan* stencil = nullptr;  // owned; released by destroy_stencil_plan
  ~MfOp() override;
  void apply(const double* x, double* y) override;
  bool apply_dot(const double* x, double* y, double* dot_out) override;
  void diagonal(double* d) override;
  bool uses_stencil() const override { return stencil != nullptr; }
  const int* skip = nullptr;
  bool set_skip(const int* flag) override {
    skip = flag;
    return stencil != nullptr || qpt.p != nullptr;
  }
};

// ---- system.cu
std::unique_ptr<System> make_system(Ctx& c, int dim, int64_t n_nodes, int64_t n_elem, const double* d_coords,
                                    const int32_t* d_conn, const int32_t* d_phase, const std::vector<DMat>& mats);
std::unique_ptr<System> make_grid_system(Ctx& c, int dim, int nx, int ny, int nz, double lx, double ly, double lz,
                                         const std::vector<double>& incl_xy, double radius,
                                         const std::vector<DMat>& mats);
void set_dirichlet(System& s, const std::vector<Constraint>& cs);
std::vector<Constraint> benchmark_bcs(const System& s, double strain);
void pattern_export(System& s, int64_t* d_row_ptr, int32_t* d_rows, int32_t* d_cols);
void batch_export(System& s, int b, int64_t* size, int32_t* h_ids, int32_t* h_dof_map);
void check_err(System& s);
DMat make_dmat(int model, double E, double nu, double sigma_y = 0.0, double hardening = 0.0);
// J2 history: commit the return-mapped state at u; reset to virgin.
void history_commit(System& s, const double* u);
void history_reset(System& s);

// ---- assembly.cu
void residual(System& s, const double* u, double* r);
void jacobian(System& s, const double* u, double* values);
void diagonal(System& s, const double* u, double* d);
void mf_apply_general(System& s, const double* state, const uint8_t* mask, const double* x, double* y);
void eliminate(System& s, double* values, double* residual, const double* u);
void constrain_residual(System& s, double* residual, const double* u);
void csr_apply(System& s, const double* values, const double* x, double* y, const int* skip = nullptr);
void csr_diagonal(System& s, const double* values, double* d);
void impose_dirichlet(System& s, double* u);

// ---- elemgrid.cu (structured grids: element-centric evaluation + ordered node gather)
void grid_geometry(System& s);
bool grid_elem_path(const System& s);
void grid_residual(System& s, const double* u, double* r);
void grid_diagonal(System& s, const double* u, double* d);
void grid_jacobian(System& s, const double* u, double* values);
void grid_history_commit(System& s, const double* u);  // 3D grids
void grid_mf_apply(System& s, const double* state, const uint8_t* mask, const double* x, double* y,
                   double* dot_out = nullptr);
bool grid_tangent_cacheable(const System& s);
void grid_tangent_cache(System& s, const double* u, DevArray<double>& qpt);
void grid_mf_apply_cached(System& s, const double* qpt, const uint8_t* mask, const double* x, double* y,
                          const int* skip = nullptr, double* dot_out = nullptr);

// ---- blas.cu (deterministic reductions; results in device scalars or host)
double dot(Ctx& c, const double* x, const double* y, int64_t n);
double free_norm(Ctx& c, const double* r, const uint8_t* mask, int64_t n);
void axpy(Ctx& c, double a, const double* x, double* y, int64_t n);
void copy(Ctx& c, const double* x, double* y, int64_t n);
void fill(Ctx& c, double v, double* y, int64_t n);
void add_scaled_dev(Ctx& c, const double* alpha_dev, double scale, const double* x, double* y, int64_t n);
void dot_dev(Ctx& c, const double* x, const double* y, int64_t n, double* out_dev);

// ---- krylov.cu
struct SolverCfg {
  int method = 0, precond = 0;
  double rtol = 1e-13;
  int max_iter = 10000, restart = 30;
};
struct SolveReport {
  bool converged = false;
  int iterations = 0;
  std::vector<double> history;
  double wall_time = 0.0;
  std::string failure;
};
void validate_cfg(const SolverCfg& c);
void solve(Operator& op, const SolverCfg& cfg, const double* b, const double* x0, double* x, SolveReport& rep);

// ---- ilu.cu (Ilu0Preconditioner, krylov.hpp:116-192)
struct Ilu0 {
  System* s = nullptr;
  DevArray<double> f;  // L (strict lower, unit diagonal implied) and U in the pattern's slots
  void setup(System& sys, const double* values);  // FactorizationError on a zero pivot
  void apply(const double* r, double* z) const;   // z = U^-1 L^-1 r
};

// ---- direct.cu (BandedFactorization, krylov.hpp:196-307): false + failure text on breakdown
bool direct_solve(System& s, const double* vals, bool chol, const double* b, double* x, std::string& failure);

// ---- csrop.cu (caller-supplied CSR: the drop-in overlay's explicit operator)
std::unique_ptr<Operator> make_csr_op(Ctx& c, int64_t n, int64_t nnz, const int32_t* h_row_ptr,
                                      const int32_t* h_cols);
double* csr_op_values(Operator& o, int64_t* nnz);  // device values of a make_csr_op operator
void eliminate_csr(Ctx& c, int64_t n, const int32_t* row_ptr, const int32_t* cols, double* values, double* residual,
                   const uint8_t* constrained, const double* prescribed, const double* u);
void constrain_masked(Ctx& c, int64_t n, double* residual, const uint8_t* constrained, const double* prescribed,
                      const double* u);

// ---- stencil.cu
StencilPlan* make_stencil_plan(System& s, const MfOp& op);  // nullptr when not applicable
void stencil_apply(StencilPlan& p, const MfOp& op, const double* x, double* y, double* dot_out = nullptr,
                   const int* skip = nullptr);
int stencil_pieces(const StencilPlan& p);
int stencil_piece_planes(const StencilPlan& p);
void stencil_apply_pieces(StencilPlan& p, const MfOp& op, const double* x, double* y, int pa, int pb);
void stencil_apply_planes(StencilPlan& p, const MfOp& op, const double* x, double* y, int kb, int ke,
                          double* dot_out = nullptr, const int* skip = nullptr);
void destroy_stencil_plan(StencilPlan* p);

}  // namespace afem
