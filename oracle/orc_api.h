/* TEST INFRASTRUCTURE ONLY — the parity oracle's C ABI.
 *
 * Two shared libraries export exactly this interface:
 *   oracle/liboracle.so            CPU restatement (oracle/restate.hpp) of the reference algorithm,
 *                                  2D quad4 + 3D hex8 (the hex8 twin is "parity pinned by restatement",
 *                                  see DESIGN.md §Oracle).
 *   oracle/_ref/libadfem_ref.so    the UNMODIFIED reference headers (/root/reference/proj/include)
 *                                  compiled in place by oracle/Makefile; 2D only (the reference has no 3D).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load
 * these libraries. The product (paper_2604_22087_b200/) never links or calls them.
 *
 * Status codes match include/afem.h (AFEM_OK = 0 ...), one per reference exception type
 * (reference errors.hpp:10-38 + std exceptions).
 */
#ifndef ORC_API_H
#define ORC_API_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_E_INVALID_ARGUMENT = 1,
  ORC_E_OUT_OF_RANGE = 2,
  ORC_E_LOGIC = 3,
  ORC_E_DOMAIN = 4,
  ORC_E_LEASE = 5,
  ORC_E_STALE_EPOCH = 6,
  ORC_E_CAPABILITY = 7,
  ORC_E_FACTORIZATION = 8,
  ORC_E_INVERTED_ELEMENT = 9,
  ORC_E_RUNTIME = 13
};

/* model: 0 linear elastic (plane strain in 2D), 1 St Venant-Kirchhoff (reference material.hpp:13);
 * restatement only (the reference has neither): 2 Neo-Hookean, 3 J2 plasticity (sigma_y, hardening). */
typedef struct {
  int32_t model;
  double E;
  double nu;
  double sigma_y;   /* J2 */
  double hardening; /* J2 */
} orc_material;

/* method: 0 CG, 1 GMRES, 2 BICGSTAB; precond: 0 NONE, 1 JACOBI (reference krylov.hpp:20-21, 43-55) */
typedef struct {
  int32_t method;
  int32_t precond;
  double rtol;
  int32_t max_iter;
  int32_t restart;
} orc_solver_cfg;

typedef struct {
  int32_t converged;
  int32_t iterations;
  int32_t n_history; /* full history length (may exceed the caller's capacity) */
  double wall_time;
  char failure[256];
} orc_solve_report;

/* operator_kind: 0 EXPLICIT, 1 MATRIX_FREE (reference backend.hpp:20) */
typedef struct {
  double rtol;
  double atol;
  int32_t max_iter;
  int32_t operator_kind;
  orc_solver_cfg linear;
} orc_newton_cfg;

typedef struct {
  int32_t converged;
  int32_t iterations;
  int32_t total_linear_iterations;
  int32_t n_norms;
  double total_time;
  char failure[256];
} orc_newton_report;

const char* orc_last_error(void);
int32_t orc_dims_supported(void); /* bitmask: 1<<2 for 2D, 1<<3 for 3D */

/* ---- meshes and boundary conditions (reference mesh.hpp:47-101) ---- */
/* 2D: generate_two_phase_mesh. Outputs sized (nx+1)(ny+1)*2, nx*ny*4, nx*ny. */
int32_t orc_mesh2d(int32_t nx, int32_t ny, double lx, double ly, double cx, double cy,
                   double radius, double* coords, int32_t* conn, int32_t* phase);
/* 3D fibre RVE (hex8 twin). fibres: n_fibres*(x,y) centres. */
int32_t orc_mesh3d(int32_t nx, int32_t ny, int32_t nz, double lx, double ly, double lz,
                   int32_t n_fibres, const double* fibres, double radius, double* coords,
                   int32_t* conn, int32_t* phase);
/* Fibre centres U(0,lx)xU(0,ly) from mt19937_64(seed). */
int32_t orc_fibres(uint64_t seed, int32_t n_fibres, double lx, double ly, double* out);
/* benchmark_bcs: returns count when node==NULL. */
int64_t orc_bcs(int32_t dim, int32_t nx, int32_t ny, int32_t nz, double lx, double strain,
                int32_t* node, int32_t* comp, double* value);

/* ---- system handle: mesh + batches + pattern + Dirichlet table ---- */
void* orc_system_create(int32_t dim, int64_t n_nodes, int64_t n_elem, const double* coords,
                        const int32_t* conn, const int32_t* phase, int32_t n_mat,
                        const orc_material* mats);
/* Same, without the sparsity pattern (sort of 576 pairs/element is infeasible at 128^3): only the
 * residual / matrix-free entry points are valid. Used for bench.py's CPU baseline. */
void* orc_system_create_lite(int32_t dim, int64_t n_nodes, int64_t n_elem, const double* coords,
                             const int32_t* conn, const int32_t* phase, int32_t n_mat,
                             const orc_material* mats);
/* structured-grid metadata so benchmark_bcs / load_stepping can regenerate loads */
int32_t orc_system_set_grid(void* sys, int32_t nx, int32_t ny, int32_t nz, double lx, double ly,
                            double lz);
void orc_system_destroy(void* sys);
int64_t orc_n_dof(void* sys);
int32_t orc_n_batches(void* sys);
int32_t orc_batch_info(void* sys, int32_t b, int64_t* size, int32_t* element_ids, int32_t* dof_map);
int32_t orc_set_dirichlet(void* sys, int64_t n, const int32_t* node, const int32_t* comp,
                          const double* value);

int64_t orc_pattern_nnz(void* sys);
int32_t orc_pattern(void* sys, int64_t* row_ptr, int32_t* rows, int32_t* cols);

int32_t orc_residual(void* sys, const double* u, double* r);
int32_t orc_element_residual(void* sys, int64_t e, const double* ue, double* re);
int32_t orc_jacobian(void* sys, const double* u, double* values);
int32_t orc_diagonal(void* sys, const double* u, double* d);
int32_t orc_eliminate(void* sys, double* values, double* residual, const double* u);
int32_t orc_constrain_residual(void* sys, double* residual, const double* u);
int32_t orc_mf_apply(void* sys, const double* u, const double* x, double* y);
int32_t orc_mf_apply_mt(void* sys, const double* u, const double* x, double* y, int32_t nthreads);
int32_t orc_mf_diagonal(void* sys, const double* u, double* d);
int32_t orc_mf_diagonal_mt(void* sys, const double* u, double* d, int32_t nthreads);  // threaded, same values
int32_t orc_csr_apply(void* sys, const double* values, const double* x, double* y);

/* op_kind 0: EXPLICIT over values (eliminated CSR values, pattern order); 1: MATRIX_FREE at state u */
int32_t orc_solve(void* sys, int32_t op_kind, const double* values_or_u, const orc_solver_cfg* cfg,
                  const double* b, const double* x0, double* x, orc_solve_report* rep,
                  double* history, int32_t hist_cap);
int32_t orc_solve_bvp(void* sys, const orc_newton_cfg* cfg, const double* x0, double* u,
                      orc_newton_report* rep, double* norms, int32_t norms_cap);
int32_t orc_load_stepping(void* sys, double total_strain, int32_t n_steps,
                          const orc_newton_cfg* cfg, double* u, int32_t* failed_step,
                          int32_t* converged, int32_t* step_iterations);

/* ---- J2 quadrature-point history (restatement only): n_elem * nq * 8 doubles, element-id indexed */
int64_t orc_history_size(void* sys);
int32_t orc_history_commit(void* sys, const double* u);
int32_t orc_history_copy(void* sys, double* out);
int32_t orc_history_set(void* sys, const double* in);

#ifdef __cplusplus
}
#endif
#endif
