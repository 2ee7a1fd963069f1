/* afem.h — C ABI of the B200-native matrix-free FEM core (libafem_b200.so).
 *
 * Drop-in boundary for the hot path of the reference (arXiv 2604.22087 "JetSCI", re-implemented in
 * /root/reference/proj/include/adfem as a header-only C++ library). Every entry point below names
 * the reference interface it replaces (file:line, paths relative to proj/include/adfem/).
 * The C++ overlay include/adfem_b200/adfem.hpp re-exposes these as the reference's own
 * namespace-adfem signatures; INTEGRATION.md shows the binding a maintainer adds.
 *
 * Conventions
 *  - Plain pointers and sizes only. Array arguments may be HOST or DEVICE pointers: the library
 *    inspects each pointer (cudaPointerGetAttributes) and copies host data in/out; device pointers
 *    are used in place (no copy), on the context's stream.
 *  - DOFs are interleaved per node (dof = dim*node + component; reference assembly.hpp:56-58).
 *  - All arithmetic is fp64. Integer outputs (connectivity, CSR pattern) are bit-exact with the
 *    reference; floating-point outputs agree within the tolerances stated in DESIGN.md §Parity.
 *  - Every function returns an afem_status. Non-zero codes map 1:1 onto the reference's exception
 *    types (errors.hpp:10-38 plus the std exceptions the reference throws); afem_last_error()
 *    returns the message (thread-local). Numerical non-convergence is NOT an error: it is reported
 *    in the report structs with converged = 0 and a failure string (krylov.hpp:66-72,
 *    newton.hpp:35-42), exactly like the reference.
 *  - Calls are synchronous with respect to the host unless stated otherwise.
 */
#ifndef AFEM_H
#define AFEM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AFEM_ABI_VERSION 1

typedef enum {
  AFEM_OK = 0,
  AFEM_E_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  AFEM_E_OUT_OF_RANGE = 2,     /* std::out_of_range */
  AFEM_E_LOGIC = 3,            /* std::logic_error (e.g. assembly.hpp:171 pattern mismatch) */
  AFEM_E_DOMAIN = 4,           /* std::domain_error (dual.hpp:97) */
  AFEM_E_LEASE = 5,            /* adfem::LeaseError (errors.hpp:10) */
  AFEM_E_STALE_EPOCH = 6,      /* adfem::StaleEpochError (errors.hpp:16) */
  AFEM_E_CAPABILITY = 7,       /* adfem::CapabilityError (errors.hpp:23) */
  AFEM_E_FACTORIZATION = 8,    /* adfem::FactorizationError (errors.hpp:29) */
  AFEM_E_INVERTED_ELEMENT = 9, /* adfem::InvertedElementError (errors.hpp:35) */
  AFEM_E_CUDA = 10,            /* CUDA runtime failure */
  AFEM_E_NCCL = 11,            /* collective failure (multi-GPU) */
  AFEM_E_NOMEM = 12,           /* device allocation failure */
  AFEM_E_RUNTIME = 13          /* other std::runtime_error */
} afem_status;

typedef struct afem_ctx_s* afem_ctx;
typedef struct afem_system_s* afem_system;
typedef struct afem_values_s* afem_values;
typedef struct afem_buffer_s* afem_buffer;
typedef struct afem_op_s* afem_op;

/* Material{model, E, nu} (material.hpp:15-27). model: 0 linear elastic (plane strain in 2D,
 * isotropic Hooke in 3D), 1 St Venant-Kirchhoff (material.hpp:49-69), and the north star's two
 * laws the reference lacks: 2 compressible Neo-Hookean (psi = mu/2 (J^-2/3 I1 - 3) +
 * kappa/2 (J-1)^2), 3 small-strain J2 plasticity with linear isotropic hardening (sigma_y,
 * hardening; quadrature-point history resident on the device). */
typedef struct {
  int32_t model;
  double E;
  double nu;
  double sigma_y;
  double hardening;
} afem_material;

/* SolverConfig (krylov.hpp:43-55). method: 0 CG, 1 GMRES, 2 BICGSTAB, 3 DIRECT_CHOL, 4 DIRECT_LU
 * (banded, backend.hpp:245-269: iterations 1, converged iff the true residual <= 1e-10, breakdown
 * reported in `failure`); precond: 0 NONE, 1 JACOBI, 2 ILU0. ILU0 and the direct methods need an
 * assembled operator (AFEM_E_CAPABILITY on a matrix-free one, like backend.hpp:151-156, 282). */
typedef struct {
  int32_t method;
  int32_t precond;
  double rtol;
  int32_t max_iter;
  int32_t restart;
} afem_solver_cfg;

/* SolveReport (krylov.hpp:66-72); the history is written to a caller buffer. */
typedef struct {
  int32_t converged;
  int32_t iterations;
  int32_t n_history;
  double wall_time;
  char failure[256];
} afem_solve_report;

/* NewtonConfig (newton.hpp:19-33). operator_kind: 0 EXPLICIT, 1 MATRIX_FREE (backend.hpp:20). */
typedef struct {
  double rtol;
  double atol;
  int32_t max_iter;
  int32_t operator_kind;
  afem_solver_cfg linear;
} afem_newton_cfg;

/* NewtonReport (newton.hpp:35-42); residual norms go to a caller buffer. */
typedef struct {
  int32_t converged;
  int32_t iterations;
  int32_t total_linear_iterations;
  int32_t n_norms;
  double total_time;
  char failure[256];
} afem_newton_report;

typedef struct {
  int32_t dim;
  int32_t nodes_per_elem;
  int64_t n_nodes;
  int64_t n_elem;
  int64_t n_dof;
  int64_t nnz;
  int32_t n_batches;  /* phases present, reference build_batches (assembly.hpp:36-67) */
  int32_t structured; /* 1 when the stencil fast path is available (grid systems) */
  int32_t nx, ny, nz;
  int64_t device_bytes; /* device memory held by the system */
} afem_system_info;

/* ------------------------------------------------------------------ context */
const char* afem_last_error(void);
int32_t afem_abi_version(void);
afem_status afem_ctx_create(int32_t device, afem_ctx* out);
afem_status afem_ctx_destroy(afem_ctx ctx);
/* Route all work onto a caller stream (e.g. torch.cuda.current_stream().cuda_stream). */
afem_status afem_ctx_set_stream(afem_ctx ctx, void* cuda_stream);
afem_status afem_ctx_synchronize(afem_ctx ctx);
/* Number of kernels this context has launched (evidence counter for bench.py). */
afem_status afem_ctx_launch_count(afem_ctx ctx, int64_t* count);
/* Measured FP64 FMA throughput of this device in TFLOP/s (the FP64 roofline denominator). */
afem_status afem_probe_fp64(afem_ctx ctx, double* tflops);

/* ------------------------------------------------------------------ mesh / system (L2-L3) */
/* Fibre centres U(0,lx)xU(0,ly) from mt19937_64(seed) (SURVEY §8d config 2 generator). Host only. */
afem_status afem_fibres(uint64_t seed, int32_t n_fibres, double lx, double ly, double* out_xy);

/* General mesh: Mesh{nodes, elements, material_of} (mesh.hpp:15-32) + build_batches
 * (assembly.hpp:36-67) + precompute_sparsity (assembly.hpp:71-99, built on the GPU, bit-exact).
 * dim 2: quad4 (4 nodes, CCW); dim 3: hex8. coords n_nodes*dim, conn n_elem*npe, phase n_elem. */
afem_status afem_system_create(afem_ctx ctx, int32_t dim, int64_t n_nodes, int64_t n_elem,
                               const double* coords, const int32_t* conn, const int32_t* phase,
                               int32_t n_mat, const afem_material* mats, afem_system* out);

/* Structured grid generated on the device: generate_two_phase_mesh (mesh.hpp:47-85) in 2D with
 * n_incl = 1 circle; its hex8 twin in 3D with n_incl fibres parallel to z (strict centroid test).
 * Enables the stencil fast path for the matrix-free operator. */
afem_status afem_system_create_grid(afem_ctx ctx, int32_t dim, int32_t nx, int32_t ny, int32_t nz,
                                    double lx, double ly, double lz, int32_t n_incl,
                                    const double* incl_xy, double radius, int32_t n_mat,
                                    const afem_material* mats, afem_system* out);
afem_status afem_system_destroy(afem_system sys);
afem_status afem_system_get_info(afem_system sys, afem_system_info* out);
/* Copy the mesh out (coords, conn, phase; any may be NULL). */
afem_status afem_system_mesh(afem_system sys, double* coords, int32_t* conn, int32_t* phase);
/* ElementBatch b (assembly.hpp:22-31): element ids [size] and dof_map [size*dim*npe]. */
afem_status afem_system_batch(afem_system sys, int32_t b, int64_t* size, int32_t* element_ids,
                              int32_t* dof_map);

/* DirichletSpec (mesh.hpp:35-43) validated like validate_dirichlet (mesh.hpp:105-116) and
 * stored as the constraint table (assembly.hpp:197-211). */
afem_status afem_set_dirichlet(afem_system sys, int64_t n, const int32_t* node, const int32_t* comp,
                               const double* value);
/* benchmark_bcs(mesh, strain) (mesh.hpp:89-101) for grid systems (and its 3D twin). */
afem_status afem_set_benchmark_dirichlet(afem_system sys, double strain);
/* Write the prescribed state: u[d] = value on constrained dofs, untouched elsewhere (newton.hpp:77-78). */
afem_status afem_impose_dirichlet(afem_system sys, double* u);

/* SparsityPattern (sparse.hpp:68-75): nnz, then row_ptr[n_dof+1] (int64), rows/cols[nnz]. */
afem_status afem_pattern_nnz(afem_system sys, int64_t* nnz);
afem_status afem_pattern(afem_system sys, int64_t* row_ptr, int32_t* rows, int32_t* cols);

/* ------------------------------------------------------------------ assembly (L1, L3) */
/* assemble_residual (assembly.hpp:126-139) over element_internal_force (element.hpp:68-125). */
afem_status afem_residual(afem_system sys, const double* u, double* r);
/* assemble_jacobian (assembly.hpp:144-173): K(u) values in pattern (CSR) order; hand-derived
 * quadrature-point tangents B^T D B (+ geometric term), no sort: slot-indexed, deterministic. */
afem_status afem_jacobian(afem_system sys, const double* u, double* values);
/* assemble_diagonal (assembly.hpp:177-188). */
afem_status afem_diagonal(afem_system sys, const double* u, double* d);
/* apply_dirichlet / eliminate_dirichlet (assembly.hpp:218-255) on pattern-ordered values. */
afem_status afem_eliminate(afem_system sys, double* values, double* residual, const double* u);
/* constrain_residual (assembly.hpp:259-264). */
afem_status afem_constrain_residual(afem_system sys, double* residual, const double* u);
/* CsrMatrix::apply (sparse.hpp:106-117) with pattern-ordered values. */
afem_status afem_csr_apply(afem_system sys, const double* values, const double* x, double* y);
/* free_norm (newton.hpp:46-51): ||r|| over unconstrained dofs. */
afem_status afem_free_norm(afem_system sys, const double* r, double* out);

/* ------------------------------------------------------------------ handoff (L4, backend.hpp:26-111) */
/* Device-resident assembled values (the CooTriplets.values the reference moves). */
afem_status afem_values_create(afem_system sys, afem_values* out);
afem_status afem_values_destroy(afem_values v);
afem_status afem_values_assemble(afem_values v, const double* u);
/* Overwrite the values with caller data (a hand-built CooTriplets.values, pattern order). */
afem_status afem_values_set(afem_values v, const double* values);
afem_status afem_values_eliminate(afem_values v, double* residual, const double* u);
afem_status afem_values_device_ptr(afem_values v, double** out);
afem_status afem_values_copy(afem_values v, double* out);

/* HandoffBuffer(pattern) (backend.hpp:35-38). */
afem_status afem_buffer_create(afem_system sys, afem_buffer* out);
afem_status afem_buffer_destroy(afem_buffer b);
/* handoff(CooTriplets&&) (backend.hpp:50-66): steals *values (no copy; *values becomes NULL),
 * state -> LeasedToSolver, ++epoch. LeaseError if already leased. */
afem_status afem_buffer_handoff(afem_buffer b, afem_values* values);
/* release() (backend.hpp:68-73). */
afem_status afem_buffer_release(afem_buffer b);
/* state: 0 OwnedByAssembly, 1 LeasedToSolver (backend.hpp:26). */
afem_status afem_buffer_state(afem_buffer b, int32_t* state, uint64_t* epoch);
/* assembly_values()/solver_values() (backend.hpp:76-87): device pointer of the shared storage. */
afem_status afem_buffer_assembly_values(afem_buffer b, double** out);
afem_status afem_buffer_solver_values(afem_buffer b, double** out);

/* ------------------------------------------------------------------ operators (L4) */
/* explicit_operator(buffer) (backend.hpp:199-214): CSR view aliasing the leased values. */
afem_status afem_op_create_explicit(afem_buffer b, afem_op* out);
/* matrix_free_operator(batches, u, dirichlet) (backend.hpp:222-236): copies u and the constraint
 * mask, assembles the Jacobi diagonal (unit on constrained dofs). */
afem_status afem_op_create_mf(afem_system sys, const double* u, afem_op* out);
/* Operator over a caller-supplied CSR pattern (HOST row_ptr n+1 / cols nnz, int32 like the
 * reference CsrMatrix, sparse.hpp:79-95): the explicit operator of the namespace-adfem drop-in
 * overlay for patterns that no device system produced. y = A x accumulates each row in column
 * order with separately rounded multiply/add, bitwise equal to CsrMatrix::apply (sparse.hpp:105-115)
 * on a non-FMA host build. Values are (re)loaded with afem_op_set_values (host or device, nnz).
 * Solvable with CG / GMRES / BiCGStab and NONE / JACOBI. */
afem_status afem_op_create_csr(afem_ctx ctx, int64_t n, int64_t nnz, const int32_t* row_ptr, const int32_t* cols,
                               afem_op* out);
afem_status afem_op_set_values(afem_op op, const double* values);
/* detail::eliminate_dirichlet (assembly.hpp:218-240) on a caller CSR (row_ptr n+1, cols / values
 * nnz, int32 indices) with a per-dof constraint table (constrained u8, prescribed f64), in place on
 * values and residual; same operation order and rounding as the reference loop (bitwise). */
afem_status afem_eliminate_csr(afem_ctx ctx, int64_t n, int64_t nnz, const int32_t* row_ptr, const int32_t* cols,
                               double* values, double* residual, const uint8_t* constrained,
                               const double* prescribed, const double* u);
/* constrain_residual (assembly.hpp:255-260) with a per-dof constraint table, in place. */
afem_status afem_constrain_masked(afem_ctx ctx, int64_t n, double* residual, const uint8_t* constrained,
                                  const double* prescribed, const double* u);
afem_status afem_op_destroy(afem_op op);
afem_status afem_op_kind(afem_op op, int32_t* kind);
afem_status afem_op_dim(afem_op op, int64_t* n);
/* LinearOperator::apply (backend.hpp:122-148). Explicit: lease/epoch validated (LeaseError /
 * StaleEpochError). Matrix-free: masked JVP, unit diagonal on constrained dofs. */
afem_status afem_op_apply(afem_op op, const double* x, double* y);
/* Enqueue the same apply on the context stream without synchronising or validating pointers
 * (both must be device pointers). For benchmarks and CUDA-graph capture. */
afem_status afem_op_apply_async(afem_op op, const double* x_dev, double* y_dev);
/* LinearOperator::diagonal (backend.hpp:160-166). */
afem_status afem_op_diagonal(afem_op op, double* d);
/* LinearOperator::csr (backend.hpp:151-156): CapabilityError on matrix-free operators. */
afem_status afem_op_csr_values(afem_op op, double** values_dev);
/* 1 when apply runs the structured stencil kernel. */
afem_status afem_op_uses_stencil(afem_op op, int32_t* flag);

/* ------------------------------------------------------------------ solvers (L5) */
/* run_solver (backend.hpp:241-286) / cg (krylov.hpp:350-408) / gmres (krylov.hpp:415-530) /
 * bicgstab (krylov.hpp:535-620).
 * x0 may be NULL (zero start). history: caller buffer of hist_cap doubles (may be NULL). */
afem_status afem_solve(afem_op op, const afem_solver_cfg* cfg, const double* b, const double* x0,
                       double* x, afem_solve_report* rep, double* history, int32_t hist_cap);

/* ------------------------------------------------------------------ Newton (L6) */
/* solve_bvp (newton.hpp:59-152) over the system's mesh, materials and Dirichlet table. */
afem_status afem_solve_bvp(afem_system sys, const afem_newton_cfg* cfg, const double* x0, double* u,
                           afem_newton_report* rep, double* norms, int32_t norms_cap);
/* solve_bvp with the per-iteration linear SolveReports (NewtonReport::linear_reports,
 * newton.hpp:38, 120): up to linear_cap reports, residual histories not included. */
afem_status afem_solve_bvp_ex(afem_system sys, const afem_newton_cfg* cfg, const double* x0, double* u,
                              afem_newton_report* rep, double* norms, int32_t norms_cap,
                              afem_solve_report* linear, int32_t linear_cap);
/* load_stepping (newton.hpp:163-186) for grid systems (benchmark_bcs regenerated per step). */
afem_status afem_load_stepping(afem_system sys, double total_strain, int32_t n_steps,
                               const afem_newton_cfg* cfg, double* u, int32_t* failed_step,
                               int32_t* converged, int32_t* step_iterations);

/* ------------------------------------------------------------------ quadrature-point history (J2)
 * The reference kernel has no state argument (element.hpp:68-70); J2 systems keep the committed
 * history (plastic strain [xx,yy,zz,yz,xz,xy], alpha, pad: 8 doubles per Gauss point, element-major)
 * resident on the device. Residuals, tangents and operators evaluate the return map from the
 * committed history; afem_load_stepping commits after every converged step. */
afem_status afem_history_size(afem_system sys, int64_t* n); /* doubles; 0 without a J2 phase */
afem_status afem_history_commit(afem_system sys, const double* u);
afem_status afem_history_reset(afem_system sys);
afem_status afem_history_copy(afem_system sys, double* out);
afem_status afem_history_set(afem_system sys, const double* in);

/* ------------------------------------------------------------------ multi-GPU slab decomposition
 * (the reference has no distribution — the paper distributes only the PETSc solve,
 * PAPER.md:296-302). One process per GPU, each owning a contiguous z-slab of element layers; the
 * node plane between slabs is shared and owned by the lower rank. The only data-path collectives
 * are a one-plane exchange with each neighbour per operator apply and scalar allreduces for the
 * Krylov dot products (NCCL over NVLink). (A threads backend that runs the same algorithm with
 * several subdomains on one device, for tests, is declared in afem_testing.h.) */
typedef struct afem_dist_s* afem_dist;

/* Element layers [z0, z1) of rank `rank` when nz layers are split over `size` ranks. Host only. */
afem_status afem_slab_range(int32_t nz, int32_t size, int32_t rank, int32_t* z0, int32_t* z1);
/* 128-byte NCCL unique id (rank 0 creates it, the host broadcasts it). */
afem_status afem_nccl_unique_id(void* out128);
afem_status afem_dist_create_nccl(afem_ctx ctx, const void* uid128, int32_t rank, int32_t size, afem_dist* out);
afem_status afem_dist_destroy(afem_dist d);
/* benchmark_bcs of the global grid restricted to this rank's slab system (the slab's local grid
 * system from afem_system_create_grid with nz = z1 - z0 and lz scaled accordingly). */
afem_status afem_dist_set_benchmark_dirichlet(afem_dist d, afem_system slab, double strain, double lx_global);
/* matrix_free_operator over the distributed system (local operator + plane halo). */
afem_status afem_dist_op_create_mf(afem_dist d, afem_system slab, const double* u, afem_op* out);
/* explicit_operator over the distributed system: the slab's own eliminated CSR values (pattern
 * order, nnz of the slab system, host or device; copied) — the local SpMV yields partial sums on
 * the shared node planes, completed by the same plane halo as the matrix-free operator. */
afem_status afem_dist_op_create_explicit(afem_dist d, afem_system slab, const double* values, afem_op* out);
/* run_solver, every rank calling collectively: CG (device-scalar loop), GMRES(restart) or BiCGStab
 * (owned-dof inner products + allreduce), NONE or JACOBI; reports are identical on all ranks. */
afem_status afem_dist_solve(afem_dist d, afem_op op, const afem_solver_cfg* cfg, const double* b, const double* x0,
                            double* x, afem_solve_report* rep, double* history, int32_t hist_cap);
/* Sum the shared planes of a slab-partial vector (e.g. a local residual) with the neighbours'
 * partials, in place (collective). */
afem_status afem_dist_assemble(afem_dist d, afem_op op, double* v);
/* solve_bvp (newton.hpp:59-152) over the slab decomposition (collective; MATRIX_FREE tangent, or
 * EXPLICIT = each slab's assembled + eliminated tangent; CG + Jacobi): residual shared planes summed
 * across neighbours, global free norm over owned dofs. */
afem_status afem_dist_solve_bvp(afem_dist d, afem_system slab, const afem_newton_cfg* cfg, const double* x0,
                                double* u, afem_newton_report* rep, double* norms, int32_t norms_cap);
/* load_stepping (newton.hpp:163-186) over the slab decomposition with the global benchmark BCs,
 * committing each rank's J2 history after every converged step (collective). */
afem_status afem_dist_load_stepping(afem_dist d, afem_system slab, double total_strain, int32_t n_steps,
                                    double lx_global, const afem_newton_cfg* cfg, double* u, int32_t* failed_step,
                                    int32_t* converged, int32_t* step_iterations);
/* Global dot over owned dofs (collective). */
afem_status afem_dist_dot(afem_dist d, afem_op op, const double* a, const double* b, double* out);

#ifdef __cplusplus
}
#endif
#endif /* AFEM_H */
