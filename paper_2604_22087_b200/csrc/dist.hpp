// Multi-GPU slab decomposition: communicator abstraction and the distributed operator (dist.cu).
#pragma once

#include <memory>
#include <vector>

#include "afem_impl.hpp"

namespace afem {

struct NcclError : std::runtime_error { using std::runtime_error::runtime_error; };

// Data-path collectives of the slab decomposition: scalar allreduces (Krylov dots) and the
// exchange of one node plane with each z neighbour.
struct Comm {
  virtual ~Comm() = default;
  int rank = 0, size = 1;
  virtual void allreduce_sum(double* d, int n, cudaStream_t s) = 0;  // device buffer, in place
  // send_lo -> rank-1 (recv_lo <- rank-1), send_hi -> rank+1 (recv_hi <- rank+1); nullptr: no neighbour
  virtual void exchange(const double* send_lo, double* recv_lo, const double* send_hi, double* recv_hi, size_t n,
                        cudaStream_t s) = 0;
};

struct ThreadGroup;
ThreadGroup* thread_group_create(int n);
void thread_group_destroy(ThreadGroup* g);
Comm* comm_create_nccl(const void* uid, int rank, int size);
Comm* comm_create_threads(ThreadGroup* g, int rank);
void nccl_unique_id(void* out);

void slab_range(int nz, int size, int rank, int* z0, int* z1);
std::vector<Constraint> slab_benchmark_bcs(const System& s, int rank, int size, double strain, double lx_global);

// Operator of one slab: local apply + plane halo add. Matrix-free (local = the slab's MfOp) or
// assembled (vals = the slab's eliminated CSR values: the local SpMV gives partial sums on the two
// shared planes exactly like the matrix-free apply).
struct DistMfOp : Operator {
  std::unique_ptr<MfOp> local;
  DevArray<double> vals;  // assembled variant (local == nullptr)
  Comm* comm = nullptr;
  int64_t plane = 0;         // dofs per z node plane
  int64_t owned_offset = 0;  // first owned dof (the bottom plane belongs to rank-1 when rank > 0)
  DevArray<double> diag, send_lo, recv_lo, send_hi, recv_hi;
  ~DistMfOp() override;
  void apply(const double* x, double* y) override;
  // y = A x and dot_out[0] = owned x.y (before the allreduce): the interior wave's fused stencil dot
  // plus the owned shared plane's, summed after its halo add; false where the operator cannot fuse
  bool apply_dot(const double* x, double* y, double* dot_out) override;
  void diagonal(double* d) override;
  const int* skip = nullptr;  // the CG loop's device done flag (stencil launches only)
  bool set_skip(const int* flag) override {
    skip = flag;
    return local && local->stencil;
  }
  bool uses_stencil() const override { return local && local->uses_stencil(); }
  const uint8_t* mask() const { return local ? local->mask.p : sys->mask.p; }
  // owned-dof inner products + allreduce (the GMRES / BiCGStab scalars, identical on every rank)
  double inner(const double* a, const double* b) override;
  void inner_dev(const double* a, const double* b, double* out_dev) override;
  double resid(const double* b, const double* x, double* scratch, double* r) override;
  int64_t dot_begin() const override { return owned_offset; }
  void allreduce_dev(double* d, int k) override { comm->allreduce_sum(d, k, sys->ctx->stream); }
  void halo_add(double* v, const double* x_for_mask, bool diag_mode);
  // the received neighbour partials added into v's shared planes (+ unit Dirichlet rows)
  void halo_finish(double* v, const double* x_for_mask, bool diag_mode, double* dot_out = nullptr);
  void apply_impl(const double* x, double* y, double* dot_out);
};

std::unique_ptr<DistMfOp> make_dist_mf_op(System& s, Comm* comm, std::unique_ptr<MfOp> local);
std::unique_ptr<DistMfOp> make_dist_csr_op(System& s, Comm* comm, const double* d_values);
void dist_solve(DistMfOp& op, const SolverCfg& cfg, const double* b, const double* x0, double* x, SolveReport& rep);
double dist_dot(DistMfOp& op, const double* a, const double* b);

}  // namespace afem
