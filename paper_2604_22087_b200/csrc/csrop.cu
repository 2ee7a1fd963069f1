// Operator over a caller-supplied CSR matrix (any pattern, no mesh behind it): the device side of
// the drop-in overlay's explicit operator (include/adfem_dropin/adfem/backend.hpp), whose CSR view
// aliases the reference HandoffBuffer's host value store (backend.hpp:199-214).
//
// y = A x runs one thread per row and accumulates the row in column order with separately
// rounded multiply and add (no FMA contraction), i.e. exactly the reference's CsrMatrix::apply
// (sparse.hpp:105-115) as a non-FMA host build computes it: the result is bitwise identical.
// This is a parity path (the overlay refreshes the values from the host store on every use); the
// performance path is the pattern-bound ExplicitOp (k_csr_apply, warp per node).
#include "afem_impl.hpp"

namespace afem {

namespace {

__global__ void k_csr_exact(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ v, const double* __restrict__ x, double* __restrict__ y,
                            int64_t n, const int* skip) {
  if (skip && *skip) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int32_t k = rp[i]; k < rp[i + 1]; ++k) s = __dadd_rn(s, __dmul_rn(v[k], x[ci[k]]));
    y[i] = s;
  }
}

// csr_diagonal (krylov.hpp:102-111): the stored diagonal entry of each row, 0 when absent
__global__ void k_csr_exact_diag(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const double* __restrict__ v, double* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double di = 0.0;
    for (int32_t k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] == i) di = v[k];
    d[i] = di;
  }
}

// detail::eliminate_dirichlet (assembly.hpp:218-240) on a caller CSR, one thread per row, with the
// reference's arithmetic order and rounding (r_i += v_ik (p_k - u_k) for constrained columns, unit
// rows; constrained residual entries become u - p): bitwise equal to the host loop.
__global__ void k_eliminate_exact(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, double* values,
                                  double* residual, const uint8_t* __restrict__ cons,
                                  const double* __restrict__ presc, const double* __restrict__ u, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool c_i = cons[i] != 0;
    double r = residual[i];
    for (int32_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int32_t j = ci[k];
      if (!c_i && cons[j]) {
        r = __dadd_rn(r, __dmul_rn(values[k], __dsub_rn(presc[j], u[j])));
        values[k] = 0.0;
      } else if (c_i) {
        values[k] = (i == j) ? 1.0 : 0.0;
      }
    }
    residual[i] = c_i ? __dsub_rn(u[i], presc[i]) : r;
  }
}

// constrain_residual (assembly.hpp:255-260)
__global__ void k_constrain_exact(double* residual, const uint8_t* __restrict__ cons, const double* __restrict__ presc,
                                  const double* __restrict__ u, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (cons[i]) residual[i] = __dsub_rn(u[i], presc[i]);
}

}  // namespace

void eliminate_csr(Ctx& c, int64_t n, const int32_t* rp, const int32_t* ci, double* values, double* residual,
                   const uint8_t* cons, const double* presc, const double* u) {
  launch(c, k_eliminate_exact, grid_for(n, 128, 148 * 16), 128, 0, rp, ci, values, residual, cons, presc, u, n);
}

void constrain_masked(Ctx& c, int64_t n, double* residual, const uint8_t* cons, const double* presc,
                      const double* u) {
  launch(c, k_constrain_exact, grid_for(n, 256, 148 * 16), 256, 0, residual, cons, presc, u, n);
}

struct CsrOp : Operator {
  std::unique_ptr<System> own;  // carries the context only (no mesh)
  DevArray<int32_t> rp, ci;
  DevArray<double> vals;
  int64_t nnz = 0;
  const int* skip = nullptr;
  void apply(const double* x, double* y) override {
    launch(*sys->ctx, k_csr_exact, grid_for(n, 128, 148 * 16), 128, 0, rp.p, ci.p, vals.p, x, y, n, skip);
  }
  void diagonal(double* d) override {
    launch(*sys->ctx, k_csr_exact_diag, grid_for(n, 128, 148 * 16), 128, 0, rp.p, ci.p, vals.p, d, n);
  }
  bool set_skip(const int* flag) override {
    skip = flag;
    return true;
  }
};

// row_ptr / cols validated like the reference CsrMatrix (sparse.hpp:119-124, 150-156).
std::unique_ptr<Operator> make_csr_op(Ctx& c, int64_t n, int64_t nnz, const int32_t* h_rp, const int32_t* h_ci) {
  if (n < 0 || nnz < 0) throw std::invalid_argument("csr operator: negative size");
  if (h_rp[0] != 0 || h_rp[n] != nnz) throw std::invalid_argument("CsrMatrix: row_ptr does not span the values");
  for (int64_t i = 0; i < n; ++i)
    if (h_rp[i + 1] < h_rp[i]) throw std::invalid_argument("CsrMatrix: row_ptr must be non-decreasing");
  for (int64_t k = 0; k < nnz; ++k)
    if (h_ci[k] < 0 || h_ci[k] >= n) throw std::out_of_range("CsrMatrix: column index outside matrix shape");
  auto op = std::make_unique<CsrOp>();
  op->own = std::make_unique<System>();
  op->own->ctx = &c;
  op->own->n_dof = n;
  op->sys = op->own.get();
  op->kind = 0;
  op->n = n;
  op->nnz = nnz;
  op->rp.alloc(n + 1);
  op->ci.alloc(nnz > 0 ? nnz : 1);
  op->vals.alloc(nnz > 0 ? nnz : 1);
  AFEM_CK(cudaMemcpyAsync(op->rp.p, h_rp, (n + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, c.stream));
  if (nnz) AFEM_CK(cudaMemcpyAsync(op->ci.p, h_ci, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, c.stream));
  fill(c, 0.0, op->vals.p, nnz);
  AFEM_CK(cudaStreamSynchronize(c.stream));
  return op;
}

double* csr_op_values(Operator& o, int64_t* nnz) {
  auto* p = dynamic_cast<CsrOp*>(&o);
  if (!p) throw std::invalid_argument("operator was not created by afem_op_create_csr");
  *nnz = p->nnz;
  return p->vals.p;
}

}  // namespace afem
