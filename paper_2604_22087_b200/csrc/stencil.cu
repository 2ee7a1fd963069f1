// Structured-grid stencil fast path for the linear matrix-free operator (placeholder: the general
// node-centric kernel in assembly.cu is used until the stencil plan is available).
#include "afem_impl.hpp"

namespace afem {
struct StencilPlan {};
StencilPlan* make_stencil_plan(System&, const MfOp&) { return nullptr; }
void stencil_apply(StencilPlan&, const MfOp&, const double*, double*) {}
void destroy_stencil_plan(StencilPlan* p) { delete p; }
}  // namespace afem
