// k_phimv_block instantiations (4, 1, 1), (4, 2, 1) (Q, V, R); split across files
// so they compile in parallel.
#include "phx_eval_kernel.cuh"

namespace phx {

bool eval_kernels_q4(int QT, int V, int R, bool part, bool dyn, bool small, bool cluster, EvalKernel* out) {
  (void)small;
  (void)cluster;
  PHX_EVAL_CASE(4, 1, 1)
  PHX_EVAL_CASE(4, 2, 1)
  return false;
}

}  // namespace phx
