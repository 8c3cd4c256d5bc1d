// k_phimv_block instantiations (1, 2, 1) batch 5 or default (Q, V, R); split across files
// so they compile in parallel.
#include "phx_eval_kernel.cuh"

namespace phx {

bool eval_kernels_q1v2a(int QT, int V, int R, bool part, bool dyn, bool small, bool cluster, EvalKernel* out) {
  (void)small;
  (void)cluster;
  PHX_EVAL_CASE2(1, 2, 1, 5)
  return false;
}

}  // namespace phx
