// k_phimv_block instantiations (1, 1, 1), (1, 1, 2) (Q, V, R); split across files
// so they compile in parallel.
#include "phx_eval_kernel.cuh"

namespace phx {

bool eval_kernels_q1v1(int QT, int V, int R, bool part, bool dyn, bool small, bool cluster, EvalKernel* out) {
  (void)small;
  (void)cluster;
  PHX_EVAL_CASE(1, 1, 1)
  PHX_EVAL_CASE(1, 1, 2)
  return false;
}

// dynamic shared memory of every k_phimv_block variant (the per-warp pipes)
size_t eval_pipe_bytes() { return kPipeBytes; }

}  // namespace phx
