// Cluster-mode k_phimv_block variants (one thread-block cluster, one CTA per
// part, blocks and CSR in shared memory): compiled with 1024-thread CTAs --
// 32 warps per part, so a 16-part cluster runs 512 warps on the small
// operators it serves (the register budget stays 64 per thread).
#define PHX_X_BLOCK 1024
#include "phx_eval_kernel.cuh"

namespace phx {

#define PHX_CL_CASE(q, v, r, bs)                                          \
  if (QT == q && V == v && R == r) {                                      \
    *out = small ? eval_kernel_cluster<q, v, r, bs>()                     \
                 : eval_kernel_cluster<q, v, r, 0>();                     \
    return out->fn != nullptr;                                            \
  }

bool eval_kernels_cl(int QT, int V, int R, bool small, EvalKernel* out) {
  PHX_CL_CASE(1, 1, 1, 0)
  PHX_CL_CASE(1, 1, 2, 0)
  PHX_CL_CASE(1, 2, 1, 5)
  PHX_CL_CASE(1, 2, 2, 2)
  return false;
}

int eval_cl_block() { return kBlock; }

}  // namespace phx
