// Latency-mode k_phimv_block variants (unpartitioned, static tiles, one CTA
// per SM, register budget 255): for operators with fewer tiles than SMs (C1,
// small integrator grids), whose grid steps are latency-bound -- with the
// registers, the gather's loads of a row batch instead of serialising.
#include "phx_eval_kernel.cuh"

namespace phx {

#define PHX_LAT_CASE(q, v, r, bs)                                                      \
  if (QT == q && V == v && R == r) {                                                   \
    *out = small ? eval_kernel<q, v, r, false, false, bs, false, true>()               \
                 : eval_kernel<q, v, r, false, false, 0, false, true>();               \
    return true;                                                                       \
  }

bool eval_kernels_lat(int QT, int V, int R, bool small, EvalKernel* out) {
  PHX_LAT_CASE(1, 1, 1, 0)
  PHX_LAT_CASE(1, 1, 2, 0)
  PHX_LAT_CASE(1, 2, 1, 5)
  PHX_LAT_CASE(1, 2, 2, 2)
  return false;
}

}  // namespace phx
