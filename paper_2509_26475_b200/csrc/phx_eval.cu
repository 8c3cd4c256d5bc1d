// Dispatch of the persistent phimv_block kernel variants (instantiated in
// phx_eval_q*.cu from phx_eval_kernel.cuh).
#include "phx_kernels.cuh"

namespace phx {

namespace {

bool select_kernel(int QT, int V, int R, bool part, bool dyn, bool small, EvalKernel* k) {
  return eval_kernels_q1v1(QT, V, R, part, dyn, small, k) ||
         eval_kernels_q1v2a(QT, V, R, part, dyn, small, k) ||
         eval_kernels_q1v2b(QT, V, R, part, dyn, small, k) ||
         eval_kernels_q2(QT, V, R, part, dyn, small, k) ||
         eval_kernels_q4(QT, V, R, part, dyn, small, k) ||
         eval_kernels_q8(QT, V, R, part, dyn, small, k);
}

}  // namespace

cudaError_t coop_grid_size(int QT, int V, int R, bool part, bool dyn, bool small, int block,
                           int* max_blocks) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  EvalKernel k{};
  if (!select_kernel(QT, V, R, part, dyn, small, &k)) return cudaErrorInvalidValue;
  int per_sm = 0;
  e = k.occ(block, &per_sm);
  if (e != cudaSuccess) return e;
  *max_blocks = per_sm * sms;
  return cudaSuccess;
}

#ifndef PHX_X_BLOCK
#define PHX_X_BLOCK 256
#endif
int eval_block_size() { return PHX_X_BLOCK; }

cudaError_t launch_phimv_block(const BlockArgs& a, int grid, int block, cudaStream_t st) {
  BlockArgs copy = a;
  void* args[] = {&copy};
  EvalKernel k{};
  if (!select_kernel(a.QT, a.vec, a.R, a.nparts > 1, a.dyn != 0, a.bsmall != 0, &k))
    return cudaErrorInvalidValue;
  count_launch();
  int per_sm = 0;  // also sets the dynamic shared memory attribute of the variant
  const cudaError_t e = k.occ(block, &per_sm);
  if (e != cudaSuccess) return e;
  return cudaLaunchCooperativeKernel(k.fn, grid, block, args, eval_pipe_bytes(), st);
}

}  // namespace phx
