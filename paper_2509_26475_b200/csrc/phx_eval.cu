// Dispatch of the persistent phimv_block kernel variants (instantiated in
// phx_eval_q*.cu from phx_eval_kernel.cuh).
#include "phx_kernels.cuh"

namespace phx {

namespace {

bool select_kernel(int QT, int V, int R, bool part, bool dyn, bool small, EvalKernel* k,
                   bool cluster = false) {
  return eval_kernels_q1v1(QT, V, R, part, dyn, small, cluster, k) ||
         eval_kernels_q1v2a(QT, V, R, part, dyn, small, cluster, k) ||
         eval_kernels_q1v2b(QT, V, R, part, dyn, small, cluster, k) ||
         eval_kernels_q2(QT, V, R, part, dyn, small, cluster, k) ||
         eval_kernels_q4(QT, V, R, part, dyn, small, cluster, k) ||
         eval_kernels_q8(QT, V, R, part, dyn, small, cluster, k);
}

}  // namespace

cudaError_t coop_grid_size(int QT, int V, int R, bool part, bool dyn, bool small, int block,
                           int* max_blocks, bool lat) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  EvalKernel k{};
  if (lat ? !eval_kernels_lat(QT, V, R, small, &k) : !select_kernel(QT, V, R, part, dyn, small, &k))
    return cudaErrorInvalidValue;
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
  if (a.lat ? !eval_kernels_lat(a.QT, a.vec, a.R, a.bsmall != 0, &k)
            : !select_kernel(a.QT, a.vec, a.R, a.nparts > 1, a.dyn != 0, a.bsmall != 0, &k))
    return cudaErrorInvalidValue;
  count_launch();
  int per_sm = 0;  // also sets the dynamic shared memory attribute of the variant
  const cudaError_t e = k.occ(block, &per_sm);
  if (e != cudaSuccess) return e;
  return cudaLaunchCooperativeKernel(k.fn, grid, block, args, k.smem, st);
}

size_t eval_cluster_smem(int32_t cl_rows, int32_t cl_nnz, int32_t tile, int32_t ldb, int32_t ldf) {
  const size_t rpad = size_t((cl_rows + tile - 1) / tile) * size_t(tile) + 1;
  return size_t(cl_rows) * (4 * size_t(ldb) + 3 * size_t(ldf)) * sizeof(double) +
         size_t(cl_nnz) * (sizeof(double) + sizeof(int)) + rpad * sizeof(int);
}

// cluster mode: nparts CTAs forming one thread-block cluster (<= 8 portable,
// <= 16 with the non-portable size), each with its part's blocks in shared
// memory; no cooperative launch needed (a cluster is co-resident)
cudaError_t launch_phimv_block_cluster(const BlockArgs& a, int nparts, int block, cudaStream_t st) {
  EvalKernel k{};
  if (!eval_kernels_cl(a.QT, a.vec, a.R, a.bsmall != 0, &k)) return cudaErrorInvalidValue;
  block = eval_cl_block();
  const size_t smem = eval_cluster_smem(a.cl_rows, a.cl_nnz, a.tile, a.ldb, a.ldf);
  cudaError_t e = cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  if (nparts > 8) {
    e = cudaFuncSetAttribute(k.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  BlockArgs copy = a;
  void* args[] = {&copy};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(nparts), 1, 1);
  cfg.blockDim = dim3(unsigned(block), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(nparts);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  count_launch();
  return cudaLaunchKernelExC(&cfg, k.fn, args);
}

}  // namespace phx
