// Developer microbenchmark (not part of the product): L2 -> SM bandwidth of
// cp.async.bulk copies (the bulk evaluator's staging path) and of LDG.128
// loads, on an L2-resident source (reads only; results discarded).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_l2 tools/microbench_l2.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

__device__ __forceinline__ unsigned su32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// each CTA: one thread issues NS x CHUNK-byte bulk copies per round into a
// ring, waits for the oldest, reissues; ITER rounds over a REGION-byte source
template <int NS>
__global__ void k_bulk(const char* src, size_t region, int chunk, int iters, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ unsigned long long bar[NS];
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  size_t off = (size_t(blockIdx.x) * 7919 * chunk) % region;
  unsigned ph[NS] = {};
  for (int it = 0; it < iters; ++it) {
    const int s = it % NS;
    if (it >= NS) {
      asm volatile(
          "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
              su32(&bar[s])),
          "r"(ph[s])
          : "memory");
      ph[s] ^= 1;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(chunk)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(sm + size_t(s) * chunk)),
                 "l"(src + off), "r"(chunk), "r"(su32(&bar[s]))
                 : "memory");
    off += size_t(chunk) * 148;
    if (off + chunk > region) off = (off + chunk) % (region - chunk);
    off &= ~size_t(127);
  }
  for (int s = 0; s < NS; ++s) {
    asm volatile(
        "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
            su32(&bar[s])),
        "r"(ph[s])
        : "memory");
  }
  if (sm[5] == 123) atomicAdd(sink, 1ull);
}

__global__ void k_ldg(const double2* src, size_t n2, int iters, unsigned long long* sink) {
  double acc = 0.0;
  size_t i = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) % n2;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (int it = 0; it < iters; ++it) {
    const double2 v = __ldcg(src + i);
    acc += v.x + v.y;
    i += stride;
    if (i >= n2) i -= n2;
  }
  if (acc == 12345.678) atomicAdd(sink, 1ull);
}

int main() {
  const size_t region = size_t(48) << 20;  // L2-resident
  char* src;
  unsigned long long* sink;
  CK(cudaMalloc(&src, region));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(src, 1, region));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int chunk : {2048, 4096, 8192, 16384}) {
    for (int cps : {1, 2, 4}) {
      const int NS = 4;
      const size_t smem = size_t(NS) * chunk;
      CK(cudaFuncSetAttribute(k_bulk<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      const int iters = int((size_t(4) << 30) / (size_t(sms) * cps * chunk));
      for (int w = 0; w < 2; ++w) {
        CK(cudaEventRecord(e0));
        k_bulk<NS><<<sms * cps, 32, smem>>>(src, region, chunk, iters, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
      }
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double bytes = double(sms) * cps * iters * chunk;
      std::printf("{\"path\": \"bulk\", \"chunk\": %d, \"ctas_per_sm\": %d, \"stages\": %d, \"TBps\": %.2f}\n", chunk,
                  cps, NS, bytes / (ms * 1e-3) / 1e12);
    }
  }
  for (int threads : {256, 512, 1024}) {
    for (int cps : {2, 4}) {
      const size_t n2 = region / 16;
      const int iters = 2000;
      for (int w = 0; w < 2; ++w) {
        CK(cudaEventRecord(e0));
        k_ldg<<<sms * cps, threads>>>(reinterpret_cast<const double2*>(src), n2, iters, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
      }
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double bytes = double(sms) * cps * threads * iters * 16.0;
      std::printf("{\"path\": \"ldg.128\", \"threads\": %d, \"ctas_per_sm\": %d, \"TBps\": %.2f}\n", threads, cps,
                  bytes / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
