// Developer microbenchmark (not part of the product): the C2 S-term pass
// stripped to its memory traffic -- one launch per term, no persistent loop,
// no stopping logic -- to measure how close a minimal kernel with the same
// access pattern gets to the HBM roofline.  Traffic per term: CSR + 48 w n
// bytes (D gather, D' write, S RMW, Vw RMW), the evaluator's S-term count.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o mb tools/microbench_sterm.cu
// ./mb [variant]   variant 0: gathers from registers, batch of 5 in flight
//                  variant 1: gathers serialised (load -> use, as ptxas does in the evaluator)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                             \
    }                                                                           \
  } while (0)

constexpr int W = 16;  // block width (p+1) r
constexpr int G = 8;   // lanes per row (double2 each)

template <bool SERIAL>
__global__ void __launch_bounds__(256, 4)
    k_sterm(int n, const int* __restrict__ rp, const int* __restrict__ ci,
            const double* __restrict__ av, const double* __restrict__ D, double* __restrict__ Dn,
            double* __restrict__ S, double* __restrict__ Vw, double kd, double ka, double tos,
            double xi, double sigma, unsigned long long* __restrict__ maxd) {
  const int lane = threadIdx.x & 31;
  const int g = lane / G, q = lane % G;
  const int c = 2 * q;
  const int rows_per_warp = 32 / G;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  unsigned long long m = 0;
  for (int base = warp_global * rows_per_warp; base < n; base += nwarps * rows_per_warp) {
    const int row = base + g;
    if (row >= n) continue;
    const size_t o = size_t(row) * W + c;
    const double2 vw = __ldcs(reinterpret_cast<const double2*>(Vw + o));
    const double2 so = __ldcs(reinterpret_cast<const double2*>(S + o));
    const double2 ds = *reinterpret_cast<const double2*>(D + o);
    double2 vwl = make_double2(0.0, 0.0);
    if (c >= 8) vwl = __ldcs(reinterpret_cast<const double2*>(Vw + o - 4));
    const int e0 = __ldg(rp + row), e1 = __ldg(rp + row + 1);
    double a0 = 0.0, a1 = 0.0;
    if (SERIAL) {
      for (int e = e0; e < e1; ++e) {
        const double2 x = *reinterpret_cast<const double2*>(D + size_t(__ldg(ci + e)) * W + c);
        const double a = __ldg(av + e);
        a0 = a0 + a * x.x;
        a1 = a1 + a * x.y;
      }
    } else {
      for (int e = e0; e < e1; e += 5) {
        double2 x[5];
        double a[5];
#pragma unroll
        for (int u = 0; u < 5; ++u) {
          const int ee = e + u < e1 ? e + u : e;
          x[u] = *reinterpret_cast<const double2*>(D + size_t(__ldg(ci + ee)) * W + c);
          a[u] = __ldg(av + ee);
        }
#pragma unroll
        for (int u = 0; u < 5; ++u)
          if (e + u < e1) {
            a0 = a0 + a[u] * x[u].x;
            a1 = a1 + a[u] * x[u].y;
          }
      }
    }
    const double g0 = (c >= 8 ? vwl.x * ka : 0.0) + vw.x * kd;
    const double g1 = (c >= 8 ? vwl.y * ka : 0.0) + vw.y * kd;
    const double y0 = (a0 - xi * ds.x) * tos + g0;
    const double y1 = (a1 - xi * ds.y) * tos + g1;
    __syncwarp();
    __stcs(reinterpret_cast<double2*>(Vw + o), make_double2(g0, g1));
    *reinterpret_cast<double2*>(Dn + o) = make_double2(y0, y1);
    __stcs(reinterpret_cast<double2*>(S + o), make_double2(so.x + y0 / sigma, so.y + y1 / sigma));
    double rs = fabs(y0) + fabs(y1);
    for (int k = 1; k < G; k <<= 1) rs += __shfl_xor_sync(0xffffffffu, rs, k);
    const unsigned long long b = __double_as_longlong(rs);
    m = b > m ? b : m;
  }
  for (int k = 16; k >= 1; k >>= 1) {
    const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, m, k);
    m = o2 > m ? o2 : m;
  }
  if (lane == 0) atomicMax(maxd, m);
}

int main(int argc, char** argv) {
  const int variant = argc > 1 ? std::atoi(argv[1]) : 0;
  const int N = 1024, n = N * N;
  std::vector<int> rp(n + 1), ci;
  std::vector<double> av;
  ci.reserve(size_t(n) * 5);
  av.reserve(size_t(n) * 5);
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < N; ++i) {
      const int r = j * N + i;
      rp[r] = int(ci.size());
      if (j > 0) { ci.push_back(r - N); av.push_back(1.0); }
      if (i > 0) { ci.push_back(r - 1); av.push_back(1.5); }
      ci.push_back(r); av.push_back(-4.0);
      if (i < N - 1) { ci.push_back(r + 1); av.push_back(0.5); }
      if (j < N - 1) { ci.push_back(r + N); av.push_back(1.0); }
    }
  rp[n] = int(ci.size());
  const size_t nnz = ci.size(), nb = size_t(n) * W;
  int *d_rp, *d_ci;
  double *d_av, *D0, *D1, *S, *Vw;
  unsigned long long* d_m;
  CK(cudaMalloc(&d_rp, (n + 1) * 4));
  CK(cudaMalloc(&d_ci, nnz * 4));
  CK(cudaMalloc(&d_av, nnz * 8));
  CK(cudaMalloc(&D0, nb * 8));
  CK(cudaMalloc(&D1, nb * 8));
  CK(cudaMalloc(&S, nb * 8));
  CK(cudaMalloc(&Vw, nb * 8));
  CK(cudaMalloc(&d_m, 8));
  CK(cudaMemcpy(d_rp, rp.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_av, av.data(), nnz * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(D0, 0, nb * 8));
  CK(cudaMemset(D1, 0, nb * 8));
  CK(cudaMemset(S, 0, nb * 8));
  CK(cudaMemset(Vw, 0, nb * 8));
  int sms = 0, per = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  auto kfn = variant ? k_sterm<true> : k_sterm<false>;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kfn, 256, 0));
  const int grid = sms * per;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int iters = 40;
  for (int it = 0; it < 5; ++it)
    kfn<<<grid, 256>>>(n, d_rp, d_ci, d_av, it & 1 ? D1 : D0, it & 1 ? D0 : D1, S, Vw, 0.9, 0.1,
                       1e-4, -2.0, 2.0, d_m);
  CK(cudaEventRecord(a));
  for (int it = 0; it < iters; ++it)
    kfn<<<grid, 256>>>(n, d_rp, d_ci, d_av, it & 1 ? D1 : D0, it & 1 ? D0 : D1, S, Vw, 0.9, 0.1,
                       1e-4, -2.0, 2.0, d_m);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  const double per_term = ms / iters * 1e-3;
  const double bytes = 12.0 * double(nnz) + 4.0 * (n + 1) + 48.0 * W * double(n);
  std::printf("{\"variant\": \"%s\", \"grid\": %d, \"ctas_per_sm\": %d, \"us_per_term\": %.2f, "
              "\"alg_GBps\": %.1f, \"frac_of_6547.5\": %.3f}\n",
              variant ? "serial" : "batched", grid, per, per_term * 1e6, bytes / per_term / 1e9,
              bytes / per_term / 1e9 / 6547.5);
  return 0;
}
