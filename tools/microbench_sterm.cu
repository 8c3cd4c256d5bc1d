// Developer microbenchmark (not part of the product): the C2 S-term pass
// stripped to its memory traffic -- one launch per term, no persistent loop,
// no stopping logic -- to measure how close a minimal kernel with the same
// access pattern gets to the HBM roofline.  Traffic per term: CSR + 48 w n
// bytes (D gather, D' write, S RMW, Vw RMW), the evaluator's S-term count.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o mb tools/microbench_sterm.cu
// ./mb [variant]   variant 0: gathers from registers, batch of 5 in flight
//                  variant 1: gathers serialised (load -> use, as ptxas does in the evaluator)
//                  variant 2: variant 1 in one persistent launch, grid.sync between terms
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

// variant 2: the same body in ONE persistent cooperative launch, a grid-wide
// barrier between terms (the evaluator's structure)
#include <cooperative_groups.h>
__global__ void __launch_bounds__(256, 4)
    k_sterm_persistent(int n, int terms, const int* __restrict__ rp, const int* __restrict__ ci,
                       const double* __restrict__ av, double* D0, double* D1,
                       double* __restrict__ S, double* __restrict__ Vw,
                       unsigned long long* __restrict__ maxd) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int lane = threadIdx.x & 31;
  const int g = lane / G, q = lane % G;
  const int c = 2 * q;
  const int rows_per_warp = 32 / G;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const double kd = 0.9, ka = 0.1, tos = 1e-4, xi = -2.0;
  double sigma = 1.0;
  for (int t = 0; t < terms; ++t) {
    const double* D = (t & 1) ? D1 : D0;
    double* Dn = (t & 1) ? D0 : D1;
    sigma *= double(t + 2);
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
      for (int e = e0; e < e1; ++e) {
        const double2 x = *reinterpret_cast<const double2*>(D + size_t(__ldg(ci + e)) * W + c);
        const double a = __ldg(av + e);
        a0 = a0 + a * x.x;
        a1 = a1 + a * x.y;
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
    if (lane == 0) atomicMax(maxd + (t % 3), m);
    grid.sync();
    if (__longlong_as_double(static_cast<long long>(maxd[t % 3])) < 0.0) return;  // read the max
  }
}

// variant 3: variant 2 with the evaluator's per-lane column coefficients
// (Kd, Ka, t/s and the column block index j per column, from global memory,
// held in registers) and a runtime xi test
template <bool SMEMC, bool RT = false>
__global__ void __launch_bounds__(256, 4)
    k_sterm_cols(int n, int terms, const int* __restrict__ rp, const int* __restrict__ ci,
                 const double* __restrict__ av, double* D0, double* D1, double* __restrict__ S,
                 double* __restrict__ Vw, const double* __restrict__ colKd,
                 const double* __restrict__ colKa, const double* __restrict__ colTos, int r,
                 double xi, unsigned long long* __restrict__ maxd, int ldb_rt = W, int g_rt = G) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int lane = threadIdx.x & 31;
  const int g = lane / G, q = lane % G;
  const int c = 2 * q;
  const int rows_per_warp = 32 / G;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const bool has_xi = xi != 0.0;
  double sigma = 1.0;
  for (int t = 0; t < terms; ++t) {
    const double* D = (t & 1) ? D1 : D0;
    double* Dn = (t & 1) ? D0 : D1;
    sigma *= double(t + 2);
    __shared__ double s_k[3][W];
    if (SMEMC && t == 0) {
      for (int k = threadIdx.x; k < W; k += blockDim.x) {
        s_k[0][k] = colKd[k];
        s_k[1][k] = colKa[k];
        s_k[2][k] = colTos[k];
      }
      __syncthreads();
    }
    int jj[2];
    double kd[2], ka[2], tos[2];
    if (!SMEMC)
      for (int e = 0; e < 2; ++e) {
        kd[e] = __ldg(colKd + c + e);
        ka[e] = __ldg(colKa + c + e);
        tos[e] = __ldg(colTos + c + e);
      }
    for (int e = 0; e < 2; ++e) jj[e] = (c + e) / r;
    unsigned long long m = 0;
    for (int base = warp_global * rows_per_warp; base < n; base += nwarps * rows_per_warp) {
      const int row = base + g;
      const bool ok = row < n;
      const unsigned LD = RT ? unsigned(ldb_rt) : unsigned(W);
      const unsigned o = unsigned(row) * LD + c;
      double2 vw = make_double2(0.0, 0.0), so = vw, ds = vw, vwl = vw;
      if (ok) {
        vw = __ldcs(reinterpret_cast<const double2*>(Vw + o));
        so = __ldcs(reinterpret_cast<const double2*>(S + o));
        if (has_xi) ds = *reinterpret_cast<const double2*>(D + o);
        if (jj[0] >= 2) vwl = __ldcs(reinterpret_cast<const double2*>(Vw + o - r));
      }
      double a0 = 0.0, a1 = 0.0;
      if (ok) {
        const int e1 = __ldg(rp + row + 1);
        for (int e = __ldg(rp + row); e < e1; ++e) {
          const double2 x = *reinterpret_cast<const double2*>(D + unsigned(__ldg(ci + e)) * LD + c);
          const double a = __ldg(av + e);
          a0 = a0 + a * x.x;
          a1 = a1 + a * x.y;
        }
      }
      if (SMEMC) {  // re-read per row from shared memory (volatile: not hoisted)
        const volatile double* vk = &s_k[0][0];
        for (int e = 0; e < 2; ++e) {
          kd[e] = vk[c + e];
          ka[e] = vk[W + c + e];
          tos[e] = vk[2 * W + c + e];
        }
      }
      double g0 = 0.0, g1 = 0.0;
      if (jj[0] >= 2) g0 = g0 + vwl.x * ka[0];
      g0 = g0 + vw.x * kd[0];
      if (jj[1] >= 2) g1 = g1 + vwl.y * ka[1];
      g1 = g1 + vw.y * kd[1];
      double y0 = a0, y1 = a1;
      if (has_xi) {
        y0 = y0 - xi * ds.x;
        y1 = y1 - xi * ds.y;
      }
      y0 = y0 * tos[0];
      y1 = y1 * tos[1];
      const double d0 = y0 + g0, d1 = y1 + g1;
      __syncwarp();
      if (ok) {
        __stcs(reinterpret_cast<double2*>(Vw + o), make_double2(g0, g1));
        *reinterpret_cast<double2*>(Dn + o) = make_double2(d0, d1);
        __stcs(reinterpret_cast<double2*>(S + o), make_double2(so.x + d0 / sigma, so.y + d1 / sigma));
      }
      double rs = ok ? fabs(d0) + fabs(d1) : 0.0;
      if (RT) {
#pragma unroll
        for (int k = 1; k < 32; k <<= 1)
          if (k < g_rt) rs = rs + __shfl_xor_sync(0xffffffffu, rs, k);
      } else {
        for (int k = 1; k < G; k <<= 1) rs += __shfl_xor_sync(0xffffffffu, rs, k);
      }
      const unsigned long long b = __double_as_longlong(rs);
      if (ok) m = b > m ? b : m;
    }
    for (int k = 16; k >= 1; k >>= 1) {
      const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, m, k);
      m = o2 > m ? o2 : m;
    }
    if (lane == 0) atomicMax(maxd + (t % 3), m);
    grid.sync();
    if (__longlong_as_double(static_cast<long long>(maxd[t % 3])) < 0.0) return;
  }
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
  {  // random block contents (argv[3] = 1), else zeros
    const bool rnd = argc > 3 && std::atoi(argv[3]) == 1;
    std::vector<double> h(nb);
    unsigned long long x = 88172645463325252ull;
    for (double* d : {D0, D1, S, Vw}) {
      for (size_t i = 0; i < nb; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        h[i] = rnd ? (double(x >> 11) * 0x1.0p-53 - 0.5) : 0.0;
      }
      CK(cudaMemcpy(d, h.data(), nb * 8, cudaMemcpyHostToDevice));
    }
  }
  int sms = 0, per = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  if (variant == 3 || variant == 4 || variant == 5) {
    auto kc = variant == 5 ? k_sterm_cols<true, true> : variant == 4 ? k_sterm_cols<true> : k_sterm_cols<false>;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kc, 256, 0));
    const int grid = sms * per;
    int terms = 29, r = 4;
    double xi = -2.0;
    std::vector<double> hk(W), ha(W), ht(W);
    for (int cc = 0; cc < W; ++cc) {
      hk[cc] = 0.9 - 0.01 * cc;
      ha[cc] = cc / r >= 2 ? 0.1 : 0.0;
      ht[cc] = 1e-4 * (1 + cc % r);
    }
    double *dk, *da, *dt;
    CK(cudaMalloc(&dk, W * 8));
    CK(cudaMalloc(&da, W * 8));
    CK(cudaMalloc(&dt, W * 8));
    CK(cudaMemcpy(dk, hk.data(), W * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(da, ha.data(), W * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dt, ht.data(), W * 8, cudaMemcpyHostToDevice));
    unsigned long long* dm3;
    CK(cudaMalloc(&dm3, 24));
    CK(cudaMemset(dm3, 0, 24));
    int ldb_rt = W, g_rt = G;
    void* args[] = {(void*)&n, (void*)&terms, (void*)&d_rp, (void*)&d_ci, (void*)&d_av,
                    (void*)&D0, (void*)&D1, (void*)&S, (void*)&Vw, (void*)&dk, (void*)&da,
                    (void*)&dt, (void*)&r, (void*)&xi, (void*)&dm3, (void*)&ldb_rt, (void*)&g_rt};
    for (int it = 0; it < 2; ++it)
      CK(cudaLaunchCooperativeKernel((void*)kc, grid, 256, args, 0, 0));
    cudaEvent_t a2, b2;
    CK(cudaEventCreate(&a2));
    CK(cudaEventCreate(&b2));
    CK(cudaEventRecord(a2));
    for (int it = 0; it < 5; ++it)
      CK(cudaLaunchCooperativeKernel((void*)kc, grid, 256, args, 0, 0));
    CK(cudaEventRecord(b2));
    CK(cudaEventSynchronize(b2));
    float ms2 = 0;
    CK(cudaEventElapsedTime(&ms2, a2, b2));
    const double per_term = ms2 / 5 / terms * 1e-3;
    const double bytes = 12.0 * double(nnz) + 4.0 * (n + 1) + 48.0 * W * double(n);
    std::printf("{\"variant\": \"persistent+columns%s\", \"grid\": %d, \"ctas_per_sm\": %d, "
                "\"us_per_term\": %.2f, \"alg_GBps\": %.1f, \"frac_of_6547.5\": %.3f}\n",
                variant == 5 ? " (smem, runtime ldb/G)" : variant == 4 ? " (smem)" : "", grid, per, per_term * 1e6, bytes / per_term / 1e9,
                bytes / per_term / 1e9 / 6547.5);
    return 0;
  }
  if (variant == 2) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sterm_persistent, 256, 0));
    const int grid = sms * per;
    int terms = 29;
    void* args[] = {(void*)&n, (void*)&terms, (void*)&d_rp, (void*)&d_ci, (void*)&d_av,
                    (void*)&D0, (void*)&D1, (void*)&S, (void*)&Vw, (void*)&d_m};
    unsigned long long* dm3;
    CK(cudaMalloc(&dm3, 24));
    CK(cudaMemset(dm3, 0, 24));
    args[9] = (void*)&dm3;
    for (int it = 0; it < 2; ++it)
      CK(cudaLaunchCooperativeKernel((void*)k_sterm_persistent, grid, 256, args, 0, 0));
    cudaEvent_t a2, b2;
    CK(cudaEventCreate(&a2));
    CK(cudaEventCreate(&b2));
    CK(cudaEventRecord(a2));
    for (int it = 0; it < 5; ++it)
      CK(cudaLaunchCooperativeKernel((void*)k_sterm_persistent, grid, 256, args, 0, 0));
    CK(cudaEventRecord(b2));
    CK(cudaEventSynchronize(b2));
    float ms2 = 0;
    CK(cudaEventElapsedTime(&ms2, a2, b2));
    const double per_term = ms2 / 5 / terms * 1e-3;
    const double bytes = 12.0 * double(nnz) + 4.0 * (n + 1) + 48.0 * W * double(n);
    std::printf("{\"variant\": \"persistent+grid.sync\", \"grid\": %d, \"ctas_per_sm\": %d, "
                "\"us_per_term\": %.2f, \"alg_GBps\": %.1f, \"frac_of_6547.5\": %.3f}\n",
                grid, per, per_term * 1e6, bytes / per_term / 1e9, bytes / per_term / 1e9 / 6547.5);
    return 0;
  }
  auto kfn = variant ? k_sterm<true> : k_sterm<false>;
  // optional unused dynamic shared memory per CTA (KB): the evaluator holds
  // ~37 KB of pipes per CTA, which shrinks the L1 the gathers hit
  const int smem_kb = argc > 2 ? std::atoi(argv[2]) : 0;
  const size_t smem = size_t(smem_kb) * 1024;
  if (smem) CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kfn, 256, smem));
  const int grid = sms * per;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int iters = 40;
  for (int it = 0; it < 5; ++it)
    kfn<<<grid, 256, smem>>>(n, d_rp, d_ci, d_av, it & 1 ? D1 : D0, it & 1 ? D0 : D1, S, Vw, 0.9,
                             0.1, 1e-4, -2.0, 2.0, d_m);
  CK(cudaEventRecord(a));
  for (int it = 0; it < iters; ++it)
    kfn<<<grid, 256, smem>>>(n, d_rp, d_ci, d_av, it & 1 ? D1 : D0, it & 1 ? D0 : D1, S, Vw, 0.9,
                             0.1, 1e-4, -2.0, 2.0, d_m);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  const double per_term = ms / iters * 1e-3;
  const double bytes = 12.0 * double(nnz) + 4.0 * (n + 1) + 48.0 * W * double(n);
  std::printf("{\"variant\": \"%s\", \"smem_kb\": %d, \"grid\": %d, \"ctas_per_sm\": %d, \"us_per_term\": %.2f, "
              "\"alg_GBps\": %.1f, \"frac_of_6547.5\": %.3f}\n",
              variant ? "serial" : "batched", smem_kb, grid, per, per_term * 1e6, bytes / per_term / 1e9,
              bytes / per_term / 1e9 / 6547.5);
  return 0;
}
