// sm_100a kernels of parameter selection (params.cpp:81-239): CSR SpMV with
// fused chunk maxima, the objective GEMV, canonical chunk sums of squares for
// Eigen's stableNorm, column scaling; plus the column-major CSR apply of the
// C ABI.  The evaluator kernel lives in phx_eval.cu.
//
// Compiled with --fmad=false: every multiply and add is individually rounded
// (the reference's numerical contract); reductions follow the canonical
// orders of oracle/phx_oracle.cpp and DESIGN.md §3.
#include <algorithm>
#include <atomic>
#include <cmath>

#include "phx_kernels.cuh"

namespace phx {

static std::atomic<int64_t> g_launches{0};
int64_t kernel_launch_count() { return g_launches.load(); }
void count_launch() { ++g_launches; }

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kBlock = 256;

__device__ __forceinline__ unsigned long long abs_bits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7FFFFFFFFFFFFFFFull;
}
__device__ __forceinline__ double from_bits(unsigned long long b) {
  return __longlong_as_double(static_cast<long long>(b));
}
__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

// ---------------------------------------------------------------------------
// Parameter-selection kernels: one CTA of 256 threads per 4096-row chunk.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void store_chunkmax(unsigned long long m,
                                               unsigned long long* chunkmax) {
  __shared__ unsigned long long red[kBlock / 32];
  for (int s = 16; s >= 1; s >>= 1) m = umax64(m, __shfl_xor_sync(kFull, m, s));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long mm = 0;
    for (int q = 0; q < kBlock / 32; ++q) mm = umax64(mm, red[q]);
    chunkmax[blockIdx.x] = mm;
  }
}

__global__ void __launch_bounds__(kBlock)
    k_spmv(int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
           const double* __restrict__ av, const double* __restrict__ x, double* __restrict__ y,
           int mode, double xi, double div, unsigned long long* chunkmax) {
  const int base = blockIdx.x * kChunk;
  unsigned long long m = 0;
  for (int q = 0; q < kChunk / kBlock; ++q) {
    const int row = base + threadIdx.x + q * kBlock;
    if (row >= n) break;
    const int e0 = __ldg(rp + row), e1 = __ldg(rp + row + 1);
    double acc = 0.0;
    int e = e0;
    for (; e + 4 <= e1; e += 4) {
      const int c0 = __ldg(ci + e), c1 = __ldg(ci + e + 1), c2 = __ldg(ci + e + 2),
                c3 = __ldg(ci + e + 3);
      const double a0 = __ldg(av + e), a1 = __ldg(av + e + 1), a2 = __ldg(av + e + 2),
                   a3 = __ldg(av + e + 3);
      const double x0 = __ldg(x + c0), x1 = __ldg(x + c1), x2 = __ldg(x + c2), x3 = __ldg(x + c3);
      acc = acc + a0 * x0;
      acc = acc + a1 * x1;
      acc = acc + a2 * x2;
      acc = acc + a3 * x3;
    }
    for (; e < e1; ++e) acc = acc + __ldg(av + e) * __ldg(x + __ldg(ci + e));
    double v = acc;
    if (mode == 1) v = v - xi * __ldg(x + row);
    else if (mode == 2) v = v / div;
    y[row] = v;
    m = umax64(m, abs_bits(v));
  }
  if (chunkmax) store_chunkmax(m, chunkmax);
}

__global__ void __launch_bounds__(kBlock)
    k_gemv(int32_t n, int32_t ncol, const double* __restrict__ B, const double* __restrict__ c,
           double* __restrict__ y, unsigned long long* chunkmax) {
  __shared__ double cs[128];
  for (int j = threadIdx.x; j < ncol; j += blockDim.x) cs[j] = c[j];
  __syncthreads();
  const int base = blockIdx.x * kChunk;
  unsigned long long m = 0;
  for (int q = 0; q < kChunk / kBlock; ++q) {
    const int row = base + threadIdx.x + q * kBlock;
    if (row >= n) break;
    double acc = 0.0;
    const double* b = B + row;
    int j = 0;
    for (; j + 8 <= ncol; j += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(b + size_t(j + u) * size_t(n));
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = acc + v[u] * cs[j + u];
    }
    for (; j < ncol; ++j) acc = acc + __ldg(b + size_t(j) * size_t(n)) * cs[j];
    y[row] = acc;
    m = umax64(m, abs_bits(acc));
  }
  if (chunkmax) store_chunkmax(m, chunkmax);
}

__global__ void __launch_bounds__(kBlock)
    k_chunkmax(int32_t n, const double* __restrict__ x, unsigned long long* chunkmax) {
  const int base = blockIdx.x * kChunk;
  unsigned long long m = 0;
  for (int q = 0; q < kChunk / kBlock; ++q) {
    const int row = base + threadIdx.x + q * kBlock;
    if (row >= n) break;
    m = umax64(m, abs_bits(x[row]));
  }
  store_chunkmax(m, chunkmax);
}

// canonical chunk sum of squares: lane l sums x[l + 256 q] sequentially from
// +0, lanes combined by a pairwise tree (butterfly within warps, then a
// pairwise tree over the 8 warp sums)
__global__ void __launch_bounds__(kBlock)
    k_chunk_ssq(int32_t n, const double* __restrict__ x, const double* __restrict__ inv,
                double* __restrict__ partial) {
  __shared__ double red[kBlock / 32];
  const int base = blockIdx.x * kChunk;
  const double mul = inv[blockIdx.x];
  double s = 0.0;
  for (int q = 0; q < kChunk / kBlock; ++q) {
    const int idx = base + threadIdx.x + q * kBlock;
    if (idx < n) {
      const double v = x[idx] * mul;
      s = s + v * v;
    }
  }
  for (int m = 1; m < 32; m <<= 1) s = s + __shfl_xor_sync(kFull, s, m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double w[kBlock / 32];
    for (int q = 0; q < kBlock / 32; ++q) w[q] = red[q];
    for (int h = 1; h < kBlock / 32; h <<= 1)
      for (int q = 0; q < kBlock / 32; q += 2 * h) w[q] = w[q] + w[q + h];
    partial[blockIdx.x] = w[0];
  }
}

__global__ void k_scale(int32_t n, double* __restrict__ x, double s, int mode) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[i] = mode == 0 ? x[i] * s : x[i] / s;
}

__global__ void k_spmm_cols(int32_t n, int32_t k, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ ci, const double* __restrict__ av,
                            const double* __restrict__ X, double* __restrict__ Y, int mode,
                            double xi) {
  const size_t total = size_t(n) * size_t(k);
  for (size_t id = size_t(blockIdx.x) * blockDim.x + threadIdx.x; id < total;
       id += size_t(gridDim.x) * blockDim.x) {
    const int row = int(id % size_t(n));
    const size_t c = id / size_t(n);
    const double* xc = X + c * size_t(n);
    double acc = 0.0;
    for (int e = __ldg(rp + row); e < __ldg(rp + row + 1); ++e)
      acc = acc + __ldg(av + e) * xc[__ldg(ci + e)];
    if (mode == 1 && xi != 0.0) acc = acc - xi * xc[row];
    Y[c * size_t(n) + row] = acc;
  }
}

int nchunks(int32_t n) { return (n + kChunk - 1) / kChunk; }

}  // namespace

cudaError_t launch_spmv(int32_t n, const int32_t* rp, const int32_t* ci, const double* av,
                        const double* x, double* y, int mode, double xi, double div,
                        unsigned long long* chunkmax, cudaStream_t st) {
  ++g_launches;
  k_spmv<<<nchunks(n), kBlock, 0, st>>>(n, rp, ci, av, x, y, mode, xi, div, chunkmax);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// expRK4s6 stage kernels (integrator.cpp:29-105): elementwise, one thread per
// row, the reference's Eigen expression order (left-associative, no FMA).
// V blocks are column-major n x (p+1) with leading dimension n; column 0 is
// zero in every call (the scheme has no phi_0 term).
__device__ __forceinline__ double rk_reaction(double gamma, double u) {
  return gamma * u * (u - 0.5) * (1.0 - u);  // problems.cpp ADRProblem::reaction
}

__global__ void __launch_bounds__(kBlock)
    k_rk_stage(RkStageArgs a) {
  const int64_t n = a.n;
  for (int64_t i = int64_t(blockIdx.x) * kBlock + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * kBlock) {
    const double ui = a.u[i];
    double* V = a.V;
    switch (a.mode) {
      case 0: {  // g_n = r(u); f_n = A u + g_n; hf = h f_n; V2 = [0, c2 hf]
        double acc = 0.0;
        for (int e = __ldg(a.rp + i), e1 = __ldg(a.rp + i + 1); e < e1; ++e)
          acc = acc + __ldg(a.av + e) * a.u[__ldg(a.ci + e)];
        const double g = rk_reaction(a.gamma, ui);
        const double hf = a.h * (acc + g);
        a.gn[i] = g;
        a.hf[i] = hf;
        V[i] = 0.0;
        V[n + i] = a.s0 * hf;
        break;
      }
      case 1: {  // u2 = u + U; d2 = r(u2) - g_n; V34 = [0, hf, (h/c2) d2]
        const double u2 = ui + a.W[i];
        const double d2 = rk_reaction(a.gamma, u2) - a.gn[i];
        V[i] = 0.0;
        V[n + i] = a.hf[i];
        V[2 * n + i] = a.s0 * d2;
        break;
      }
      case 2: {  // two stages (ca, cb): V = [0, hf, A(B da + C db), D(da/ca - db/cb)]
        const double ua = ui + a.W[i], ub = ui + a.W[n + i];
        const double da = rk_reaction(a.gamma, ua) - a.gn[i];
        const double db = rk_reaction(a.gamma, ub) - a.gn[i];
        V[i] = 0.0;
        V[n + i] = a.hf[i];
        V[2 * n + i] = a.s0 * (a.s1 * da + a.s2 * db);
        V[3 * n + i] = a.s3 * (da / a.ca - db / a.cb);
        break;
      }
      default: {  // u_next = u + U; flag a non-finite entry
        const double un = ui + a.W[i];
        a.out[i] = un;
        if (!isfinite(un)) atomicOr(a.flag, 1);
        break;
      }
    }
  }
}

cudaError_t launch_rk_stage(const RkStageArgs& a, cudaStream_t st) {
  ++g_launches;
  const int64_t blocks = (a.n + kBlock - 1) / kBlock;
  const int grid = int(std::min<int64_t>(blocks, 148 * 16));
  k_rk_stage<<<grid, kBlock, 0, st>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// block_series_direct term (phi_block.cpp:186-209): one thread per row;
// term(i,k) = (sum_q X(i,q) M(q,k) from +0, ascending q) * tpow_k,
// G(i,k) += term(i,k); the canonical |.| row sums of term and G (pairwise
// tree over pow2-padded columns) max-reduced into slots[0], slots[1].
__global__ void __launch_bounds__(kBlock)
    k_series_term(int32_t n, int32_t p1, int32_t r, const double* __restrict__ X,
                  const double* __restrict__ M, const double* __restrict__ tpow, double* G,
                  unsigned long long* slots) {
  unsigned long long mt = 0, mg = 0;
  int len = 1;
  while (len < r) len <<= 1;
  for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
    double ta[kSeriesMaxR], ga[kSeriesMaxR];
    for (int k = 0; k < len; ++k) {
      if (k < r) {
        double acc = 0.0;
        for (int q = 0; q < p1; ++q) acc = acc + X[i + size_t(q) * n] * M[q + k * p1];
        acc = acc * tpow[k];
        const double g = G[i + size_t(k) * n] + acc;
        G[i + size_t(k) * n] = g;
        ta[k] = fabs(acc);
        ga[k] = fabs(g);
      } else {
        ta[k] = ga[k] = 0.0;
      }
    }
    for (int h = 1; h < len; h <<= 1)
      for (int l = 0; l < len; l += 2 * h) {
        ta[l] = ta[l] + ta[l + h];
        ga[l] = ga[l] + ga[l + h];
      }
    mt = umax64(mt, abs_bits(ta[0]));
    mg = umax64(mg, abs_bits(ga[0]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    mt = umax64(mt, __shfl_xor_sync(0xffffffffu, mt, o));
    mg = umax64(mg, __shfl_xor_sync(0xffffffffu, mg, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(slots, mt);
    atomicMax(slots + 1, mg);
  }
}

cudaError_t launch_series_term(int32_t n, int32_t p1, int32_t r, const double* X, const double* M,
                               const double* tpow, double* G, unsigned long long* slots,
                               cudaStream_t st) {
  if (r > kSeriesMaxR) return cudaErrorInvalidValue;
  ++g_launches;
  const int grid = std::max(1, std::min(148 * 8, (n + kBlock - 1) / kBlock));
  k_series_term<<<grid, kBlock, 0, st>>>(n, p1, r, X, M, tpow, G, slots);
  return cudaGetLastError();
}

cudaError_t launch_gemv(int32_t n, int32_t ncol, const double* B, const double* c, double* y,
                        unsigned long long* chunkmax, cudaStream_t st) {
  if (ncol > 128) return cudaErrorInvalidValue;
  ++g_launches;
  k_gemv<<<nchunks(n), kBlock, 0, st>>>(n, ncol, B, c, y, chunkmax);
  return cudaGetLastError();
}

cudaError_t launch_chunkmax(int32_t n, const double* x, unsigned long long* chunkmax,
                            cudaStream_t st) {
  ++g_launches;
  k_chunkmax<<<nchunks(n), kBlock, 0, st>>>(n, x, chunkmax);
  return cudaGetLastError();
}

cudaError_t launch_chunk_ssq(int32_t n, const double* x, const double* inv, double* partial,
                             cudaStream_t st) {
  ++g_launches;
  k_chunk_ssq<<<nchunks(n), kBlock, 0, st>>>(n, x, inv, partial);
  return cudaGetLastError();
}

cudaError_t launch_scale(int32_t n, double* x, double s, int mode, cudaStream_t st) {
  ++g_launches;
  const int grid = std::min(4096, (n + kBlock - 1) / kBlock);
  k_scale<<<grid, kBlock, 0, st>>>(n, x, s, mode);
  return cudaGetLastError();
}

// stableNorm's per-chunk invScale on the device, in parallel.  Eigen's
// sequential block-scale update (scale / invScale, with its NaN, overflow and
// tiny-maximum branches; restated on the host in stable_norm_dev) leaves
// after chunk b: scale_b = the running maximum of F(x_j) = max(x_j, 1/DBL_MAX)
// over the chunks j <= b with a positive maximum x_j before the first NaN
// chunk (0 if none), and invScale_b = G(scale_b): 1 for 0 or inf, else
// fl(1/scale_b) capped at DBL_MAX; after the first NaN chunk invScale no
// longer changes.  (Checked against the sequential update on 2e5 random
// sequences of zeros, subnormals, 1/DBL_MAX, normals, DBL_MAX, inf and NaN.)
// One CTA: the first NaN chunk by a min-reduction, then an inclusive max-scan
// of the masked keys (non-negative doubles order as their bit patterns).
constexpr int kInvBlock = 1024;
__global__ void __launch_bounds__(kInvBlock)
    k_stable_inv(int32_t nch, const unsigned long long* __restrict__ chunkmax, double* __restrict__ inv) {
  __shared__ int s_first;
  __shared__ unsigned long long s_w[kInvBlock / 32];
  __shared__ unsigned long long s_carry;
  const double dmax = 1.7976931348623157e308;
  const unsigned long long tiny = static_cast<unsigned long long>(__double_as_longlong(1.0 / dmax));
  const unsigned long long infb = 0x7FF0000000000000ull;
  if (threadIdx.x == 0) {
    s_first = nch;
    s_carry = 0ull;
  }
  __syncthreads();
  int first = nch;
  for (int b = threadIdx.x; b < nch; b += blockDim.x)
    if (chunkmax[b] > infb) first = min(first, b);
  atomicMin(&s_first, first);
  __syncthreads();
  first = s_first;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int p0 = 0; p0 < nch; p0 += kInvBlock) {
    const int b = p0 + int(threadIdx.x);
    unsigned long long key = 0ull;
    if (b < nch && b < first) {
      const unsigned long long x = chunkmax[b];
      if (x != 0ull) key = x > tiny ? x : tiny;  // F(x) = max(x, 1/DBL_MAX)
    }
    for (int o = 1; o < 32; o <<= 1) {  // warp inclusive max-scan
      const unsigned long long y = __shfl_up_sync(kFull, key, o);
      if (lane >= o) key = key > y ? key : y;
    }
    if (lane == 31) s_w[wid] = key;
    __syncthreads();
    if (wid == 0) {
      unsigned long long v = s_w[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v = v > y ? v : y;
      }
      s_w[lane] = v;
    }
    __syncthreads();
    unsigned long long sc = key;
    if (wid > 0) sc = sc > s_w[wid - 1] ? sc : s_w[wid - 1];
    sc = sc > s_carry ? sc : s_carry;
    if (b < nch) {
      double g = 1.0;
      if (sc != 0ull && sc != infb) {
        const double t = 1.0 / __longlong_as_double(static_cast<long long>(sc));
        g = t > dmax ? dmax : t;
      }
      inv[b] = g;
    }
    __syncthreads();
    if (threadIdx.x == kInvBlock - 1) s_carry = sc;  // the piece's last (inclusive) value
    __syncthreads();
  }
}

cudaError_t launch_stable_inv(int32_t nch, const unsigned long long* chunkmax, double* inv,
                              cudaStream_t st) {
  ++g_launches;
  k_stable_inv<<<1, kInvBlock, 0, st>>>(nch, chunkmax, inv);
  return cudaGetLastError();
}

cudaError_t launch_spmm_cols(int32_t n, int32_t k, const int32_t* rp, const int32_t* ci,
                             const double* av, const double* X, double* Y, int mode, double xi,
                             cudaStream_t st) {
  ++g_launches;
  const size_t total = size_t(n) * size_t(k);
  const int grid = int(std::min<size_t>(8192, (total + kBlock - 1) / kBlock));
  k_spmm_cols<<<grid, kBlock, 0, st>>>(n, k, rp, ci, av, X, Y, mode, xi);
  return cudaGetLastError();
}

}  // namespace phx
