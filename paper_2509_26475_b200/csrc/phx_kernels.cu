// sm_100a kernels of the phi-combination engine.
//
// Compiled with --fmad=false: every multiply and add is individually rounded,
// which is the numerical contract of the reference (a baseline x86-64 Eigen
// build has no FMA) and of the oracle.  All reductions follow the canonical
// orders documented in oracle/phx_oracle.cpp and DESIGN.md §3, so the device
// path reproduces the oracle bit for bit.
//
// Hot kernel: k_phimv_block, ONE persistent cooperative launch per
// phimv_block call (phi_block.cpp:48-157).  Every Taylor term is a grid step:
// each row group (GS or GF lanes of a warp) gathers the CSR row's block rows
// (row-interleaved, one coalesced load per gathered row), fuses the shift,
// scaling, J-term, accumulator updates and both |.| row sums, and publishes a
// per-CTA max with one atomicMax; after grid.sync() every CTA reads the two
// maxima and takes the same stopping decision, so the loop control never
// leaves the device.
#include <cooperative_groups.h>

#include <atomic>
#include <cmath>

#include "phx_kernels.cuh"

namespace cg = cooperative_groups;

namespace phx {

static std::atomic<int64_t> g_launches{0};
int64_t kernel_launch_count() { return g_launches.load(); }

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

// Canonical row sum of |x| over one row held by a G-lane group (Q columns
// per lane, column c = lg + G*q): pairwise tree in natural column order
// padded to a power of two.  Lanes holding no column pass 0.
template <int Q>
__device__ __forceinline__ double group_rowsum(const double (&v)[Q], int G, int qp) {
  double T[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    double x = v[q];
    for (int m = 1; m < G; m <<= 1) x = x + __shfl_xor_sync(kFull, x, m);
    T[q] = x;
  }
  // qp = power-of-two count of column chunks (1 when the row fits in G lanes)
#pragma unroll
  for (int h = 1; h < Q; h <<= 1) {
    if (h < qp) {
#pragma unroll
      for (int q = 0; q + h < Q; q += 2 * h) T[q] = T[q] + T[q + h];
    }
  }
  return T[0];
}

// CTA-wide max of two bit patterns -> one atomicMax each into slot s.
__device__ __forceinline__ void publish2(unsigned long long a, unsigned long long b,
                                         unsigned long long* slot,
                                         unsigned long long (*red)[kBlock / 32]) {
  for (int m = 16; m >= 1; m >>= 1) {
    a = umax64(a, __shfl_xor_sync(kFull, a, m));
    b = umax64(b, __shfl_xor_sync(kFull, b, m));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][warp] = a;
    red[1][warp] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ma = 0, mb = 0;
    for (int q = 0; q < int(blockDim.x >> 5); ++q) {
      ma = umax64(ma, red[0][q]);
      mb = umax64(mb, red[1][q]);
    }
    atomicMax(slot, ma);
    atomicMax(slot + 1, mb);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Warp tiles.  A warp processes RW = (32/G)*R consecutive rows at a time:
// lane group g = lane/G (G lanes per row, Q columns per lane), R rows per
// group (row = base + rr*(32/G) + g, so for each rr the warp's groups cover
// consecutive rows and every block-row load is one contiguous segment).  The
// warp tile's CSR slice is staged once in warp-private shared memory with
// coalesced loads (row_ptr, then the contiguous entry range); tiles whose
// slice exceeds the staging capacity read the entries from global memory.
// ---------------------------------------------------------------------------
constexpr int kWarps = kBlock / 32;
constexpr int kWCap = 256;   // staged CSR entries per warp
constexpr int kMaxRW = 64;   // rows per warp tile

struct WarpStage {
  int rp[kMaxRW + 1];
  int ci[kWCap];
  double av[kWCap];
};

struct TileCsr {
  const int* ci;
  const double* av;
  int e_lo;
};

// Stage the CSR slice of rows [base, base+RW) (rows past n are empty).
__device__ __forceinline__ TileCsr stage_csr(const BlockArgs& a, int base, int RW,
                                             WarpStage& st, int lane) {
  __syncwarp();  // every lane is done with the previous tile's slice
  for (int l = lane; l <= RW; l += 32) st.rp[l] = __ldg(a.rp + min(base + l, a.n));
  __syncwarp();
  TileCsr tc;
  tc.e_lo = st.rp[0];
  const int E = st.rp[RW] - tc.e_lo;
  if (E <= kWCap) {
    for (int e = lane; e < E; e += 32) {
      st.ci[e] = __ldg(a.ci + tc.e_lo + e);
      st.av[e] = __ldg(a.av + tc.e_lo + e);
    }
    tc.ci = st.ci;
    tc.av = st.av;
  } else {
    tc.ci = a.ci + tc.e_lo;
    tc.av = a.av + tc.e_lo;
  }
  __syncwarp();
  return tc;
}

// acc[rr][q] = sum over row rr's entries, in storage order from +0, of
// av[e] * X[ci[e]*ld + c_q].  Gathers are plain (L1-cached) loads: X was
// written before the last grid.sync(), which invalidates L1 (CCTL.IVALL).
template <int Q, int R, int B>
__device__ __forceinline__ void gather_tile(const TileCsr& tc, const int (&rs)[R],
                                            const int (&cnt)[R], const double* X, int ld,
                                            const int (&cq)[Q], const bool (&vq)[Q],
                                            double (&acc)[R][Q]) {
  int maxc = 0;
#pragma unroll
  for (int rr = 0; rr < R; ++rr) maxc = max(maxc, cnt[rr]);
  for (int u0 = 0; u0 < maxc; u0 += B) {
    double xv[B][R][Q];
#pragma unroll
    for (int u = 0; u < B; ++u)
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        const bool ok = u0 + u < cnt[rr];
        const int col = ok ? tc.ci[rs[rr] + u0 + u] : 0;
#pragma unroll
        for (int q = 0; q < Q; ++q)
          xv[u][rr][q] = (ok && vq[q]) ? X[size_t(col) * size_t(ld) + cq[q]] : 0.0;
      }
#pragma unroll
    for (int u = 0; u < B; ++u)
#pragma unroll
      for (int rr = 0; rr < R; ++rr)
        if (u0 + u < cnt[rr]) {
          const double av = tc.av[rs[rr] + u0 + u];
#pragma unroll
          for (int q = 0; q < Q; ++q) acc[rr][q] = acc[rr][q] + av * xv[u][rr][q];
        }
  }
}

template <int Q>
struct Tr {  // rows per group per warp tile, gather batch
  static constexpr int R = Q == 1 ? 2 : 1;
  static constexpr int B = Q == 1 ? 4 : (Q == 2 ? 4 : 2);
};

struct Layout {
  int G, gpw, g, lg, RW, qn, qp, width;
};

__device__ __forceinline__ Layout make_layout(int G, int qn, int width, int R) {
  Layout L;
  const int lane = threadIdx.x & 31;
  L.G = G;
  L.gpw = 32 / G;
  L.g = lane / G;
  L.lg = lane % G;
  L.RW = L.gpw * R;
  L.qn = qn;
  L.width = width;
  // power-of-two count of 32-column chunks (1 when the row fits in G lanes)
  int chunks = (width + 31) / 32;
  int qp = 1;
  while (qp < chunks) qp <<= 1;
  L.qp = width > 32 ? qp : 1;
  return L;
}

// Persistent evaluator.  See the file header.
template <int Q>
__global__ void __launch_bounds__(kBlock, 3) k_phimv_block(BlockArgs a) {
  constexpr int R = Tr<Q>::R;
  constexpr int B = Tr<Q>::B;
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long red[2][kWarps];
  __shared__ WarpStage stage[kWarps];
  const double INF = __longlong_as_double(0x7FF0000000000000ll);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpStage& st = stage[warp];

  const int n = a.n, r = a.r, p = a.p, ldb = a.ldb, ldf = a.ldf;
  const int ntiles = (n + a.tile - 1) / a.tile;
  const bool has_xi = a.xi != 0.0;
  const bool master = blockIdx.x == 0 && threadIdx.x == 0;
  const Layout LS = make_layout(a.GS, a.QS, a.w, R);
  const Layout LF = make_layout(a.GF, a.QF, a.fcols, R);

  int step = 0;
  int tr_len = 0;
  auto trace = [&](double kind, double x, double y) {
    if (master && a.trace != nullptr && tr_len + 3 <= a.trace_cap) {
      a.trace[tr_len] = kind;
      a.trace[tr_len + 1] = x;
      a.trace[tr_len + 2] = y;
    }
    tr_len += 3;
  };
  // publish this CTA's maxima for the current step, zero the slot of the next
  // step (its last readers finished before the previous grid sync),
  // grid-sync, read the global maxima.
  auto sync_step = [&](unsigned long long ma, unsigned long long mb, double& ra, double& rb) {
    unsigned long long* slot = a.slots + 2 * (step % 3);
    publish2(ma, mb, slot, red);
    if (master) {
      unsigned long long* nxt = a.slots + 2 * ((step + 1) % 3);
      nxt[0] = 0ull;
      nxt[1] = 0ull;
    }
    grid.sync();
    ra = from_bits(__ldcg(reinterpret_cast<const unsigned long long*>(slot)));
    rb = from_bits(__ldcg(reinterpret_cast<const unsigned long long*>(slot + 1)));
    ++step;
  };
  auto finish = [&](int err, int idx, int L_S, int extra_steps) {
    if (master) {
      a.status[0] = err;
      a.status[1] = idx;
      a.status[2] = L_S;
      a.status[3] = 0;
      a.status[4] = step + extra_steps;
      a.status[5] = min(tr_len, a.trace_cap);
    }
  };

  // per-lane column bookkeeping of a layout (recomputed per phase)
  auto cols = [&](const Layout& L, int (&c)[Q], bool (&v)[Q]) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      c[q] = L.lg + L.G * q;
      v[q] = (q < L.qn) && (c[q] < L.width);
    }
  };

  // ================= init: Vw = V[src]*g, D = S = Vw (phi_block.cpp:76-92)
  unsigned long long m0 = 0;
  {
    int c[Q];
    bool v[Q];
    cols(LS, c, v);
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int wt = warp; wt < a.tile / LS.RW; wt += kWarps) {
        const int base = t * a.tile + wt * LS.RW;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int row = base + rr * LS.gpw + LS.g;
          const bool rv = row < n;
          double x[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            x[q] = 0.0;
            if (rv && v[q]) {
              const int j = c[q] / r, i = c[q] - j * r;
              const int src = j == 0 ? 0 : p + 1 - j;
              x[q] = __ldg(a.V + size_t(src) * size_t(n) + row) * __ldg(a.g + i);
              const size_t o = size_t(row) * size_t(ldb) + c[q];
              a.Vw[o] = x[q];
              a.D0[o] = x[q];
              a.S[o] = x[q];
            }
            x[q] = fabs(x[q]);
          }
          const double rsum = group_rowsum<Q>(x, LS.G, LS.qp);
          if (rv) m0 = umax64(m0, abs_bits(rsum));
        }
      }
  }
  double mD, mSn;
  sync_step(m0, m0, mD, mSn);
  double c1 = INF, c2 = mD, nS = mSn;  // c2 = inf_norm(D), ||S|| at k = 1
  trace(0.0, c2, nS);

  // ================= S series (phi_block.cpp:93-106)
  int k = 1;
  double sigma = 1.0;
  double* Dc = a.D0;
  double* Dn = a.D1;
  int err = kStOk, err_idx = 0;
  while (c1 + c2 > a.tol * nS) {
    if (k >= 500) {
      err = kStSeriesCap;
      err_idx = 500;
      break;
    }
    ++k;
    c1 = c2;
    sigma *= k;
    unsigned long long mdb = 0, msb = 0;
    {
      int c[Q], jj[Q];
      bool v[Q];
      double kd[Q], ka[Q], tos[Q];
      cols(LS, c, v);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        jj[q] = v[q] ? c[q] / r : 0;
        kd[q] = v[q] ? __ldg(a.colKd + c[q]) : 0.0;
        ka[q] = v[q] ? __ldg(a.colKa + c[q]) : 0.0;
        tos[q] = v[q] ? __ldg(a.colTos + c[q]) : 0.0;
      }
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int wt = warp; wt < a.tile / LS.RW; wt += kWarps) {
          const int base = t * a.tile + wt * LS.RW;
          // row-local streams first (independent of the CSR slice)
          double vw[R][Q], vwl[R][Q], so[R][Q], ds[R][Q], acc[R][Q];
          bool vq[R][Q];
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const int row = base + rr * LS.gpw + LS.g;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              vq[rr][q] = row < n && v[q];
              const size_t o = size_t(row) * size_t(ldb) + c[q];
              vw[rr][q] = vq[rr][q] ? a.Vw[o] : 0.0;
              vwl[rr][q] = (vq[rr][q] && jj[q] >= 2) ? a.Vw[o - r] : 0.0;
              so[rr][q] = vq[rr][q] ? a.S[o] : 0.0;
              ds[rr][q] = (vq[rr][q] && has_xi) ? Dc[o] : 0.0;
              acc[rr][q] = 0.0;
            }
          }
          const TileCsr tc = stage_csr(a, base, LS.RW, st, lane);
          int rs[R], cnt[R];
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const int li = rr * LS.gpw + LS.g;
            rs[rr] = st.rp[li] - tc.e_lo;
            cnt[rr] = st.rp[li + 1] - st.rp[li];
          }
          gather_tile<Q, R, B>(tc, rs, cnt, Dc, ldb, c, v, acc);
          double vn[R][Q], dn[R][Q], sn[R][Q];
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              // Vw = Vw * Kiter: ascending source column from +0 (:98)
              double g2 = 0.0;
              if (jj[q] >= 2) g2 = g2 + vwl[rr][q] * ka[q];
              g2 = g2 + vw[rr][q] * kd[q];
              vn[rr][q] = g2;
              // D = (A - xi I) D (:99), * t_i/s (:101), + Vw (:102)
              double y = acc[rr][q];
              if (has_xi) y = y - a.xi * ds[rr][q];
              y = y * tos[q];
              dn[rr][q] = y + g2;
              sn[rr][q] = so[rr][q] + dn[rr][q] / sigma;  // S += D/sigma (:105)
            }
          __syncwarp();
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const int row = base + rr * LS.gpw + LS.g;
            double ad[Q], as[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              if (vq[rr][q]) {
                const size_t o = size_t(row) * size_t(ldb) + c[q];
                a.Vw[o] = vn[rr][q];
                Dn[o] = dn[rr][q];
                a.S[o] = sn[rr][q];
              }
              ad[q] = vq[rr][q] ? fabs(dn[rr][q]) : 0.0;
              as[q] = vq[rr][q] ? fabs(sn[rr][q]) : 0.0;
            }
            const double rd = group_rowsum<Q>(ad, LS.G, LS.qp);
            const double rsm = group_rowsum<Q>(as, LS.G, LS.qp);
            if (row < n) {
              mdb = umax64(mdb, abs_bits(rd));
              msb = umax64(msb, abs_bits(rsm));
            }
          }
        }
    }
    double maxD, maxS;
    sync_step(mdb, msb, maxD, maxS);
    c2 = maxD / sigma;  // :103
    if (!isfinite(c2)) {
      err = kStSeriesDiverged;
      err_idx = k;
      break;
    }
    nS = maxS;
    trace(1.0, c2, nS);
    double* tmp = Dc;
    Dc = Dn;
    Dn = tmp;
  }
  const int L_S = k;
  if (err != kStOk) {
    finish(err, err_idx, L_S, 0);
    return;
  }

  // ================= promotion (phi_block.cpp:109-120)
  // F_L = fl(fl(A S_L * t_i) + v0) (unshifted A), F_R = S block p.
  double* Fc = a.F0;
  double* Fn = a.F1;
  const bool sweeps = a.s_eff > 1;
  unsigned long long mf = 0;
  {
    int c[Q];
    bool v[Q], vl[Q];
    cols(LF, c, v);
#pragma unroll
    for (int q = 0; q < Q; ++q) vl[q] = v[q] && c[q] < r;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int wt = warp; wt < a.tile / LF.RW; wt += kWarps) {
        const int base = t * a.tile + wt * LF.RW;
        double acc[R][Q];
#pragma unroll
        for (int rr = 0; rr < R; ++rr)
#pragma unroll
          for (int q = 0; q < Q; ++q) acc[rr][q] = 0.0;
        const TileCsr tc = stage_csr(a, base, LF.RW, st, lane);
        int rs[R], cnt[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int li = rr * LF.gpw + LF.g;
          rs[rr] = st.rp[li] - tc.e_lo;
          cnt[rr] = st.rp[li + 1] - st.rp[li];
        }
        gather_tile<Q, R, B>(tc, rs, cnt, a.S, ldb, c, vl, acc);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int row = base + rr * LF.gpw + LF.g;
          const bool rv = row < n;
          double f[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            f[q] = 0.0;
            if (rv && v[q]) {
              const int i = c[q] < r ? c[q] : c[q] - r;
              const size_t srow = size_t(row) * size_t(ldb) + size_t(p) * size_t(r);
              if (c[q] < r) {
                const double sc = acc[rr][q] * __ldg(a.t + i);
                f[q] = sc + __ldg(a.V + row);
              } else {
                f[q] = a.S[srow + i];
              }
              const size_t o = size_t(row) * size_t(ldf) + c[q];
              if (sweeps) {
                Fc[o] = f[q];
                a.E[o] = f[q];
              } else if (c[q] < r) {
                // assembly W = F_L + fl(F_R * alpha) (:148-154)
                double wv = f[q];
                double fr = 0.0;
                if (p > 0) {
                  fr = a.S[srow + i];
                  wv = wv + fr * __ldg(a.alpha + i);
                }
                a.W[size_t(i) * size_t(n) + row] = wv;
                if (a.FLo) a.FLo[size_t(i) * size_t(n) + row] = f[q];
                if (a.FRo) a.FRo[size_t(i) * size_t(n) + row] = fr;
              }
            }
            f[q] = fabs(f[q]);
          }
          if (sweeps) {
            const double rf = group_rowsum<Q>(f, LF.G, LF.qp);
            if (rv) mf = umax64(mf, abs_bits(rf));
          }
        }
      }
  }
  if (!sweeps) {
    finish(kStOk, 0, L_S, 1);
    return;
  }
  double fnorm, dummy;
  sync_step(mf, mf, fnorm, dummy);

  // ================= recovery sweeps (phi_block.cpp:122-146)
  for (int sweep = 1; sweep < a.s_eff; ++sweep) {
    int kk = 0;
    double d1 = INF, d2 = fnorm, nE = fnorm;  // E = F
    trace(2.0, d2, nE);
    while (d1 + d2 > a.tol * nE) {
      if (kk >= 300) {
        err = kStRecoveryCap;
        err_idx = 300;
        break;
      }
      ++kk;
      d1 = d2;
      const double fac = a.single_variant ? a.t_single / (double(a.s_eff) * kk) : 0.0;
      unsigned long long mfb = 0, meb = 0;
      {
        int c[Q];
        bool v[Q];
        double tosF[Q];
        cols(LF, c, v);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int i = c[q] < r ? c[q] : c[q] - r;
          tosF[q] = v[q] ? __ldg(a.colTos + i) : 0.0;
        }
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
          for (int wt = warp; wt < a.tile / LF.RW; wt += kWarps) {
            const int base = t * a.tile + wt * LF.RW;
            double eo[R][Q], fs[R][Q], acc[R][Q];
            bool vq[R][Q];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
              const int row = base + rr * LF.gpw + LF.g;
#pragma unroll
              for (int q = 0; q < Q; ++q) {
                vq[rr][q] = row < n && v[q];
                const size_t o = size_t(row) * size_t(ldf) + c[q];
                eo[rr][q] = vq[rr][q] ? a.E[o] : 0.0;
                fs[rr][q] = (vq[rr][q] && has_xi) ? Fc[o] : 0.0;
                acc[rr][q] = 0.0;
              }
            }
            const TileCsr tc = stage_csr(a, base, LF.RW, st, lane);
            int rs[R], cnt[R];
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
              const int li = rr * LF.gpw + LF.g;
              rs[rr] = st.rp[li] - tc.e_lo;
              cnt[rr] = st.rp[li + 1] - st.rp[li];
            }
            gather_tile<Q, R, B>(tc, rs, cnt, Fc, ldf, c, v, acc);
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
              const int row = base + rr * LF.gpw + LF.g;
              double ay[Q], ae[Q];
#pragma unroll
              for (int q = 0; q < Q; ++q) {
                double y = acc[rr][q];
                if (has_xi) y = y - a.xi * fs[rr][q];
                if (a.single_variant) {
                  y = fac * y;  // phi_single.cpp:106
                } else {
                  y = y / double(kk);  // phi_block.cpp:132
                  y = y * tosF[q];     // :134-135
                }
                const double en = eo[rr][q] + y;  // E += F (:138)
                if (vq[rr][q]) {
                  const size_t o = size_t(row) * size_t(ldf) + c[q];
                  Fn[o] = y;
                  a.E[o] = en;
                }
                ay[q] = vq[rr][q] ? fabs(y) : 0.0;
                ae[q] = vq[rr][q] ? fabs(en) : 0.0;
              }
              const double ry = group_rowsum<Q>(ay, LF.G, LF.qp);
              const double re = group_rowsum<Q>(ae, LF.G, LF.qp);
              if (row < n) {
                mfb = umax64(mfb, abs_bits(ry));
                meb = umax64(meb, abs_bits(re));
              }
            }
          }
      }
      double maxF2, maxE;
      sync_step(mfb, meb, maxF2, maxE);
      d2 = maxF2;
      if (!isfinite(d2)) {
        err = kStRecoveryDiverged;
        err_idx = kk;
        break;
      }
      nE = maxE;
      trace(3.0, d2, nE);
      double* tmp = Fc;
      Fc = Fn;
      Fn = tmp;
    }
    if (err != kStOk) break;
    if (master) a.lensF[sweep - 1] = kk;

    // ---- sweep end (:141-145): E *= mu; Sadv = Sadv*Jexp; F refresh
    // phase A (S layout): Sadv blocks 1..p in place, ascending source column
    {
      int c[Q];
      bool v[Q];
      cols(LS, c, v);
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int wt = warp; wt < a.tile / LS.RW; wt += kWarps) {
          const int base = t * a.tile + wt * LS.RW;
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const int row = base + rr * LS.gpw + LS.g;
            double nv[Q];
            bool wq[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              const int j = v[q] ? c[q] / r : 0, i = c[q] - j * r;
              wq[q] = row < n && v[q] && j >= 1;
              nv[q] = 0.0;
              if (wq[q]) {
                const double* srow = a.S + size_t(row) * size_t(ldb);
                const double* cc = a.jc + size_t(i) * size_t(p + 1);
                double accv = 0.0;
                for (int l = 1; l <= j; ++l) accv = accv + srow[l * r + i] * __ldg(cc + (j - l));
                nv[q] = accv;
              }
            }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < Q; ++q)
              if (wq[q]) a.S[size_t(row) * size_t(ldb) + c[q]] = nv[q];
          }
        }
    }
    __syncthreads();
    // phase B (F layout): F_L = E_L*mu, F_R = E_R*mu + Sadv_p; E = F
    const bool last = sweep == a.s_eff - 1;
    unsigned long long mfe = 0;
    {
      int c[Q];
      bool v[Q];
      cols(LF, c, v);
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int wt = warp; wt < a.tile / LF.RW; wt += kWarps) {
          const int base = t * a.tile + wt * LF.RW;
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const int row = base + rr * LF.gpw + LF.g;
            const bool rv = row < n;
            double f[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              f[q] = 0.0;
              if (rv && v[q]) {
                const int i = c[q] < r ? c[q] : c[q] - r;
                const size_t o = size_t(row) * size_t(ldf) + c[q];
                const size_t srow = size_t(row) * size_t(ldb) + size_t(p) * size_t(r);
                const double en = a.E[o] * __ldg(a.mu + i);
                double fv = en;
                if (c[q] >= r) fv = en + a.S[srow + i];
                f[q] = fv;
                if (last && c[q] < r) {
                  double wv = fv;
                  double fr = 0.0;
                  if (p > 0) {
                    const double er = a.E[size_t(row) * size_t(ldf) + r + i] * __ldg(a.mu + i);
                    fr = er + a.S[srow + i];
                    wv = wv + (a.single_variant ? __ldg(a.alpha + i) * fr : fr * __ldg(a.alpha + i));
                  }
                  a.W[size_t(i) * size_t(n) + row] = wv;
                  if (a.FLo) a.FLo[size_t(i) * size_t(n) + row] = fv;
                  if (a.FRo) a.FRo[size_t(i) * size_t(n) + row] = fr;
                }
              }
            }
            if (!last) {
              __syncwarp();
              double af[Q];
#pragma unroll
              for (int q = 0; q < Q; ++q) {
                if (rv && v[q]) {
                  const size_t o = size_t(row) * size_t(ldf) + c[q];
                  Fc[o] = f[q];
                  a.E[o] = f[q];
                }
                af[q] = (rv && v[q]) ? fabs(f[q]) : 0.0;
              }
              const double rf = group_rowsum<Q>(af, LF.G, LF.qp);
              if (rv) mfe = umax64(mfe, abs_bits(rf));
            }
          }
        }
    }
    if (!last) {
      double dmy;
      sync_step(mfe, mfe, fnorm, dmy);
    }
  }
  finish(err, err_idx, L_S, 0);
}

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

cudaError_t coop_grid_size(int QT, int block, int* max_blocks) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  switch (QT) {
    case 1: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_phimv_block<1>, block, 0); break;
    case 2: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_phimv_block<2>, block, 0); break;
    case 4: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_phimv_block<4>, block, 0); break;
    case 8: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_phimv_block<8>, block, 0); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  *max_blocks = per_sm * sms;
  return cudaSuccess;
}

cudaError_t launch_phimv_block(const BlockArgs& a, int grid, int block, cudaStream_t st) {
  BlockArgs copy = a;
  void* args[] = {&copy};
  ++g_launches;
  switch (a.QT) {
    case 1: return cudaLaunchCooperativeKernel((void*)k_phimv_block<1>, grid, block, args, 0, st);
    case 2: return cudaLaunchCooperativeKernel((void*)k_phimv_block<2>, grid, block, args, 0, st);
    case 4: return cudaLaunchCooperativeKernel((void*)k_phimv_block<4>, grid, block, args, 0, st);
    case 8: return cudaLaunchCooperativeKernel((void*)k_phimv_block<8>, grid, block, args, 0, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_spmv(int32_t n, const int32_t* rp, const int32_t* ci, const double* av,
                        const double* x, double* y, int mode, double xi, double div,
                        unsigned long long* chunkmax, cudaStream_t st) {
  ++g_launches;
  k_spmv<<<nchunks(n), kBlock, 0, st>>>(n, rp, ci, av, x, y, mode, xi, div, chunkmax);
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
