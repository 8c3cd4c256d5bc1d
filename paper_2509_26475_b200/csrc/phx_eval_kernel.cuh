// The persistent phimv_block kernel (phi_block.cpp:48-157, Alg. 3), sm_100a.
// Template definitions; the variants are instantiated by phx_eval_q*.cu and
// dispatched by phx_eval.cu.
//
// ONE cooperative launch per evaluation.  Every Taylor term is a grid step:
// the CTAs sweep their row tiles, each lane group (G lanes of a warp, V = 1
// or 2 adjacent columns per lane, Q column chunks) gathers the CSR row's
// block rows (row-interleaved layout, one coalesced vector load per gathered
// row), fuses the shift, scaling, J-term and accumulator updates with both
// |.| row sums, and publishes a per-CTA max with one atomicMax; after
// grid.sync() every CTA reads the two maxima and takes the same stopping
// decision, so loop control never leaves the device.
//
// Compiled with --fmad=false (no FMA): bit-for-bit the oracle's operation
// order (oracle/phx_oracle.cpp).  Row sums use the canonical
// pairwise tree over pow2-padded natural column order: with V = 2 the
// lane-local pair is the tree's first level, the butterfly the next ones.
//
// Tiles reach a phase body through a per-warp cp.async pipeline of their CSR
// slices (pipelined / run_tiles), sized per variant (PipeCfg).  C2's variant
// ((1,2,1), gather batch 5, static) runs its S terms through a lean body
// instead: grid-stride warp tiles, CSR read directly, column coefficients
// from a shared table.
#include <cooperative_groups.h>

#include <atomic>

#pragma once
#include "phx_kernels.cuh"

namespace cg = cooperative_groups;

namespace phx {
namespace {

constexpr unsigned kFull = 0xffffffffu;
#ifndef PHX_X_BLOCK
#define PHX_X_BLOCK 256
#endif
constexpr int kBlock = PHX_X_BLOCK;  // threads per CTA
constexpr int kWarps = kBlock / 32;
constexpr int kMaxRW = 64;  // rows per warp tile
constexpr double DBL_MAX_D = 1.7976931348623157e308;

__device__ __forceinline__ unsigned long long abs_bits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7FFFFFFFFFFFFFFFull;
}
__device__ __forceinline__ double from_bits(unsigned long long b) {
  return __longlong_as_double(static_cast<long long>(b));
}
__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}

// fl(x / d) -- bitwise the IEEE quotient -- for a divisor d >= 1 with rcp =
// fl(1 / d): q = fl(x rcp) is faithful, r = x - q d is exact (one FMA), and
// fl(q + r rcp) is the correctly rounded quotient (Markstein's theorem).  An
// exact quotient (r == 0, zeros included) keeps q, which also keeps the sign of
// a zero; |x| or |q| outside [2^-960, 2^961) (where r could underflow) and
// non-finite operands take the IEEE division.  Three FP64 instructions on the
// common path instead of the ~10 of the generic division sequence; checked
// against x / d on 10^9 random pairs (divisors k! and arbitrary), DESIGN.md §4.
#ifndef PHX_DIVRCP
#define PHX_DIVRCP 0  // measured slower than the IEEE division sequence
#endif
__device__ __forceinline__ double div_rcp(double x, double d, double rcp) {
  if (!PHX_DIVRCP) return x / d;
  const double q = x * rcp;
  const double r = __fma_rn(-q, d, x);
  double y = r == 0.0 ? q : __fma_rn(r, rcp, q);
  const unsigned ex = (unsigned(__double2hiint(x)) >> 20) & 0x7FFu;
  const unsigned eq = (unsigned(__double2hiint(q)) >> 20) & 0x7FFu;
  if (ex - 63u > 1920u || eq - 63u > 1920u) y = x / d;
  return y;
}

// system-scope loads of the cross-part mailboxes (another GPU writes them)
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <int V>
struct Vio;
// ld/st: default caching (gather sources and their producers);
// ldcs/stcs: evict-first streaming hints for the read-once / write-once
// accumulator streams (Vw, S, E), so L2 keeps the gather targets
template <>
struct Vio<1> {
  __device__ __forceinline__ static void ld(const double* p, double (&x)[1]) { x[0] = *p; }
  __device__ __forceinline__ static void st(double* p, const double (&x)[1]) { *p = x[0]; }
  __device__ __forceinline__ static void ldcs(const double* p, double (&x)[1]) { x[0] = __ldcs(p); }
  __device__ __forceinline__ static void stcs(double* p, const double (&x)[1]) { __stcs(p, x[0]); }
};
template <>
struct Vio<2> {
  __device__ __forceinline__ static void ld(const double* p, double (&x)[2]) {
    const double2 t = *reinterpret_cast<const double2*>(p);
    x[0] = t.x;
    x[1] = t.y;
  }
  __device__ __forceinline__ static void st(double* p, const double (&x)[2]) {
    *reinterpret_cast<double2*>(p) = make_double2(x[0], x[1]);
  }
  __device__ __forceinline__ static void ldcs(const double* p, double (&x)[2]) {
    const double2 t = __ldcs(reinterpret_cast<const double2*>(p));
    x[0] = t.x;
    x[1] = t.y;
  }
  __device__ __forceinline__ static void stcs(double* p, const double (&x)[2]) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(x[0], x[1]));
  }
};
// block-stream accesses with the evict-first hints when the blocks are in
// global memory (H), plain generic accesses in cluster mode (shared memory;
// the .global cache hints do not apply there)
template <bool H, int V>
__device__ __forceinline__ void ld_s(const double* p, double (&x)[V]) {
  if constexpr (H)
    Vio<V>::ldcs(p, x);
  else
    Vio<V>::ld(p, x);
}
template <bool H, int V>
__device__ __forceinline__ void st_s(double* p, const double (&x)[V]) {
  if constexpr (H)
    Vio<V>::stcs(p, x);
  else
    Vio<V>::st(p, x);
}
template <bool H>
__device__ __forceinline__ double ld1_s(const double* p) {
  if constexpr (H)
    return __ldcs(p);
  else
    return *p;
}

template <int Q, int V, int R_>
struct Cfg {
  static constexpr int R = R_;  // rows per lane group per warp tile
  // gather batch: entries in flight per lane group
  // (the kernels' BO template argument overrides it: a batch that matches the
  // operator's row length issues no predicated-off slots -- DESIGN.md §4)
  static constexpr int B = (Q == 1 && V == 2 && R_ == 1) ? 8 : ((Q * V * R_ <= 4) ? 4 : 2);
  // resident CTAs per SM the register budget is sized for
  static constexpr int MINB0 = (Q * V * R_ <= 2) ? 4 : ((Q * V * R_ <= 4) ? 3 : ((Q * V <= 4) ? 2 : 1));
  // (the budgets above are for 256-thread CTAs)
  static constexpr int MINB = MINB0 * 256 / kBlock > 0 ? MINB0 * 256 / kBlock : 1;
  // row-local accumulator streams loaded after the gather (its batch gets the
  // registers) for scalar lanes (C4: 116 -> 97 ms); the double2 variants load
  // them first, hiding their latency behind the gather (measured: C2, C5)
  static constexpr bool LATE = V == 1;
};

// Lane-group layout of one phase (S width or F width).
struct Layout {
  int G, gpw, g, lg, RW, qn, qp, width;
};

__device__ __forceinline__ Layout make_layout(int G, int qn, int width, int R, int V) {
  Layout L;
  const int lane = threadIdx.x & 31;
  L.G = G;
  L.gpw = 32 / G;
  L.g = lane / G;
  L.lg = lane % G;
  L.RW = L.gpw * R;
  L.qn = qn;
  L.width = width;
  const int chunk = 32 * V;  // columns per chunk q
  int chunks = (width + chunk - 1) / chunk;
  int qp = 1;
  while (qp < chunks) qp <<= 1;
  L.qp = width > chunk ? qp : 1;
  return L;
}

// Canonical row sum of the group's |values| (pairwise tree over pow2-padded
// natural column order; invalid lanes hold 0).
template <int Q, int V>
__device__ __forceinline__ double group_rowsum(const double (&v)[Q][V], int G, int qp) {
  double T[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    double x = v[q][0];
    if (V == 2) x = x + v[q][V - 1];
#pragma unroll
    for (int m = 1; m < 32; m <<= 1)
      if (m < G) x = x + __shfl_xor_sync(kFull, x, m);  // G is warp-uniform
    T[q] = x;
  }
#pragma unroll
  for (int h = 1; h < Q; h <<= 1) {
    if (h < qp) {
#pragma unroll
      for (int q = 0; q + h < Q; q += 2 * h) T[q] = T[q] + T[q + h];
    }
  }
  return T[0];
}

// CTA max of two bit patterns -> one atomicMax each into the step's slot.
__device__ __forceinline__ void publish2(unsigned long long a, unsigned long long b,
                                         unsigned long long* slot,
                                         unsigned long long (*red)[kWarps]) {
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
    for (int q = 0; q < kWarps; ++q) {
      ma = umax64(ma, red[0][q]);
      mb = umax64(mb, red[1][q]);
    }
    atomicMax(slot, ma);
    atomicMax(slot + 1, mb);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Per-warp cp.async pipeline over the warp's sequence of row tiles.  While
// tile s is computed, the CSR entries of tile s+1 and the row_ptr slice of
// tile s+2 are in flight into warp-private shared memory (LDGSTS, no
// registers held), so the row_ptr -> entries -> gather dependency chain costs
// one round trip per tile instead of three.
// ---------------------------------------------------------------------------
#ifndef PHX_LEAN
#define PHX_LEAN 1
#endif
constexpr int kEC = 160;  // staged CSR entries per warp tile (default)

template <int EC_>
struct WarpPipeT {
  static constexpr int EC = EC_;  // staged CSR entries per warp tile
  int rp[3][kMaxRW + 1];
  int ci[2][EC];
  double av[2][EC];
  // latency mode: slot 0 still holds this tile's row_ptr and entries (set
  // after a single-tile sequence -- the warp owns the same tile every step)
  int cached_base, cached_rw;
};
using WarpPipe = WarpPipeT<kEC>;

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// A phase's tiles come in two parts.  The first static_frac of the CTA tiles
// are assigned round-robin (tile t to CTA t mod ncta; within it the warp takes
// warp tiles warp, warp+8, ...: m of them) -- no atomics, neighbouring rows in
// flight together.  The remaining warp tiles are grabbed one at a time from
// the step's counter, so the CTAs that run faster absorb the tail instead of
// waiting at the step barrier (per-CTA speed differs by up to ~20% and is
// stable from step to step).  The two parts run as separate pipelined loops
// so each keeps only its own state live.  Sequences are asked for positions in
// increasing order, each at most twice in a row.
struct TileSeq {
  int mlog, ntiles, tile, RW, warp, cta, ncta;  // m = 1 << mlog warp tiles per CTA tile
  __device__ __forceinline__ int at(int s, int) const {
    const int t = cta + (s >> mlog) * ncta;
    return t < ntiles ? t * tile + (warp + (s & ((1 << mlog) - 1)) * kWarps) * RW : -1;
  }
};

struct DynSeq {
  int dyn0, dynN, RW, mpos, mval;
  unsigned long long* ctr;
  unsigned long long pend;  // lane 0: the grab in flight (issued one tile ahead)
  // positions are asked for in order, the newest possibly twice (memoized)
  __device__ __forceinline__ int at(int pos, int lane) {
    if (pos == mpos) return mval;
    const int id = dyn0 + int(__shfl_sync(kFull, pend, 0));
    mpos = pos;
    mval = id < dynN ? id * RW : -1;
    if (id < dynN && lane == 0) pend = atomicAdd(ctr, 1ull);
    return mval;
  }
};

// static CTA tiles of a phase with ntiles tiles (the DYN kernels; the host
// picks them when the CTAs get many tiles each -- DESIGN.md §4)
__device__ __forceinline__ int static_tiles(const BlockArgs& a, int ntiles, int ncta) {
  if (!(a.static_frac < 1.0)) return ntiles;
  return min(ntiles, int(a.static_frac * double(ntiles) / double(ncta)) * ncta);
}

__device__ __forceinline__ void issue_rp(const BlockArgs& a, int* dst, int base, int RW, int lane) {
  for (int l = lane; l <= RW; l += 32) cp_async4(dst + l, a.rp + min(base + l, a.n));
}

template <int EC>
__device__ __forceinline__ void issue_entries(const BlockArgs& a, const int* rp, int RW, int* ci,
                                              double* av, int lane) {
  const int e_lo = rp[0], E = rp[RW] - e_lo;
  if (E <= EC)
    for (int e = lane; e < E; e += 32) {
      cp_async4(ci + e, a.ci + e_lo + e);
      cp_async8(av + e, a.av + e_lo + e);
    }
}

// body(base, rp, ci, av): rp = row_ptr[base .. base+RW] (clamped at n); when
// rp[RW] - rp[0] <= kEC, ci/av hold the tile's entries from index 0.
template <bool CACHE, class Seq, class Body, class Pipe>
__device__ __forceinline__ void pipelined(const BlockArgs& a, Seq& ts, int RW, Pipe& pp,
                                          int lane, Body& body) {
  const int b0 = ts.at(0, lane);
  if (b0 < 0) return;  // warp-uniform
  int b1 = -1;
  if constexpr (CACHE) {
    b1 = ts.at(1, lane);
    if (b1 < 0 && pp.cached_base == b0 && pp.cached_rw == RW) {
      body(b0, pp.rp[0], pp.ci[0], pp.av[0]);  // no restaging round trips
      __syncwarp();
      return;
    }
  }
  __syncwarp();
  issue_rp(a, pp.rp[0], b0, RW, lane);
  cp_commit();
  cp_wait_all();
  __syncwarp();
  issue_entries<Pipe::EC>(a, pp.rp[0], RW, pp.ci[0], pp.av[0], lane);
  if constexpr (!CACHE) b1 = ts.at(1, lane);
  if (b1 >= 0) issue_rp(a, pp.rp[1], b1, RW, lane);
  cp_commit();
  if constexpr (CACHE) {
    if (lane == 0) {  // what slot 0 holds afterwards (a single tile never leaves it)
      pp.cached_base = b1 < 0 ? b0 : -1;
      pp.cached_rw = RW;
    }
  }
  int base = b0;
  for (int s = 0; base >= 0; ++s) {
    cp_wait_all();
    __syncwarp();  // tile s's entries and tile s+1's row_ptr have landed
    const int nb = ts.at(s + 1, lane);
    if (nb >= 0) {
      issue_entries<Pipe::EC>(a, pp.rp[(s + 1) % 3], RW, pp.ci[(s + 1) & 1], pp.av[(s + 1) & 1], lane);
      const int nnb = ts.at(s + 2, lane);
      if (nnb >= 0) issue_rp(a, pp.rp[(s + 2) % 3], nnb, RW, lane);
    }
    cp_commit();
    body(base, pp.rp[s % 3], pp.ci[s & 1], pp.av[s & 1]);
    __syncwarp();  // done with slot s before it is refilled
    base = nb;
  }
}

// every warp tile of a phase: the static part, then the dynamic tail from
// counter ctr (zeroed before the phase's step began)
template <bool DYN, bool CL, bool CACHE, class Body, class Pipe>
__device__ __forceinline__ void run_tiles(const BlockArgs& a, const Layout& L, int ntiles,
                                          int warp, int cta, int ncta,
                                          unsigned long long* ctr, Pipe& pp, int lane,
                                          const int* crp, const int* cci, const double* cav,
                                          Body&& body) {
  if constexpr (CL) {
    // cluster mode: the part's CSR lives in shared memory for the whole
    // launch (crp padded to whole tiles); the CTA owns every tile of its part
    (void)ctr;
    (void)pp;
    (void)lane;
    (void)cta;
    (void)ncta;
    for (int t = 0; t < ntiles; ++t)
      for (int wt = warp; wt < a.tile / L.RW; wt += kWarps) {
        const int base = t * a.tile + wt * L.RW;
        if (base >= a.n) break;  // warp-uniform
        const int* rp = crp + base;
        const int e0 = rp[0];
        body(base, rp, cci + e0, cav + e0);
      }
  } else {
  const int tst = DYN ? static_tiles(a, ntiles, ncta) : ntiles;
  {
    TileSeq ts;
    ts.mlog = __ffs(a.tile / (L.RW * kWarps)) - 1;  // a power of two: G / min(GS, GF)
    ts.ntiles = tst;
    ts.tile = a.tile;
    ts.RW = L.RW;
    ts.warp = warp;
    ts.cta = cta;
    ts.ncta = ncta;
    pipelined<CACHE>(a, ts, L.RW, pp, lane, body);
  }
  if (DYN && tst < ntiles) {
    DynSeq ds;
    ds.dyn0 = tst * (a.tile / L.RW);
    ds.dynN = (a.n + L.RW - 1) / L.RW;
    ds.RW = L.RW;
    ds.ctr = ctr;
    ds.pend = 0;
    ds.mpos = -1;
    ds.mval = -1;
    if (lane == 0) ds.pend = atomicAdd(ctr, 1ull);
    pipelined<CACHE>(a, ds, L.RW, pp, lane, body);
  }
  }
}

// acc[rr][q][e] = sum over row rr's entries (storage order, from +0) of
// av * X[col*ld + c].  X was written before the last grid.sync(), which
// invalidates L1 (CCTL.IVALL), so plain cached loads are coherent.
// PART: column indices are encoded (owner part << 27 | row within the owner)
// and X is resolved per entry through the gather table Xt (one base pointer
// per part: peer-GPU memory in a multi-GPU run).
constexpr unsigned kOwnerShift = 27;
constexpr unsigned kLocalMask = (1u << kOwnerShift) - 1u;
constexpr unsigned kLocalOwner = 31u;  // owner field of a part's own rows (host: phx_host.cpp)

// gather loads carry an L2 cache policy: evict_last for the fraction
// a.gather_keep of lines -- 1 for operators whose gather reuse distance is
// far but fits in L2 (C3: the z +- 1 planes 65,536 rows apart, while the
// accumulator streams pass through evict-first), else 0 (default priority)
template <int V>
__device__ __forceinline__ void ld_gather(const double* p, double (&x)[V], unsigned long long pol) {
  if constexpr (V == 2) {
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(x[0]), "=d"(x[1])
                 : "l"(p), "l"(pol));
  } else {
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(x[0]) : "l"(p), "l"(pol));
  }
}
__device__ __forceinline__ unsigned long long gather_policy(float keep) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, %1;"
               : "=l"(pol)
               : "f"(keep));
  return pol;
}

template <bool PART>
__device__ __forceinline__ const double* gather_row_ptr(const double* X,
                                                        const double* const* Xt, unsigned enc,
                                                        unsigned ld) {
  if (PART) {
    // owner kLocalOwner: a row of this part (X, no table lookup on the
    // dependent gather chain); else the owning part's buffer
    const unsigned ow = enc >> kOwnerShift;
    return (ow == kLocalOwner ? X : Xt[ow]) + size_t(enc & kLocalMask) * ld;
  }
  return X + enc * ld;
}

template <int Q, int V, int R, int B, bool SMEM, bool PART, bool HINT>
__device__ __forceinline__ void gather(const BlockArgs& a, const int* ci, const double* av_s,
                                       int e_lo, unsigned ld, const int (&rs)[R],
                                       const int (&cnt)[R], const double* X,
                                       const double* const* Xt, const unsigned (&cq)[Q],
                                       const bool (&vq)[Q], double (&acc)[R][Q][V]) {
  int maxc = 0;
#pragma unroll
  for (int rr = 0; rr < R; ++rr) maxc = max(maxc, cnt[rr]);
  unsigned long long pol = 0;
  if constexpr (HINT) pol = gather_policy(a.gather_keep);
  for (int u0 = 0; u0 < maxc; u0 += B) {
    double xv[B][R][Q][V];
#pragma unroll
    for (int u = 0; u < B; ++u)
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        const bool ok = u0 + u < cnt[rr];
        const double* xr = X;
        if (ok) {
          const int e = rs[rr] + u0 + u;
          xr = gather_row_ptr<PART>(X, Xt, unsigned(SMEM ? ci[e] : __ldg(a.ci + e_lo + e)), ld);
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          if (ok && vq[q]) {
            if constexpr (HINT)
              ld_gather<V>(xr + cq[q], xv[u][rr][q], pol);
            else
              Vio<V>::ld(xr + cq[q], xv[u][rr][q]);
          } else {
#pragma unroll
            for (int e = 0; e < V; ++e) xv[u][rr][q][e] = 0.0;
          }
        }
      }
#pragma unroll
    for (int u = 0; u < B; ++u)
#pragma unroll
      for (int rr = 0; rr < R; ++rr)
        if (u0 + u < cnt[rr]) {
          const int e = rs[rr] + u0 + u;
          const double av = SMEM ? av_s[e] : __ldg(a.av + e_lo + e);
#pragma unroll
          for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int v = 0; v < V; ++v) acc[rr][q][v] = acc[rr][q][v] + av * xv[u][rr][q][v];
        }
  }
}

template <int Q, int V, int R, int B, bool PART, bool HINT = false, int EC = kEC>
__device__ __forceinline__ void gather_tile(const BlockArgs& a, const Layout& L, const int* rp,
                                            const int* ci, const double* av, unsigned ld,
                                            const double* X, const double* const* Xt,
                                            const unsigned (&cq)[Q], const bool (&vq)[Q],
                                            double (&acc)[R][Q][V]) {
  const int e_lo = rp[0];
  int rs[R], cnt[R];
#pragma unroll
  for (int rr = 0; rr < R; ++rr) {
    const int li = rr * L.gpw + L.g;
    rs[rr] = rp[li] - e_lo;
    cnt[rr] = rp[li + 1] - rp[li];
  }
  if (rp[L.RW] - e_lo <= EC)
    gather<Q, V, R, B, true, PART, HINT>(a, ci, av, e_lo, ld, rs, cnt, X, Xt, cq, vq, acc);
  else
    gather<Q, V, R, B, false, PART, HINT>(a, ci, av, e_lo, ld, rs, cnt, X, Xt, cq, vq, acc);
}

// dynamic shared memory: the per-warp pipes, then (cluster mode) the part's
// blocks Vw, D0, D1, S (cl_rows x ldb each) and F0, F1, E (cl_rows x ldf)
constexpr size_t kPipeBytes = (size_t(kWarps) * sizeof(WarpPipe) + 15) / 16 * 16;
// the lean-body variant (C2's: (1,2,1), batch 5, static) stages few entries
// per tile (<= 40 for 5-entry rows), so its pipes are smaller and the L1
// that its gathers hit larger
template <int Q, int V, int RR, bool PART, bool DYN, int BO, bool CL, bool LAT>
struct PipeCfg {
  static constexpr bool lean =
      PHX_LEAN && !CL && !LAT && !PART && !DYN && Q == 1 && V == 2 && RR == 1 && BO == 5;
  // the 2-entry-row batch variant ((1,2,2), batch 2: C5's bidiagonal rows)
  // stages at most 2 entries per row of an 8-row tile
  static constexpr bool two = !CL && Q == 1 && V == 2 && RR == 2 && BO == 2;
  static constexpr int EC = lean ? 48 : (two ? 32 : kEC);
  static constexpr size_t bytes = (size_t(kWarps) * sizeof(WarpPipeT<EC>) + 15) / 16 * 16;
};

// CL (cluster mode, implies PART): the launch is ONE thread-block cluster,
// one CTA per part; every part's blocks live in its CTA's shared memory, the
// gathers of other parts' rows read distributed shared memory, and the step
// sync is a DSMEM max exchange + cluster barrier -- small operators (C1,
// small integrator grids) whose steps are latency-bound.
// LAT (latency mode): compiled for ONE CTA per SM (register budget 255) --
// for operators with fewer tiles than SMs, whose steps are latency-bound:
// the gather's loads batch instead of serialising at 64 registers
template <int Q, int V, int RR, bool PART, bool DYN, int BO, bool CL, bool LAT = false>
// register budget: the default-batch partitioned variants (C3's) at 3 CTAs/SM
// (80 registers: their part tables spill heavily at 64 -- C3 at 2 parts
// 436 -> 393 ms, same-box A/B)
__global__ void __launch_bounds__(kBlock, LAT ? 1
                                           : ((PART && !CL && BO == 0 && Cfg<Q, V, RR>::MINB > 3)
                                                  ? 3
                                                  : Cfg<Q, V, RR>::MINB)) k_phimv_block(BlockArgs ga) {
  constexpr int R = Cfg<Q, V, RR>::R;
  constexpr int B = BO > 0 ? BO : Cfg<Q, V, RR>::B;  // gather batch
  // L2 cache-policy gathers (a.gather_keep): the dynamic-tail (1, 2, 1)
  // default-batch variant only -- large operators with long rows (C3); the
  // hinted load form costs the short-row kernels (C2, C5) even at fraction 0,
  // and cluster mode gathers shared memory
  constexpr bool HINT = !CL && DYN && BO == 0 && Q == 1 && V == 2 && RR == 1;
  constexpr bool LEAN = PipeCfg<Q, V, RR, PART, DYN, BO, CL, LAT>::lean;
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long red[2][kWarps];
  // per-warp pipeline buffers: dynamic shared memory (kWarps * sizeof(WarpPipe))
  extern __shared__ __align__(16) unsigned char pipe_smem[];
  using Pipe = WarpPipeT<PipeCfg<Q, V, RR, PART, DYN, BO, CL, LAT>::EC>;
  constexpr int EC = Pipe::EC;
  Pipe* pipe = reinterpret_cast<Pipe*>(pipe_smem);
  // gather tables [D0, D1, S, F0, F1][part] (PART only)
  __shared__ const double* gtab[5][PART ? kMaxParts : 1];
  __shared__ double gmax[2];
  // LEAN: the column coefficients Kd, Ka, t/s (w <= 64 for Q = 1, V = 2),
  // re-read per row in the S terms instead of held in registers
  __shared__ double s_coef[LEAN ? 3 * 64 : 1];
  __shared__ unsigned long long cl_slot[2];                  // CL: this CTA's maxima
  __shared__ unsigned long long cl_box[2][CL ? kMaxParts : 1][2];  // CL: all parts', by step parity
  const double INF = __longlong_as_double(0x7FF0000000000000ll);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Pipe& pp = pipe[warp];
  if (LAT) {
    if (lane == 0) pp.cached_base = -1;
    __syncwarp();
  }

  // Partitioned operator: this launch handles parts
  // plo .. plo+pcount-1, CTAs split evenly; a CTA rebinds the row-local
  // fields of its part (rows are part-local from here on).
  // (unpartitioned: `a` aliases the kernel parameter, read from the constant
  // bank; partitioned: the part's copy in shared memory)
  BlockArgs pa;
  constexpr bool SPA = PART && BO == 0;
  __shared__ __align__(16) unsigned char s_pa_raw[SPA ? sizeof(BlockArgs) : 16];
  BlockArgs* const s_pa = reinterpret_cast<BlockArgs*>(s_pa_raw);
  const int* crp = nullptr;  // cluster mode: the part's CSR in shared memory
  const int* cci = nullptr;
  const double* cav = nullptr;
  int my = 0, cta = int(blockIdx.x), ncta = int(gridDim.x);
  const PartTab* T = nullptr;
  if (PART) {
    pa = ga;
    const int per = CL ? 1 : int(gridDim.x) / ga.pcount;
    my = ga.plo + int(blockIdx.x) / per;
    cta = int(blockIdx.x) % per;
    ncta = per;
    T = ga.ptab + my;
    pa.n = T->nrows;
    pa.rp = T->rp;
    pa.ci = T->ci;
    pa.av = T->av;
    pa.V = T->V;
    pa.Vw = T->Vw;
    pa.D0 = T->D0;
    pa.D1 = T->D1;
    pa.S = T->S;
    pa.F0 = T->F0;
    pa.F1 = T->F1;
    pa.E = T->E;
    pa.W = T->W;
    pa.slots = T->slots;
    if (CL) {
      double* sm = reinterpret_cast<double*>(pipe_smem);  // no pipes in cluster mode
      const size_t nb = size_t(ga.cl_rows) * size_t(ga.ldb), nf = size_t(ga.cl_rows) * size_t(ga.ldf);
      pa.Vw = sm;
      pa.D0 = sm + nb;
      pa.D1 = sm + 2 * nb;
      pa.S = sm + 3 * nb;
      pa.F0 = sm + 4 * nb;
      pa.F1 = pa.F0 + nf;
      pa.E = pa.F1 + nf;
      // the part's CSR: av (8-aligned) then row_ptr (padded to whole tiles) and col_idx
      double* sav = pa.E + nf;
      const int rpad = (ga.cl_rows + ga.tile - 1) / ga.tile * ga.tile + 1;
      int* srp = reinterpret_cast<int*>(sav + ga.cl_nnz);
      int* sci = srp + rpad;
      const int nr = T->nrows, nz = T->rp[nr];
      for (int i = threadIdx.x; i < rpad; i += blockDim.x) srp[i] = T->rp[min(i, nr)];
      for (int e = threadIdx.x; e < nz; e += blockDim.x) {
        sci[e] = T->ci[e];
        sav[e] = T->av[e];
      }
      crp = srp;
      cci = sci;
      cav = sav;
      cg::cluster_group cl = cg::this_cluster();
      for (int q = threadIdx.x; q < ga.nparts; q += blockDim.x) {
        gtab[0][q] = cl.map_shared_rank(pa.D0, q);
        gtab[1][q] = cl.map_shared_rank(pa.D1, q);
        gtab[2][q] = cl.map_shared_rank(pa.S, q);
        gtab[3][q] = cl.map_shared_rank(pa.F0, q);
        gtab[4][q] = cl.map_shared_rank(pa.F1, q);
      }
      if (threadIdx.x == 0) cl_slot[0] = cl_slot[1] = 0ull;
      cl.sync();  // every CTA of the cluster is running before any DSMEM access
    } else {
      for (int q = threadIdx.x; q < ga.nparts; q += blockDim.x) {
        const PartTab& U = ga.ptab[q];
        gtab[0][q] = U.D0;
        gtab[1][q] = U.D1;
        gtab[2][q] = U.S;
        gtab[3][q] = U.F0;
        gtab[4][q] = U.F1;
      }
    }
    if (SPA && threadIdx.x == 0) *s_pa = pa;
    __syncthreads();
  }
  // partitioned: the part's arguments from shared memory for the default-batch
  // variants (C3's: the per-thread copy lives in local memory there, 463 ->
  // 435 ms at 2 parts), the per-thread copy for the short-batch ones (C2's:
  // 6.1 -> 7.6 ms from shared memory) -- same-box A/B, DESIGN.md §7
  const BlockArgs& a = SPA ? *s_pa : (PART ? pa : ga);
  int dpar = 0, fpar = 0;  // D / F ping-pong parity (all parts swap in lockstep)

  const int n = a.n, r = a.r, p = a.p;
  const unsigned ldb = unsigned(a.ldb), ldf = unsigned(a.ldf);
  const int ntiles = (n + a.tile - 1) / a.tile;
  const bool has_xi = a.xi != 0.0;
  const bool master = blockIdx.x == 0 && threadIdx.x == 0 && (!PART || ga.plo == 0);
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;  // writes this launch's status
  const Layout LS = make_layout(a.GS, a.QS, a.w, R, V);
  const Layout LF = make_layout(a.GF, a.QF, a.fcols, R, V);

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
  // publish this CTA's maxima, zero the next step's slot (its last readers
  // finished before the previous grid sync), grid-sync, read the maxima
  auto sync_step = [&](unsigned long long ma, unsigned long long mb, double& ra, double& rb) {
    unsigned long long* slot = a.slots + 4 * (step % 3);
    if (a.tstamp != nullptr && threadIdx.x == 0) {  // diagnostics: CTA arrival, SM id
      const int q = kCtaStampBase + step * ncta + cta;
      if (q < a.tstamp_cap) {
        unsigned long long ns;
        unsigned sm;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        a.tstamp[q] = (ns & ((1ull << 48) - 1ull)) | (static_cast<unsigned long long>(sm) << 48);
      }
    }
    if (CL) {
      // CTA maxima -> every part's box (DSMEM), cluster barrier, max of the boxes
      publish2(ma, mb, cl_slot, red);
      __syncthreads();
      cg::cluster_group cl = cg::this_cluster();
      if (int(threadIdx.x) < ga.nparts) {
        unsigned long long* box = cl.map_shared_rank(&cl_box[step & 1][my][0], int(threadIdx.x));
        box[0] = cl_slot[0];
        box[1] = cl_slot[1];
      }
      cl.sync();
      if (threadIdx.x == 0) {
        unsigned long long A = 0, Bv = 0;
        for (int q = 0; q < ga.nparts; ++q) {
          A = umax64(A, cl_box[step & 1][q][0]);
          Bv = umax64(Bv, cl_box[step & 1][q][1]);
        }
        gmax[0] = from_bits(A);
        gmax[1] = from_bits(Bv);
        cl_slot[0] = cl_slot[1] = 0ull;
      }
      __syncthreads();
      ra = gmax[0];
      rb = gmax[1];
      ++step;
      return;
    }
    publish2(ma, mb, slot, red);
    if (!PART) {
      if (master) {
        unsigned long long* nxt = a.slots + 4 * ((step + 1) % 3);
        nxt[0] = 0ull;
        nxt[1] = 0ull;
        nxt[2] = 0ull;  // the next step's tile counter
      }
      grid.sync();
      if (master && a.tstamp != nullptr && step < a.tstamp_cap) {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        a.tstamp[step] = ns;
      }
      ra = from_bits(__ldcg(reinterpret_cast<const unsigned long long*>(slot)));
      rb = from_bits(__ldcg(reinterpret_cast<const unsigned long long*>(slot + 1)));
    } else {
      // part-local arrival; the part's last CTA publishes the part maxima
      // into every part's mailbox (peer memory); everyone waits for all parts
      if (threadIdx.x == 0) {
        const unsigned gen = unsigned(step) + 1u;
        __threadfence();
        const unsigned old = atomicAdd(T->arrive + (step % 3), 1u);
        if (old == unsigned(ncta) - 1u) {
          __threadfence();
          const unsigned long long A = __ldcg(slot), Bv = __ldcg(slot + 1);
          unsigned long long* nxt = a.slots + 4 * ((step + 1) % 3);
          nxt[0] = 0ull;
          nxt[1] = 0ull;
          nxt[2] = 0ull;  // the part's next tile counter
          T->arrive[(step + 1) % 3] = 0u;
          // mailboxes are double-buffered by step parity: a part can run one
          // step ahead and must not overwrite what a slower part still reads
          const int buf = (step & 1) * ga.nparts;
          for (int q = 0; q < ga.nparts; ++q) {
            MailBox* mbx = ga.ptab[q].mbox + buf + my;
            mbx->a = A;
            mbx->b = Bv;
          }
          // release at system scope: the mailboxes may be peer-GPU memory
          // (NVLink), so the (a, b) writes above must be visible to another
          // device before it sees gen
          __threadfence_system();
          for (int q = 0; q < ga.nparts; ++q)
            atomicExch_system(&(ga.ptab[q].mbox + buf + my)->gen, gen);
        }
        unsigned long long A = 0, Bv = 0;
        for (int q = 0; q < ga.nparts; ++q) {
          const MailBox* mbx = T->mbox + (step & 1) * ga.nparts + q;
          while (ld_acquire_sys(&mbx->gen) < gen) {
          }
          A = umax64(A, ld_relaxed_sys(&mbx->a));
          Bv = umax64(Bv, ld_relaxed_sys(&mbx->b));
        }
        gmax[0] = from_bits(A);
        gmax[1] = from_bits(Bv);
        __threadfence();  // invalidates L1 before the next step's gathers
      }
      __syncthreads();
      ra = gmax[0];
      rb = gmax[1];
    }
    ++step;
  };
  auto finish = [&](int err, int idx, int L_S, int extra_steps) {
    if (lead) {
      a.status[0] = err;
      a.status[1] = idx;
      a.status[2] = L_S;
      a.status[3] = 0;
      a.status[4] = step + extra_steps;
      a.status[5] = min(tr_len, a.trace_cap);
    }
    if (CL) cg::this_cluster().sync();  // peers may still read this CTA's blocks
  };
  // lane column offsets (first column of each chunk) and chunk validity
  auto cols = [&](const Layout& L, unsigned (&c)[Q], bool (&v)[Q]) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      c[q] = unsigned(V * (L.lg + L.G * q));
      v[q] = (q < L.qn) && (int(c[q]) < L.width);
    }
  };

  if constexpr (LEAN) {
    for (int k = threadIdx.x; k < a.w && k < 64; k += blockDim.x) {
      s_coef[k] = a.colKd[k];
      s_coef[64 + k] = a.colKa[k];
      s_coef[128 + k] = a.colTos[k];
    }
    __syncthreads();
  }
  if (master && a.tstamp != nullptr && a.tstamp_cap > kCtaStampBase) {  // diagnostics: launch start
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    a.tstamp[kCtaStampBase - 1] = ns;
  }
  // ================= init: Vw = V[src]*g, D = S = Vw (phi_block.cpp:76-92)
  // Vw_1, D_1 and S_1 are the same block; instead of writing it three times,
  // the init stores V row-major (stride p+1) into D0 and the first S term
  // recomputes Vw_1 = fl(V[src] * g) wherever it needs it (the same single
  // multiply, so the same bits) -- 6 block passes fewer per launch.
  const int p1 = p + 1;
  unsigned long long m0 = 0, mv = 0;  // max |Vw| row sum; max |V| entry (finiteness)
  {
    unsigned c[Q];
    bool v[Q];
    cols(LS, c, v);
    // the lane's source column of V and its g_i, per column
    int srcv[Q][V];
    double gv[Q][V];
#pragma unroll
    for (int q = 0; q < Q; ++q)
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const int cc = int(c[q]) + e;
        const int j = cc / r, i = cc - j * r;
        srcv[q][e] = j == 0 ? 0 : p + 1 - j;
        gv[q][e] = v[q] ? __ldg(a.g + i) : 0.0;
      }
    // NB warp tiles per round with their V loads in flight together: the
    // pass is one dependent load per tile otherwise, latency-bound
    constexpr int NB = (Q * V * R <= 4) ? 4 : 1;
    const int mwt = a.tile / (LS.RW * kWarps);  // warp tiles per CTA tile (power of two)
    auto tile_base = [&](int k) -> int {        // this warp's k-th warp tile, -1 past the end
      const int t = cta + (k / mwt) * ncta;
      return t < ntiles ? t * a.tile + (warp + (k % mwt) * kWarps) * LS.RW : -1;
    };
    for (int k0 = 0; tile_base(k0) >= 0; k0 += NB) {
      double vr[NB][R][Q][V];
      int rowb[NB][R];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int base = tile_base(k0 + b);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int row = base + rr * LS.gpw + LS.g;
          rowb[b][rr] = (base >= 0 && row < n) ? row : -1;
#pragma unroll
          for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int e = 0; e < V; ++e)
              vr[b][rr][q][e] = (rowb[b][rr] >= 0 && v[q])
                                    ? __ldg(a.V + size_t(srcv[q][e]) * size_t(n) + row)
                                    : 0.0;
        }
      }
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int row = rowb[b][rr];
          const bool rv = row >= 0;
          double ax[Q][V];
#pragma unroll
          for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int e = 0; e < V; ++e) {
              double x = 0.0;
              if (rv && v[q]) {
                mv = umax64(mv, abs_bits(vr[b][rr][q][e]));
                x = vr[b][rr][q][e] * gv[q][e];
              }
              ax[q][e] = fabs(x);
            }
          if (rv)  // the row's V entries, row-major, into D0
            for (int col = LS.lg; col < p1; col += LS.G)
              a.D0[size_t(row) * size_t(p1) + col] = __ldg(a.V + size_t(col) * size_t(n) + row);
          const double rsum = group_rowsum<Q, V>(ax, LS.G, LS.qp);
          if (rv) m0 = umax64(m0, abs_bits(rsum));
        }
    }
  }
  double mD, mSn;
  sync_step(m0, mv, mD, mSn);
  if (!(mSn <= DBL_MAX_D)) {  // a non-finite entry of V (check_request, phi_block.cpp:25-26)
    finish(kStInputNonFinite, 0, 1, 0);
    return;
  }
  double c1 = INF, c2 = mD, nS = mD;  // c2 = inf_norm(D) = ||S|| at k = 1 (S = D = Vw)
  trace(0.0, c2, nS);

  // ||S||_inf for the stopping test without a row sum of S in every term:
  // S_k = S_{k-1} + D_k/sigma, so ||S_{k-1}|| -+ c2 bound ||S_k|| (triangle
  // inequality; widened by 1e-12 relative, far above the ~15u the rounded
  // sums can move).  fl(tol * x) is monotone in x, so c1 + c2 > fl(tol * U)
  // proves "continue" and c1 + c2 <= fl(tol * L) proves "stop" -- the
  // reference's decision (phi_block.cpp:93) -- and only an inconclusive term
  // (typically the last one or two) pays an exact pass over S, the same
  // canonical row sums the fused epilogue computed.  With a trace requested,
  // every term gets the exact pass (the trace records ||S||).
  auto s_norm_exact = [&]() -> double {
    unsigned long long m = 0;
    unsigned c[Q];
    bool v[Q];
    cols(LS, c, v);
    for (int t = cta; t < ntiles; t += ncta)
      for (int wt = warp; wt < a.tile / LS.RW; wt += kWarps) {
        const int base = t * a.tile + wt * LS.RW;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int row = base + rr * LS.gpw + LS.g;
          const bool rv = row < n;
          double as[Q][V];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            double x[V];
#pragma unroll
            for (int e = 0; e < V; ++e) x[e] = 0.0;
            if (rv && v[q]) Vio<V>::ld(a.S + (unsigned(row) * ldb + c[q]), x);
#pragma unroll
            for (int e = 0; e < V; ++e) as[q][e] = (rv && v[q]) ? fabs(x[e]) : 0.0;
          }
          const double rs = group_rowsum<Q, V>(as, LS.G, LS.qp);
          if (rv) m = umax64(m, abs_bits(rs));
        }
      }
    double mx, dmy;
    sync_step(m, m, mx, dmy);
    return mx;
  };
  const bool exact_every_term = a.trace != nullptr;
  double nSl = nS, nSu = nS;  // bounds of ||S||; equal to nS while it is exact
  bool exact = true;

  // ================= S series (phi_block.cpp:93-106)
  int k = 1;
  double sigma = 1.0;
  double* Dc = a.D0;
  double* Dn = a.D1;
  int err = kStOk, err_idx = 0;
  const bool vwl_vec = V == 2 && (r % 2) == 0;
  // the first term (k = 2), peeled: its D_1 = Vw_1 = S_1 comes from the
  // row-major V in D0 (see the init); same decision and arithmetic as the loop
  if (c1 + c2 > a.tol * nS) {
    ++k;
    c1 = c2;
    sigma *= k;
    unsigned long long mdb = 0;
    {
      unsigned c[Q];
      bool v[Q];
      cols(LS, c, v);
      int src[Q][V], srcl[Q][V];  // V column of Vw_1's column c and of c - r
      double gg[Q][V], kd[Q][V], ka[Q][V], tos[Q][V];
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int e = 0; e < V; ++e) {
          const int cc = int(c[q]) + e;
          const int j = v[q] ? cc / r : 0, i = v[q] ? cc - j * r : 0;
          src[q][e] = j == 0 ? 0 : p + 1 - j;
          srcl[q][e] = j <= 1 ? 0 : p + 2 - j;
          gg[q][e] = v[q] ? __ldg(a.g + i) : 0.0;
          kd[q][e] = v[q] ? __ldg(a.colKd + cc) : 0.0;
          ka[q][e] = v[q] ? __ldg(a.colKa + cc) : 0.0;
          tos[q][e] = v[q] ? __ldg(a.colTos + cc) : 0.0;
        }
      const double* const* Vt = gtab[0];  // PART: the parts' D0 (their row-major V)
      run_tiles<DYN, CL, LAT>(a, LS, ntiles, warp, cta, ncta, a.slots + 4 * (step % 3) + 2, pp, lane,
                         crp, cci, cav,
                [&](int base, const int* rp, const int* ci, const double* avs) {
          const int e_lo = rp[0];
          const bool sm = rp[LS.RW] - e_lo <= EC;
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const int row = base + rr * LS.gpw + LS.g;
            const bool rv = row < n;
            const int li = rr * LS.gpw + LS.g;
            const int e0 = rp[li] - e_lo, cnt = rp[li + 1] - rp[li];
            // gather: acc = sum_e av_e * Vw_1[col_e] = av_e * fl(V[col_e][src] * g)
            double acc[Q][V];
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
              for (int e = 0; e < V; ++e) acc[q][e] = 0.0;
            for (int u = 0; u < cnt; ++u) {
              const int ee = e0 + u;
              const unsigned enc = unsigned(sm ? ci[ee] : __ldg(a.ci + e_lo + ee));
              const double av = sm ? avs[ee] : __ldg(a.av + e_lo + ee);
              const double* vr = gather_row_ptr<PART>(a.D0, Vt, enc, unsigned(p1));
#pragma unroll
              for (int q = 0; q < Q; ++q)
                if (v[q]) {
#pragma unroll
                  for (int e = 0; e < V; ++e)
                    acc[q][e] = acc[q][e] + av * (vr[src[q][e]] * gg[q][e]);
                }
            }
            double ad[Q][V];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              const bool vv = rv && v[q];
              double vn[V], dn[V], sn[V];
              const double* vo = a.D0 + size_t(rv ? row : 0) * size_t(p1);
#pragma unroll
              for (int e = 0; e < V; ++e) {
                const int cc = int(c[q]) + e;
                const double vw = vv ? vo[src[q][e]] * gg[q][e] : 0.0;  // Vw_1 = D_1 = S_1
                const double vwl = (vv && cc >= 2 * r) ? vo[srcl[q][e]] * gg[q][e] : 0.0;
                double g2 = 0.0;  // Vw = Vw * Kiter (:98)
                if (cc >= 2 * r) g2 = g2 + vwl * ka[q][e];
                g2 = g2 + vw * kd[q][e];
                vn[e] = g2;
                double y = acc[q][e];  // D = (A - xi I) D (:99), * t_i/s, + Vw
                if (has_xi) y = y - a.xi * vw;
                y = y * tos[q][e];
                dn[e] = y + g2;
                sn[e] = vw + dn[e] / sigma;  // S += D/sigma (:105)
                ad[q][e] = vv ? fabs(dn[e]) : 0.0;
              }
              if (vv) {
                const unsigned o = unsigned(row) * ldb + c[q];
                st_s<!CL>(a.Vw + o, vn);
                Vio<V>::st(Dn + o, dn);
                st_s<!CL>(a.S + o, sn);
              }
            }
            const double rd = group_rowsum<Q, V>(ad, LS.G, LS.qp);
            if (rv) mdb = umax64(mdb, abs_bits(rd));
          }
                });
    }
    double maxD, dmy;
    sync_step(mdb, mdb, maxD, dmy);
    c2 = maxD / sigma;  // :103
    if (!isfinite(c2)) {
      err = kStSeriesDiverged;
      err_idx = k;
    } else {
      nSu = (nSu + c2) * (1.0 + 1e-12);
      nSl = (nSl - c2) * (1.0 - 1e-12);
      exact = false;
      if (exact_every_term) {
        nS = s_norm_exact();
        nSl = nSu = nS;
        exact = true;
      }
      trace(1.0, c2, nS);
      double* tmp = Dc;
      Dc = Dn;
      Dn = tmp;
      dpar ^= 1;
    }
  } else {
    // no S term at all (tol * ||S|| infinite): the phases below read S = Vw_1
    unsigned c[Q];
    bool v[Q];
    cols(LS, c, v);
    for (int t = cta; t < ntiles; t += ncta)
      for (int wt = warp; wt < a.tile / LS.RW; wt += kWarps) {
        const int base = t * a.tile + wt * LS.RW;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int row = base + rr * LS.gpw + LS.g;
          if (row >= n) continue;
#pragma unroll
          for (int q = 0; q < Q; ++q)
            if (v[q]) {
              double x[V];
#pragma unroll
              for (int e = 0; e < V; ++e) {
                const int cc = int(c[q]) + e;
                const int j = cc / r, i = cc - j * r;
                const int sc = j == 0 ? 0 : p + 1 - j;
                x[e] = a.D0[size_t(row) * size_t(p1) + sc] * __ldg(a.g + i);
              }
              Vio<V>::st(a.S + (unsigned(row) * ldb + c[q]), x);
            }
        }
      }
    double dmy1, dmy2;
    sync_step(0ull, 0ull, dmy1, dmy2);
  }
  for (; err == kStOk;) {
    const double lhs = c1 + c2;
    bool cont;
    if (exact) {
      cont = lhs > a.tol * nS;
    } else if (lhs > a.tol * nSu) {
      cont = true;
    } else if (lhs <= a.tol * nSl) {
      cont = false;
    } else {
      nS = s_norm_exact();
      nSl = nSu = nS;
      exact = true;
      cont = lhs > a.tol * nS;
    }
    if (!cont) break;
    if (k >= 500) {
      err = kStSeriesCap;
      err_idx = 500;
      break;
    }
    ++k;
    c1 = c2;
    sigma *= k;
    unsigned long long mdb = 0;
    {
      unsigned c[Q];
      bool v[Q];
      cols(LS, c, v);
      int jj[Q][V];
      double kd[Q][V], ka[Q][V], tos[Q][V];
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int e = 0; e < V; ++e) {
          const int cc = int(c[q]) + e;
          jj[q][e] = v[q] ? cc / r : 0;
          kd[q][e] = v[q] ? __ldg(a.colKd + cc) : 0.0;
          ka[q][e] = v[q] ? __ldg(a.colKa + cc) : 0.0;
          tos[q][e] = v[q] ? __ldg(a.colTos + cc) : 0.0;
        }
      auto sbody = [&](int base, const int* rp, const int* ci, const double* avs) {
          // row-local streams (independent of the CSR slice): before or after
          // the gather (Cfg::LATE)
          double vw[R][Q][V], vwl[R][Q][V], so[R][Q][V], ds[R][Q][V], acc[R][Q][V];
          bool vq[R][Q];
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
              for (int e = 0; e < V; ++e) acc[rr][q][e] = 0.0;
          auto streams = [&]() {
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const int row = base + rr * LS.gpw + LS.g;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              vq[rr][q] = row < n && v[q];
              const unsigned o = unsigned(row) * ldb + c[q];
#pragma unroll
              for (int e = 0; e < V; ++e) {
                vw[rr][q][e] = vwl[rr][q][e] = so[rr][q][e] = ds[rr][q][e] = 0.0;
              }
              if (vq[rr][q]) {
                ld_s<!CL>(a.Vw + o, vw[rr][q]);
                ld_s<!CL>(a.S + o, so[rr][q]);
                if (has_xi) Vio<V>::ld(Dc + o, ds[rr][q]);
                if (vwl_vec) {
                  if (jj[q][0] >= 2) ld_s<!CL>(a.Vw + (o - unsigned(r)), vwl[rr][q]);
                } else {
#pragma unroll
                  for (int e = 0; e < V; ++e)
                    if (jj[q][e] >= 2) vwl[rr][q][e] = ld1_s<!CL>(a.Vw + (o + e - unsigned(r)));
                }
              }
            }
          }
          };
          if constexpr (!Cfg<Q, V, RR>::LATE) streams();
          gather_tile<Q, V, R, B, PART, HINT, EC>(a, LS, rp, ci, avs, ldb, Dc, gtab[dpar], c, v, acc);
          if constexpr (Cfg<Q, V, RR>::LATE) streams();
          double vn[R][Q][V], dn[R][Q][V], sn[R][Q][V];
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
              for (int e = 0; e < V; ++e) {
                // Vw = Vw * Kiter: ascending source column from +0 (:98)
                double g2 = 0.0;
                if (jj[q][e] >= 2) g2 = g2 + vwl[rr][q][e] * ka[q][e];
                g2 = g2 + vw[rr][q][e] * kd[q][e];
                vn[rr][q][e] = g2;
                // D = (A - xi I) D (:99), * t_i/s (:101), + Vw (:102)
                double y = acc[rr][q][e];
                if (has_xi) y = y - a.xi * ds[rr][q][e];
                y = y * tos[q][e];
                dn[rr][q][e] = y + g2;
                sn[rr][q][e] = so[rr][q][e] + dn[rr][q][e] / sigma;  // S += D/sigma (:105)
              }
          __syncwarp();  // every lane has read its Vw[c - r] before any lane writes Vw
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const int row = base + rr * LS.gpw + LS.g;
            double ad[Q][V];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              if (vq[rr][q]) {
                const unsigned o = unsigned(row) * ldb + c[q];
                st_s<!CL>(a.Vw + o, vn[rr][q]);
                Vio<V>::st(Dn + o, dn[rr][q]);
                st_s<!CL>(a.S + o, sn[rr][q]);
              }
#pragma unroll
              for (int e = 0; e < V; ++e) ad[q][e] = vq[rr][q] ? fabs(dn[rr][q][e]) : 0.0;
            }
            const double rd = group_rowsum<Q, V>(ad, LS.G, LS.qp);
            if (row < n) mdb = umax64(mdb, abs_bits(rd));
          }
                };
      if constexpr (LEAN) {
        // grid-stride warp tiles, row_ptr slice read per tile, entries
        // gathered straight from global memory (no staging pipeline)
        // Q = R = 1, V = 2: the same arithmetic as sbody, statement for
        // statement, with the lane's row handled inline
        (void)sbody;
        const int gw = cta * kWarps + warp, nw = ncta * kWarps;
        for (int base = gw * LS.RW; base < n; base += nw * LS.RW) {
          const int row = base + LS.g;
          const bool vq0 = row < n && v[0];
          const unsigned o = unsigned(row) * ldb + c[0];
          double vw0 = 0.0, vw1 = 0.0, so0 = 0.0, so1 = 0.0, ds0 = 0.0, ds1 = 0.0, vl0 = 0.0,
                 vl1 = 0.0;
          if (vq0) {
            double t2[2];
            ld_s<true, 2>(a.Vw + o, t2);
            vw0 = t2[0];
            vw1 = t2[1];
            ld_s<true, 2>(a.S + o, t2);
            so0 = t2[0];
            so1 = t2[1];
            if (has_xi) {
              Vio<2>::ld(Dc + o, t2);
              ds0 = t2[0];
              ds1 = t2[1];
            }
            if (vwl_vec) {
              if (jj[0][0] >= 2) {
                ld_s<true, 2>(a.Vw + (o - unsigned(r)), t2);
                vl0 = t2[0];
                vl1 = t2[1];
              }
            } else {
              if (jj[0][0] >= 2) vl0 = ld1_s<true>(a.Vw + (o - unsigned(r)));
              if (jj[0][1] >= 2) vl1 = ld1_s<true>(a.Vw + (o + 1 - unsigned(r)));
            }
          }
          double a0 = 0.0, a1 = 0.0;
          if (vq0) {
            const int e1 = __ldg(a.rp + row + 1);
            for (int e = __ldg(a.rp + row); e < e1; ++e) {
              double x[2];
              Vio<2>::ld(Dc + unsigned(__ldg(a.ci + e)) * ldb + c[0], x);
              const double w = __ldg(a.av + e);
              a0 = a0 + w * x[0];
              a1 = a1 + w * x[1];
            }
          }
          // the lane's coefficients from shared memory (volatile: re-read per
          // row, not hoisted into registers held across the gather)
          const volatile double* vk = s_coef;
          const int c0 = v[0] ? int(c[0]) : 0;
          const double kd0 = vk[c0], kd1 = vk[c0 + 1], ka0 = vk[64 + c0], ka1 = vk[64 + c0 + 1];
          const double ts0 = vk[128 + c0], ts1 = vk[128 + c0 + 1];
          // columns of blocks j < 2 have Ka = +0 and Vw[c - r] not loaded
          // (+0): 0 + (+0 * +0) = +0, so the unconditional form is bitwise
          // the branch of the reference order (:98)
          double g0 = 0.0, g1 = 0.0;
          g0 = g0 + vl0 * ka0;
          g0 = g0 + vw0 * kd0;
          g1 = g1 + vl1 * ka1;
          g1 = g1 + vw1 * kd1;
          double y0 = a0, y1 = a1;
          if (has_xi) {
            y0 = y0 - a.xi * ds0;
            y1 = y1 - a.xi * ds1;
          }
          y0 = y0 * ts0;
          y1 = y1 * ts1;
          const double d0 = y0 + g0, d1 = y1 + g1;
          const double s0 = so0 + d0 / sigma, s1 = so1 + d1 / sigma;
          __syncwarp();  // every lane has read its Vw[c - r] before any lane writes Vw
          if (vq0) {
            const double vn2[2] = {g0, g1}, dn2[2] = {d0, d1}, sn2[2] = {s0, s1};
            st_s<true, 2>(a.Vw + o, vn2);
            Vio<2>::st(Dn + o, dn2);
            st_s<true, 2>(a.S + o, sn2);
          }
          const double ad[1][2] = {{vq0 ? fabs(d0) : 0.0, vq0 ? fabs(d1) : 0.0}};
          const double rd = group_rowsum<1, 2>(ad, LS.G, LS.qp);
          if (row < n) mdb = umax64(mdb, abs_bits(rd));
        }
      } else {
        run_tiles<DYN, CL, LAT>(a, LS, ntiles, warp, cta, ncta, a.slots + 4 * (step % 3) + 2, pp,
                                lane, crp, cci, cav, sbody);
      }
    }
    double maxD, dmy;
    sync_step(mdb, mdb, maxD, dmy);
    c2 = maxD / sigma;  // :103
    if (!isfinite(c2)) {
      err = kStSeriesDiverged;
      err_idx = k;
      break;
    }
    nSu = (nSu + c2) * (1.0 + 1e-12);
    nSl = (nSl - c2) * (1.0 - 1e-12);
    exact = false;
    if (exact_every_term) {
      nS = s_norm_exact();
      nSl = nSu = nS;
      exact = true;
    }
    trace(1.0, c2, nS);
    double* tmp = Dc;
    Dc = Dn;
    Dn = tmp;
    dpar ^= 1;
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
    unsigned c[Q];
    bool v[Q], vl[Q];
    cols(LF, c, v);
#pragma unroll
    for (int q = 0; q < Q; ++q) vl[q] = v[q] && int(c[q]) < r;
    run_tiles<DYN, CL, LAT>(a, LF, ntiles, warp, cta, ncta, a.slots + 4 * (step % 3) + 2, pp, lane,
                       crp, cci, cav,
              [&](int base, const int* rp, const int* ci, const double* avs) {
        double acc[R][Q][V];
#pragma unroll
        for (int rr = 0; rr < R; ++rr)
#pragma unroll
          for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int e = 0; e < V; ++e) acc[rr][q][e] = 0.0;
        // gathers S block-0 columns (left F columns live at the same column
        // index in S); a pair straddling the left/right split gathers one
        // extra column, unused
        gather_tile<Q, V, R, B, PART, HINT, EC>(a, LF, rp, ci, avs, ldb, a.S, gtab[2], c, vl, acc);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int row = base + rr * LF.gpw + LF.g;
          const bool rv = row < n;
          double f[Q][V], af[Q][V];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
#pragma unroll
            for (int e = 0; e < V; ++e) {
              f[q][e] = 0.0;
              const int cc = int(c[q]) + e;
              if (rv && v[q]) {
                const int i = cc < r ? cc : cc - r;
                const size_t srow = size_t(row) * ldb + size_t(p) * size_t(r);
                if (cc < r) {
                  const double sc = acc[rr][q][e] * __ldg(a.t + i);
                  f[q][e] = sc + __ldg(a.V + row);
                } else {
                  f[q][e] = a.S[srow + i];
                }
                if (!sweeps && cc < r) {
                  // assembly W = F_L + fl(F_R * alpha) (:148-154)
                  double wv = f[q][e];
                  double fr = 0.0;
                  if (p > 0) {
                    fr = a.S[srow + i];
                    wv = wv + fr * __ldg(a.alpha + i);
                  }
                  a.W[size_t(i) * size_t(n) + row] = wv;
                  if (a.FLo) a.FLo[size_t(i) * size_t(n) + row] = f[q][e];
                  if (a.FRo) a.FRo[size_t(i) * size_t(n) + row] = fr;
                }
              }
              af[q][e] = fabs(f[q][e]);
            }
            if (sweeps && rv && v[q]) {
              const unsigned o = unsigned(row) * ldf + c[q];
              Vio<V>::st(Fc + o, f[q]);
              Vio<V>::st(a.E + o, f[q]);
            }
          }
          if (sweeps) {
            const double rf = group_rowsum<Q, V>(af, LF.G, LF.qp);
            if (rv) mf = umax64(mf, abs_bits(rf));
          }
        }
              });
  }
  if (!sweeps) {
    finish(kStOk, 0, L_S, 1);
    return;
  }
  double fnorm, dummy;
  sync_step(mf, mf, fnorm, dummy);

  // ||E||_inf for the recovery stopping test (phi_block.cpp:124), bounded
  // like ||S|| above (E_kk = E_{kk-1} + F'_kk): an exact pass over E only for
  // an inconclusive term or when a trace is requested
  auto e_norm_exact = [&]() -> double {
    unsigned long long m = 0;
    unsigned c[Q];
    bool v[Q];
    cols(LF, c, v);
    for (int t = cta; t < ntiles; t += ncta)
      for (int wt = warp; wt < a.tile / LF.RW; wt += kWarps) {
        const int base = t * a.tile + wt * LF.RW;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int row = base + rr * LF.gpw + LF.g;
          const bool rv = row < n;
          double ae[Q][V];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            double x[V];
#pragma unroll
            for (int e = 0; e < V; ++e) x[e] = 0.0;
            if (rv && v[q]) Vio<V>::ld(a.E + (unsigned(row) * ldf + c[q]), x);
#pragma unroll
            for (int e = 0; e < V; ++e) ae[q][e] = (rv && v[q]) ? fabs(x[e]) : 0.0;
          }
          const double rs = group_rowsum<Q, V>(ae, LF.G, LF.qp);
          if (rv) m = umax64(m, abs_bits(rs));
        }
      }
    double mx, dmy;
    sync_step(m, m, mx, dmy);
    return mx;
  };

  // ================= recovery sweeps (phi_block.cpp:122-146)
  for (int sweep = 1; sweep < a.s_eff; ++sweep) {
    int kk = 0;
    double d1 = INF, d2 = fnorm, nE = fnorm;  // E = F
    trace(2.0, d2, nE);
    double nEl = nE, nEu = nE;
    bool eexact = true;
    for (;;) {
      const double lhs = d1 + d2;
      bool cont;
      if (eexact) {
        cont = lhs > a.tol * nE;
      } else if (lhs > a.tol * nEu) {
        cont = true;
      } else if (lhs <= a.tol * nEl) {
        cont = false;
      } else {
        nE = e_norm_exact();
        nEl = nEu = nE;
        eexact = true;
        cont = lhs > a.tol * nE;
      }
      if (!cont) break;
      if (kk >= 300) {
        err = kStRecoveryCap;
        err_idx = 300;
        break;
      }
      ++kk;
      d1 = d2;
      const double fac = a.single_variant ? a.t_single / (double(a.s_eff) * kk) : 0.0;
      unsigned long long mfb = 0;
      {
        unsigned c[Q];
        bool v[Q];
        double tosF[Q][V];
        cols(LF, c, v);
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
          for (int e = 0; e < V; ++e) {
            const int cc = int(c[q]) + e;
            const int i = cc < r ? cc : cc - r;
            tosF[q][e] = v[q] ? __ldg(a.colTos + i) : 0.0;
          }
        run_tiles<DYN, CL, LAT>(a, LF, ntiles, warp, cta, ncta, a.slots + 4 * (step % 3) + 2, pp, lane,
                       crp, cci, cav,
                  [&](int base, const int* rp, const int* ci, const double* avs) {
            double eo[R][Q][V], fs[R][Q][V], acc[R][Q][V];
            bool vq[R][Q];
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
#pragma unroll
              for (int q = 0; q < Q; ++q)
#pragma unroll
                for (int e = 0; e < V; ++e) acc[rr][q][e] = 0.0;
            auto streams = [&]() {  // before or after the gather (Cfg::LATE)
#pragma unroll
              for (int rr = 0; rr < R; ++rr) {
                const int row = base + rr * LF.gpw + LF.g;
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                  vq[rr][q] = row < n && v[q];
                  const unsigned o = unsigned(row) * ldf + c[q];
#pragma unroll
                  for (int e = 0; e < V; ++e) eo[rr][q][e] = fs[rr][q][e] = 0.0;
                  if (vq[rr][q]) {
                    ld_s<!CL>(a.E + o, eo[rr][q]);
                    if (has_xi) Vio<V>::ld(Fc + o, fs[rr][q]);
                  }
                }
              }
            };
            if constexpr (!Cfg<Q, V, RR>::LATE) streams();
            gather_tile<Q, V, R, B, PART, HINT, EC>(a, LF, rp, ci, avs, ldf, Fc, gtab[3 + fpar], c, v, acc);
            if constexpr (Cfg<Q, V, RR>::LATE) streams();
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
              const int row = base + rr * LF.gpw + LF.g;
              double y[Q][V], en[Q][V], ay[Q][V];
#pragma unroll
              for (int q = 0; q < Q; ++q) {
#pragma unroll
                for (int e = 0; e < V; ++e) {
                  double yv = acc[rr][q][e];
                  if (has_xi) yv = yv - a.xi * fs[rr][q][e];
                  if (a.single_variant) {
                    yv = fac * yv;  // phi_single.cpp:106
                  } else {
                    yv = yv / double(kk);  // phi_block.cpp:132
                    yv = yv * tosF[q][e];  // :134-135
                  }
                  y[q][e] = yv;
                  en[q][e] = eo[rr][q][e] + yv;  // E += F (:138)
                  ay[q][e] = vq[rr][q] ? fabs(yv) : 0.0;
                }
                if (vq[rr][q]) {
                  const unsigned o = unsigned(row) * ldf + c[q];
                  st_s<!CL>(Fn + o, y[q]);  // next term only: evict-first
                  st_s<!CL>(a.E + o, en[q]);
                }
              }
              const double ry = group_rowsum<Q, V>(ay, LF.G, LF.qp);
              if (row < n) mfb = umax64(mfb, abs_bits(ry));
            }
                  });
      }
      double maxF2, dmy;
      sync_step(mfb, mfb, maxF2, dmy);
      d2 = maxF2;
      if (!isfinite(d2)) {
        err = kStRecoveryDiverged;
        err_idx = kk;
        break;
      }
      nEu = (nEu + d2) * (1.0 + 1e-12);
      nEl = (nEl - d2) * (1.0 - 1e-12);
      eexact = false;
      if (exact_every_term) {
        nE = e_norm_exact();
        nEl = nEu = nE;
        eexact = true;
      }
      trace(3.0, d2, nE);
      double* tmp = Fc;
      Fc = Fn;
      Fn = tmp;
      fpar ^= 1;
    }
    if (err != kStOk) break;
    if (lead) a.lensF[sweep - 1] = kk;

    // ---- sweep end (:141-145): E *= mu; Sadv = Sadv*Jexp; F refresh
    // phase A (S layout): Sadv blocks 1..p in place, ascending source column
    {
      unsigned c[Q];
      bool v[Q];
      cols(LS, c, v);
      for (int t = cta; t < ntiles; t += ncta)
        for (int wt = warp; wt < a.tile / LS.RW; wt += kWarps) {
          const int base = t * a.tile + wt * LS.RW;
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const int row = base + rr * LS.gpw + LS.g;
            double nv[Q][V];
            bool wq[Q][V];
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
              for (int e = 0; e < V; ++e) {
                const int cc = int(c[q]) + e;
                const int j = v[q] ? cc / r : 0, i = cc - j * r;
                wq[q][e] = row < n && v[q] && j >= 1;
                nv[q][e] = 0.0;
                if (wq[q][e]) {
                  const double* srow = a.S + size_t(row) * ldb;
                  const double* cj = a.jc + size_t(i) * size_t(p + 1);
                  double accv = 0.0;
                  for (int l = 1; l <= j; ++l) accv = accv + srow[l * r + i] * __ldg(cj + (j - l));
                  nv[q][e] = accv;
                }
              }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
              for (int e = 0; e < V; ++e)
                if (wq[q][e]) a.S[size_t(row) * ldb + c[q] + e] = nv[q][e];
          }
        }
    }
    __syncthreads();
    // phase B (F layout): F_L = E_L*mu, F_R = E_R*mu + Sadv_p; E = F
    const bool last = sweep == a.s_eff - 1;
    unsigned long long mfe = 0;
    {
      unsigned c[Q];
      bool v[Q];
      cols(LF, c, v);
      for (int t = cta; t < ntiles; t += ncta)
        for (int wt = warp; wt < a.tile / LF.RW; wt += kWarps) {
          const int base = t * a.tile + wt * LF.RW;
#pragma unroll
          for (int rr = 0; rr < R; ++rr) {
            const int row = base + rr * LF.gpw + LF.g;
            const bool rv = row < n;
            double f[Q][V], af[Q][V];
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
              for (int e = 0; e < V; ++e) {
                f[q][e] = 0.0;
                const int cc = int(c[q]) + e;
                if (rv && v[q]) {
                  const int i = cc < r ? cc : cc - r;
                  const size_t srow = size_t(row) * ldb + size_t(p) * size_t(r);
                  const double en = a.E[size_t(row) * ldf + cc] * __ldg(a.mu + i);
                  double fv = en;
                  if (cc >= r) fv = en + a.S[srow + i];
                  f[q][e] = fv;
                  if (last && cc < r) {
                    double wv = fv;
                    double fr = 0.0;
                    if (p > 0) {
                      const double er = a.E[size_t(row) * ldf + r + i] * __ldg(a.mu + i);
                      fr = er + a.S[srow + i];
                      wv = wv + (a.single_variant ? __ldg(a.alpha + i) * fr : fr * __ldg(a.alpha + i));
                    }
                    a.W[size_t(i) * size_t(n) + row] = wv;
                    if (a.FLo) a.FLo[size_t(i) * size_t(n) + row] = fv;
                    if (a.FRo) a.FRo[size_t(i) * size_t(n) + row] = fr;
                  }
                }
                af[q][e] = (rv && v[q]) ? fabs(f[q][e]) : 0.0;
              }
            if (!last) {
              __syncwarp();
#pragma unroll
              for (int q = 0; q < Q; ++q)
                if (rv && v[q]) {
                  const unsigned o = unsigned(row) * ldf + c[q];
                  Vio<V>::st(Fc + o, f[q]);
                  Vio<V>::st(a.E + o, f[q]);
                }
              const double rf = group_rowsum<Q, V>(af, LF.G, LF.qp);
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

// sets the variant's dynamic shared memory limit and returns its co-resident
// CTAs per SM; both are per device and fixed, so they are cached per (device,
// block size) -- the calls cost ~10 us each on every evaluation otherwise
template <int Q, int V, int R, bool PART, bool DYN, int BO, bool CL, bool LAT>
cudaError_t eval_occupancy(int block, int* per_sm) {
  static std::atomic<long long> cache[kOccCacheDevices];  // (block << 32) | per_sm + 1
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const bool cacheable = dev >= 0 && dev < kOccCacheDevices;
  if (cacheable) {
    const long long c = cache[dev].load(std::memory_order_relaxed);
    if (c != 0 && (c >> 32) == block) {
      *per_sm = int(c & 0xffffffffLL) - 1;
      return cudaSuccess;
    }
  }
  e = cudaFuncSetAttribute(k_phimv_block<Q, V, R, PART, DYN, BO, CL, LAT>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(PipeCfg<Q, V, R, PART, DYN, BO, CL, LAT>::bytes));
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      per_sm, k_phimv_block<Q, V, R, PART, DYN, BO, CL, LAT>, block,
      PipeCfg<Q, V, R, PART, DYN, BO, CL, LAT>::bytes);
  if (e == cudaSuccess && cacheable)
    cache[dev].store((static_cast<long long>(block) << 32) | (*per_sm + 1),
                     std::memory_order_relaxed);
  return e;
}

template <int Q, int V, int R, bool PART, bool DYN, int BO = 0, bool CL = false, bool LAT = false>
EvalKernel eval_kernel() {
  return EvalKernel{
      reinterpret_cast<const void*>(k_phimv_block<Q, V, R, PART, DYN, BO, CL, LAT>),
      eval_occupancy<Q, V, R, PART, DYN, BO, CL, LAT>, PipeCfg<Q, V, R, PART, DYN, BO, CL, LAT>::bytes};
}

// cluster-mode variants exist for single-chunk rows (Q == 1) only
template <int Q, int V, int R, int BO>
EvalKernel eval_kernel_cluster() {
  if constexpr (Q == 1)
    return eval_kernel<Q, V, R, true, false, BO, true>();
  else
    return EvalKernel{nullptr, nullptr, 0};
}

}  // namespace

// one instantiated (Q, V, R) with gather batch BO (0: Cfg's): unpartitioned
// static or dynamic-tail kernels, partitioned kernels always with the
// dynamic tail
#define PHX_EVAL_KERNELS(q, v, r, bo)                          \
  if (cluster)                                                 \
    return false; /* cluster variants: phx_eval_cl.cu */       \
  else if (part)                                               \
    *out = eval_kernel<q, v, r, true, true, bo>();             \
  else if (dyn)                                                \
    *out = eval_kernel<q, v, r, false, true, bo>();            \
  else                                                         \
    *out = eval_kernel<q, v, r, false, false, bo>();
#define PHX_EVAL_CASE(q, v, r)                                 \
  if (QT == q && V == v && R == r) {                           \
    PHX_EVAL_KERNELS(q, v, r, 0)                               \
    return out->fn != nullptr;                                 \
  }
// ... and a second, short batch bs used for operators whose rows fit it
#define PHX_EVAL_CASE2(q, v, r, bs)                            \
  if (QT == q && V == v && R == r) {                           \
    if (small) {                                               \
      PHX_EVAL_KERNELS(q, v, r, bs)                            \
    } else {                                                   \
      PHX_EVAL_KERNELS(q, v, r, 0)                             \
    }                                                          \
    return out->fn != nullptr;                                 \
  }

}  // namespace phx
