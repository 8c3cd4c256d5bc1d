// The bulk-copy persistent phimv_block kernel (phi_block.cpp:48-157, Alg. 3)
// for large operators, sm_100a.
//
// Same algorithm, operation order and stopping logic as k_phimv_block
// (phx_eval_kernel.cuh; bit-for-bit the oracle), but the two phases that carry
// almost all of the traffic -- the S-series terms (phi_block.cpp:93-106) and
// the recovery terms (:124-139) -- run as a warp-specialised TMA-engine
// pipeline instead of register gathers:
//
//   * one PRODUCER warp per CTA grabs tiles of kPlanT rows dynamically (batches
//     of 4 positions from the step's counter, so all CTAs sweep the rows
//     together and the gathers' L2 reuse window stays small) and, from the
//     operator's tile plan (phx_plan.cpp), issues cp.async.bulk copies of
//     every contiguous range the tile needs -- its row_ptr / slot / value
//     slices, the gather window, the offset groups, single rows, and the
//     row-local accumulator tiles -- into a ring of shared-memory stages,
//     completing on an mbarrier (complete_tx);
//   * eight CONSUMER warps wait on the stage's barrier, accumulate every row's
//     entries in CSR order from shared memory (one-byte slots), run the same
//     fused epilogue (J-term, shift, scaling, D' / S' or F' / E', |.| row
//     sums) and stream the results to HBM with evict-first stores, then release
//     the stage.
//
// Nothing a consumer reads comes from global memory, so memory-level
// parallelism no longer depends on registers: C3's S term went from 0.47 of
// the HBM roofline (register gathers) to 0.73 in the microbenchmark
// (tools/microbench_c3.cu, profiles/r2_microbench_c3.jsonl).  The remaining
// phases (init, the peeled first S term, promotion, sweep end, exact norm
// passes: a few percent of the traffic) run as plain grid-stride loops.
//
// Compiled with --fmad=false: each multiply and add rounds separately.
#include <cooperative_groups.h>

#include "phx_eval_kernel.cuh"

namespace cg = cooperative_groups;

namespace phx {
namespace {

// PHX_CHECKS=1 (libphx_checked.so, `make checked`): device-side bounds checks
// on every staged copy and slot -- the self-check used in place of
// compute-sanitizer, which this pool does not allow
#ifndef PHX_CHECKS
#define PHX_CHECKS 0
#endif
#define PHX_CHECK(cond)              \
  do {                               \
    if (PHX_CHECKS && !(cond)) __trap(); \
  } while (0)

constexpr int kBW = kBulkConsumers + 1;  // warps per CTA
constexpr int kProd = kBulkConsumers;    // the producer warp
constexpr int kPB = 4;                   // tile positions per counter grab
constexpr int kMaxMerge = 8;             // window-only plans: tiles merged per stage

// columns per consumer lane of a bulk phase (compile time)
template <int N>
struct IC {
  static constexpr int value = N;
};
#ifndef PHX_CPL4
#define PHX_CPL4 1  // S terms with 4 columns per consumer lane
#endif
#ifndef PHX_FAST_S
#define PHX_FAST_S 1  // specialised S-term / recovery-term consumers (see s_fast, r_fast)
#endif

// canonical |.| row sum (group_rowsum's pairwise tree) of a CPL-4 row: the
// lane holds columns (c, c+1) and (c + 2GL, c + 2GL + 1); the tree's levels
// below 2GL columns run on both halves, its last level is lo + hi
__device__ __forceinline__ double quad_rowsum(const double (&v)[4], int GL) {
  double lo = v[0] + v[1], hi = v[2] + v[3];
#pragma unroll
  for (int m = 1; m < 32; m <<= 1)
    if (m < GL) {  // GL is warp-uniform
      lo = lo + __shfl_xor_sync(kFull, lo, m);
      hi = hi + __shfl_xor_sync(kFull, hi, m);
    }
  return lo + hi;
}

__device__ __forceinline__ unsigned su32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// the same wait with a suspend-time hint: a warp whose phase has not
// completed sleeps (up to the hint) instead of re-issuing the probe
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx)
               : "memory");
}
// global -> shared bulk copy (TMA engine), completion counted on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// CTA max of two bit patterns (kBW warps) -> one atomicMax each into the slot
__device__ __forceinline__ void publish_b(unsigned long long a, unsigned long long b,
                                          unsigned long long* slot,
                                          unsigned long long (*red)[kBW]) {
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
    for (int q = 0; q < kBW; ++q) {
      ma = umax64(ma, red[0][q]);
      mb = umax64(mb, red[1][q]);
    }
    atomicMax(slot, ma);
    atomicMax(slot + 1, mb);
  }
  __syncthreads();
}

// PART: a row-partitioned operator.  The launch runs parts
// plo .. plo+pcount-1 with the CTAs split evenly (interleaved); a CTA binds its part's
// row-local buffers, CSR and tile plan (rows are part-local from there on).
// The plan's window / group / single source rows are GLOBAL rows: the
// producer cuts every staged range at the part boundaries and copies each
// piece from its owner's buffer (peer-GPU memory over NVLink in a multi-GPU
// run), so the consumers -- and every row's arithmetic -- are unchanged.  The
// per-step maxima are combined through the parts' mailboxes (system scope),
// which is also the step barrier across devices.
#ifdef PHX_BULK_MAXNREG
#define PHX_BULK_BOUNDS __maxnreg__(PHX_BULK_MAXNREG)
#else
#ifndef PHX_BULK_MINB
#define PHX_BULK_MINB (kBulkConsumers > 8 ? 1 : 2)  // CTAs per SM the register budget is sized for
#endif
#define PHX_BULK_BOUNDS __launch_bounds__(kBulkThreads, PHX_BULK_MINB)
#endif
// the kernel's parameter: one BlockArgs, or (PART) every part's BlockArgs
// (n = the part's rows, its buffers, CSR and plan) in the parameter space --
// indexed by the CTA's part, so the per-part arguments stay in the constant
// bank like the unpartitioned kernel's instead of a shared-memory copy
template <bool PART>
struct BulkParam {
  using type = BlockArgs;
};
template <>
struct BulkParam<true> {
  using type = BulkPartArgs;
};
__device__ __forceinline__ const BlockArgs& part_args(const BlockArgs& g, int) { return g; }
__device__ __forceinline__ const BlockArgs& part_args(const BulkPartArgs& g, int q) { return g.pa[q]; }

// SW: the launch has recovery sweeps (s_eff > 1).  Launches without (C2, C3,
// C4: s_eff = 1) run an instantiation that compiles no recovery, sweep-end or
// F-promotion code, so the S-term loop gets the registers to itself.
template <bool PART, bool SW = true>
__global__ void PHX_BULK_BOUNDS k_phimv_bulk(const __grid_constant__ typename BulkParam<PART>::type gp) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ unsigned long long bar_full[kBulkMaxStages], bar_empty[kBulkMaxStages];
  __shared__ unsigned long long red[2][kBW];
  __shared__ __align__(16) int pdesc[2][kPB][kPlanDesc];  // producer: descriptor batches
  __shared__ const double* gtab[5][PART ? kMaxParts : 1];  // [D0, D1, S, F0, F1][part]
  __shared__ int sbnd[PART ? kMaxParts + 1 : 1];           // part row boundaries (global)
  __shared__ double gmax[2];
  // the S-term column coefficients Kd, Ka, t/s and Ka of column c - r
  // (columns 0..31, zeros past w) for the specialised S-term consumer
  __shared__ __align__(16) double ctab[4][32];
  const double INF = __longlong_as_double(0x7FF0000000000000ll);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const BlockArgs& ga = part_args(gp, 0);  // the fields common to all parts
  int my = 0, cta = int(blockIdx.x), ncta = int(gridDim.x);
  const PartTab* T = nullptr;
  int Ng = ga.n;  // global rows
  if (PART) {
    // parts interleaved over the CTAs (CTA b works for part plo + b mod
    // pcount): on one device every part's CTAs spread over all SMs alike
    const int per = int(gridDim.x) / ga.pcount;
    my = ga.plo + int(blockIdx.x) % ga.pcount;
    cta = int(blockIdx.x) / ga.pcount;
    ncta = per;
    T = ga.ptab + my;
    Ng = ga.ptab[ga.nparts - 1].row0 + ga.ptab[ga.nparts - 1].nrows;
    for (int q = threadIdx.x; q < ga.nparts; q += blockDim.x) {
      const PartTab& U = ga.ptab[q];
      gtab[0][q] = U.D0;
      gtab[1][q] = U.D1;
      gtab[2][q] = U.S;
      gtab[3][q] = U.F0;
      gtab[4][q] = U.F1;
      sbnd[q] = U.row0;
    }
    if (threadIdx.x == 0) sbnd[ga.nparts] = Ng;
    __syncthreads();
  }
  const BlockArgs& a = part_args(gp, my);
  const int row0 = PART ? T->row0 : 0;
  const int NS = a.bulk_ns, SB = a.bulk_stage_bytes;
  const bool sleepw = (a.bulk_flags & 2) != 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], kBulkConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int n = a.n, r = a.r, p = a.p, p1 = p + 1;
  const int w = a.w, fc = a.fcols;
  const unsigned ldb = unsigned(a.ldb), ldf = unsigned(a.ldf);
  const bool has_xi = a.xi != 0.0;
  const bool master = blockIdx.x == 0 && threadIdx.x == 0 && (!PART || ga.plo == 0);
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;  // writes this launch's status
  const int nblk = (n + kPlanT - 1) / kPlanT;  // row blocks = plan tiles
  // ring position (the same sequence in the producer and the consumers):
  // stage index and the parity of its use, advanced without division
  int kst = 0;
  unsigned kpar = 0;
  auto ring_next = [&]() {
    if (++kst == NS) {
      kst = 0;
      kpar ^= 1u;
    }
  };
#ifndef PHX_PROBE
#define PHX_PROBE 0  // developer diagnostics: SM-cycle totals of ring waits and work
#endif
  long long pr_pwait = 0, pr_pwork = 0, pr_cwait = 0, pr_cwork = 0, pr_stages = 0;
  int step = 0, tr_len = 0;

  if (master && a.tstamp != nullptr && a.tstamp_cap > kCtaStampBase) {  // diagnostics: launch start
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    a.tstamp[kCtaStampBase - 1] = ns;
  }
  auto trace = [&](double kind, double x, double y) {
    if (master && a.trace != nullptr && tr_len + 3 <= a.trace_cap) {
      a.trace[tr_len] = kind;
      a.trace[tr_len + 1] = x;
      a.trace[tr_len + 2] = y;
    }
    tr_len += 3;
  };
  auto sync_step = [&](unsigned long long ma, unsigned long long mb, double& ra, double& rb) {
    unsigned long long* slot = a.slots + 4 * (step % 3);
    publish_b(ma, mb, slot, red);
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
      // part-local arrival; the part's last CTA publishes the part's maxima
      // into every part's mailbox (peer memory, double-buffered by step
      // parity) and everyone waits until all parts have published this step
      // (the same protocol as k_phimv_block's partitioned variants)
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
          const int buf = (step & 1) * ga.nparts;
          for (int q = 0; q < ga.nparts; ++q) {
            MailBox* mbx = ga.ptab[q].mbox + buf + my;
            mbx->a = A;
            mbx->b = Bv;
          }
          // release at system scope: the mailboxes may be peer-GPU memory
          __threadfence_system();
          for (int q = 0; q < ga.nparts; ++q) atomicExch_system(&(ga.ptab[q].mbox + buf + my)->gen, gen);
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
        if (master && a.tstamp != nullptr && step < a.tstamp_cap) {
          unsigned long long ns;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
          a.tstamp[step] = ns;
        }
        // the next step's bulk copies read other parts' rows written before
        // their arrival: make them visible to this CTA's async proxy
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence();
      }
      __syncthreads();
      ra = gmax[0];
      rb = gmax[1];
    }
    ++step;
  };
  // PHX_PROBE: lane 0 of the producer and of consumer warp 0 add their
  // totals into tstamp[cap - 8 ..] (SM cycles): producer wait / work,
  // consumer wait / work, consumer stages
  auto probe_flush = [&]() {
    if (PHX_PROBE && a.tstamp != nullptr && lane == 0 && (warp == kProd || warp == 0)) {
      unsigned long long* o = a.tstamp + (a.tstamp_cap - 8);
      if (warp == kProd) {
        atomicAdd(o + 0, (unsigned long long)pr_pwait);
        atomicAdd(o + 1, (unsigned long long)pr_pwork);
      } else {
        atomicAdd(o + 2, (unsigned long long)pr_cwait);
        atomicAdd(o + 3, (unsigned long long)pr_cwork);
        atomicAdd(o + 4, (unsigned long long)pr_stages);
      }
    }
  };
  auto finish = [&](int err, int idx, int L_S, int extra_steps) {
    probe_flush();
    if (lead) {
      a.status[0] = err;
      a.status[1] = idx;
      a.status[2] = L_S;
      a.status[3] = 0;
      a.status[4] = step + extra_steps;
      a.status[5] = min(tr_len, a.trace_cap);
    }
  };
  // plain phases: row blocks of kPlanT rows round-robin over the CTAs (the
  // same block -> CTA map in every plain phase), lane groups of G lanes over
  // the rows of a block; body(row, valid, lg) is called warp-uniformly
  auto plain_rows = [&](int G, auto&& body) {
    const int gpw = 32 / G, g = lane / G, lg = lane % G;
    for (int blk = cta; blk < nblk; blk += ncta)
      for (int r0 = warp * gpw; r0 < kPlanT; r0 += kBW * gpw) {
        const int row = blk * kPlanT + r0 + g;
        body(row, r0 + g < kPlanT && row < n, lg);
      }
  };
  const int GS = a.GS, GF = a.GF;

  // ================= the bulk phases: S term (kind 0) / recovery term (kind 1)
  // X: gather source (width `width`), A: stream A (Vw | E), B: stream B (S)
  // G: lanes per row of the output layout, ow: output width, width: row
  // width of the gather source X; gath(row_ptrs...) accumulates a row's
  // entries, epi(...) finishes it
  // Window-only plans (every gathered row inside its tile's window: banded
  // operators such as C5's bidiagonal rows) merge M consecutive tiles per
  // stage -- one window copy, one stream copy each -- with M as large as the
  // stage holds (narrow recovery terms: up to kMaxMerge): fewer, larger
  // copies and barrier handshakes per byte.  A sub-tile's slots address its
  // own window; the consumer shifts them into the merged window.
  // stage `cnt` GLOBAL rows from g0 of gather source X (row width `width`;
  // PART: buffer xsel of each owning part) into dst
  auto copy_rows = [&](unsigned char* dst, const double* X, int xsel, int width, int g0, int cnt,
                       unsigned long long* bf, unsigned long long pol) {
    const unsigned rb = unsigned(width) * 8u;
    if (!PART || (g0 >= row0 && g0 + cnt <= row0 + n)) {  // the part's own rows
      bulk_g2s(dst, X + size_t(g0 - row0) * width, unsigned(cnt) * rb, bf, pol);
      return;
    }
    while (cnt > 0) {
      int q = 0;
      while (sbnd[q + 1] <= g0) ++q;
      const int c = min(cnt, sbnd[q + 1] - g0);
      const double* src = (q == my ? X : gtab[xsel][q]) + size_t(g0 - sbnd[q]) * width;
      bulk_g2s(dst, src, unsigned(c) * rb, bf, pol);
      dst += size_t(c) * rb;
      g0 += c;
      cnt -= c;
    }
  };
  // cpl: columns per consumer lane (compile time).  2: lane lg of a row's G
  // lanes owns columns (2lg, 2lg+1).  4: lane lg of a row's G/2 lanes owns
  // (2lg, 2lg+1) and (G+2lg, G+2lg+1) -- twice the rows per warp, so the
  // per-entry slot / value / address work and the per-row loop, store and
  // shuffle work are shared by twice the columns; each staged row is still
  // read as contiguous 128-byte runs (no bank conflicts), and the canonical
  // row-sum tree is unchanged (its last level becomes the in-lane lo + hi).
  auto bulk_phase = [&](auto cpl, int G, int ow, int width, const double* X, int xsel, const double* A,
                        const double* B, auto&& gath, auto&& epi) -> unsigned long long {
    constexpr int CPL = decltype(cpl)::value;
    const int nst = (A ? 1 : 0) + (B ? 1 : 0);
    int M = 1;
    if (a.plan_merge)
      while (M < kMaxMerge &&
             bulk_stage(kPlanT * 2 * M + 2, a.plan_emax * 2 * M, width, nst, kPlanT * 2 * M).bytes <= SB)
        M *= 2;
    const int TM = kPlanT * M;  // rows per stage
    const BulkStage L = M > 1 ? bulk_stage(TM + 2, a.plan_emax * M, width, nst, TM)
                              : bulk_stage(a.plan_rows, a.plan_emax, width, nst);
    const int npos = (nblk + M - 1) / M;
    unsigned long long* ctr = a.slots + 4 * (step % 3) + 2;
    unsigned long long mx = 0;
    if (warp == kProd) {
      // the part's CSR / plan pointers in registers (PART: `a` lives in shared
      // memory, and the producer's per-tile chain should not wait on it)
      const int* const c_rp = a.rp;
      const uint8_t* const c_slot = a.plan_slot;
      const double* const c_av = a.av;
      const int* const c_desc = a.plan_desc;
      const int* const c_sgl = a.plan_sgl;
      // Batches of kPB tile positions from the step's counter.  The atomic
      // for a batch is issued one batch ahead; its descriptors are copied
      // (cp.async, 16 lanes x 16 B) into pdesc[nxt] while the current batch
      // is issued, so neither latency is on the producer's path.
      unsigned long long pfirst = 0, plast = 0;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pfirst));
      if (a.bulk_flags & 1)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(plast));
      else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(plast));
      auto fetch = [&](int pos, int buf) {
        const int q = pos + (lane >> 2);
        if (M == 1) {
          if (lane < 4 * kPB && q < nblk)
            cp_async16(&pdesc[buf][lane >> 2][4 * (lane & 3)],
                       c_desc + size_t(q) * kPlanDesc + 4 * (lane & 3));
        } else if (lane < 4 * kPB && (lane & 3) < 2 && q < npos) {
          // merged: e_lo from the first sub-tile's descriptor, e_hi from the last's
          const int sub = (lane & 1) ? min(q * M + M - 1, nblk - 1) : q * M;
          cp_async16(&pdesc[buf][lane >> 2][4 * (lane & 1)],
                     c_desc + size_t(sub) * kPlanDesc + 4 * (lane & 1));
        }
        cp_commit();
      };
      unsigned long long pa_ = 0, pb_ = 0;
      if (lane == 0) pa_ = atomicAdd(ctr, (unsigned long long)kPB);
      int posA = int(__shfl_sync(kFull, pa_, 0));  // positions: stages of M tiles
      fetch(posA, 0);
      if (lane == 0) pb_ = atomicAdd(ctr, (unsigned long long)kPB);
      int cur = 0;
      for (bool more = true; more;) {
        const int posB = int(__shfl_sync(kFull, pb_, 0));
        fetch(posB, cur ^ 1);
        if (lane == 0) pb_ = atomicAdd(ctr, (unsigned long long)kPB);  // used a batch later
        cp_wait_1();
        __syncwarp();
#pragma unroll 1
        for (int j = 0; j < kPB; ++j) {
          const int* d = pdesc[cur][j];
          // descriptors in processing order (merged stages: natural order)
          const int t = posA + j < npos ? (M == 1 ? d[5] : posA + j) : -1;
          const int s = kst;
          const long long pc0 = PHX_PROBE ? clock64() : 0;
          if (sleepw)
            mbar_wait_sleep(&bar_empty[s], kpar ^ 1u);
          else
            mbar_wait(&bar_empty[s], kpar ^ 1u);
          const long long pc1 = PHX_PROBE ? clock64() : 0;
          unsigned char* st = ring + size_t(s) * size_t(SB);
          unsigned long long* bf = &bar_full[s];
          const int nsgl = (t >= 0 && M == 1) ? d[1] : 0;
          if (lane == 0) {
            *reinterpret_cast<int*>(st + L.hdr) = t;
            if (t < 0) {
              mbar_arrive(bf);  // end of the phase: the consumers leave
            } else {
              const int base = t * TM, rows = min(TM, n - base);
              const int ng = M == 1 ? d[0] : 0;
              const int e_lo = d[3], e_hi = d[4];
              const int wlo = max(row0 + base - 1, 0), whi = min(row0 + base + rows + 1, Ng);
              const int c0 = e_lo & ~15, cn = (e_hi - c0 + 15) & ~15;  // slot bytes
              const int a0 = e_lo & ~1, an = (e_hi - a0 + 1) & ~1;    // values (16 B granules)
              const int rn = (rows + 1 + 3) & ~3;                     // row_ptr entries
              unsigned nrow = unsigned(whi - wlo + nsgl + ((A ? 1 : 0) + (B ? 1 : 0)) * rows);
              for (int g = 0; g < ng; ++g) nrow += unsigned(d[12 + g] & 0xffff);
              const unsigned rb = unsigned(width) * 8u;
              // the copies fit their stage regions
              PHX_CHECK(whi - wlo <= (M > 1 ? TM + 2 : kPlanT + 2));
              PHX_CHECK(e_hi - e_lo <= a.plan_emax * M && e_lo >= 0);
              PHX_CHECK(L.sl + cn <= L.rp && L.av + an * 8 <= L.sl && L.rp + rn * 4 <= L.hdr);
              PHX_CHECK(L.bytes <= SB && nsgl <= a.plan_sgl_cap);
              for (int g = 0; g < ng; ++g)
                PHX_CHECK((d[12 + g] >> 16) + (d[12 + g] & 0xffff) <= a.plan_rows &&
                          d[8 + g] >= 0 && d[8 + g] + (d[12 + g] & 0xffff) <= Ng);
              mbar_arrive_tx(bf, unsigned(rn * 4 + cn + an * 8) + nrow * rb);
              bulk_g2s(st + L.rp, c_rp + base, unsigned(rn) * 4u, bf, pfirst);
              if (cn) bulk_g2s(st + L.sl, c_slot + c0, unsigned(cn), bf, pfirst);
              if (an) bulk_g2s(st + L.av, c_av + a0, unsigned(an) * 8u, bf, pfirst);
              copy_rows(st + L.dr, X, xsel, width, wlo, whi - wlo, bf, plast);
              for (int g = 0; g < ng; ++g) {
                const int cnt = d[12 + g] & 0xffff, dst = d[12 + g] >> 16;
                copy_rows(st + L.dr + dst * int(rb), X, xsel, width, d[8 + g], cnt, bf, plast);
              }
              if (A) bulk_g2s(st + L.sa, A + size_t(base) * width, unsigned(rows) * rb, bf, pfirst);
              if (B) bulk_g2s(st + L.sb, B + size_t(base) * width, unsigned(rows) * rb, bf, pfirst);
            }
          }
          if (t >= 0 && lane < nsgl) {  // single rows, one lane each
            const int col = __ldg(c_sgl + d[2] + lane);
            copy_rows(st + L.dr + (kPlanT + 2 + lane) * width * 8, X, xsel, width, col, 1, bf, plast);
          }
          __syncwarp();
          if (PHX_PROBE) {
            pr_pwait += pc1 - pc0;
            pr_pwork += clock64() - pc1;
          }
          ring_next();
          if (t < 0) {
            more = false;
            break;
          }
        }
        posA = posB;
        cur ^= 1;
      }
      cp_wait_all();  // the last prefetch (positions past the end) drains
      __syncwarp();
      return mx;
    }
    // ---- consumers
    const int GL = CPL == 4 ? (G > 1 ? G >> 1 : 1) : G;  // lanes per row
    const int gpw = 32 / GL, g = lane / GL, lg = lane % GL;
    const int c = 2 * lg, ch = c + 2 * GL;  // ch: the lane's second pair (CPL 4)
    const bool cv = c < ow, cvh = ch < ow;
    for (;;) {
      const int s = kst;
      const long long cc0 = PHX_PROBE ? clock64() : 0;
      if (sleepw)
        mbar_wait_sleep(&bar_full[s], kpar);
      else
        mbar_wait(&bar_full[s], kpar);
      const long long cc1 = PHX_PROBE ? clock64() : 0;
      const unsigned char* st = ring + size_t(s) * size_t(SB);
      const int t = *reinterpret_cast<const int*>(st + L.hdr);
      ring_next();
      if constexpr (CPL == 8) {
        // the specialised S-term consumer: `gath` is the stage body
        if (t >= 0) mx = umax64(mx, gath(st, L, t, TM, M));
      } else if (t >= 0) {
        const int* rps = reinterpret_cast<const int*>(st + L.rp);
        const double* dr = reinterpret_cast<const double*>(st + L.dr);
        const double* sa = reinterpret_cast<const double*>(st + L.sa);
        const double* sb = reinterpret_cast<const double*>(st + L.sb);
        const int e_lo = rps[0];
        const unsigned char* sls = st + L.sl + (e_lo & 15);
        const double* avs = reinterpret_cast<const double*>(st + L.av) + (e_lo & 1);
        const int base = t * TM, rows = min(TM, n - base);
        const int wlo = max(row0 + base - 1, 0);  // global
        for (int r0 = warp * gpw; r0 < rows; r0 += kBulkConsumers * gpw) {
          const int rr = r0 + g;
          const bool v = rr < rows && cv;
          // merged stages: the sub-tile's window starts dj rows into the stage's
          const int dj = max(row0 + base + (rr / kPlanT) * kPlanT - 1, 0) - wlo;
          if (PHX_CHECKS && v)
            for (int e = rps[rr] - e_lo; e < rps[rr + 1] - e_lo; ++e)
              PHX_CHECK(e >= 0 && e < a.plan_emax * M && int(sls[e]) + dj < (M > 1 ? TM + 2 : a.plan_rows));
          const double* self = dr + (row0 + base + rr - wlo) * width;  // the row itself (window)
          if constexpr (CPL == 4) {
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            if (v) gath(dr + dj * width, sls, avs, rps[rr] - e_lo, rps[rr + 1] - e_lo, c, ch, cvh, acc);
            const unsigned long long m = epi(v, v && cvh, rr < rows, base + rr, c, ch, acc, self,
                                             sa + rr * width, sb + rr * width, GL);
            mx = umax64(mx, m);
          } else {
            double a0 = 0.0, a1 = 0.0;
            if (v) gath(dr + dj * width, sls, avs, rps[rr] - e_lo, rps[rr + 1] - e_lo, c, a0, a1);
            const unsigned long long m =
                epi(v, rr < rows, base + rr, c, a0, a1, self, sa + rr * width + c, sb + rr * width + c, lg, G);
            mx = umax64(mx, m);
          }
        }
      }
      __syncwarp();
      if (PHX_PROBE) {
        pr_cwait += cc1 - cc0;
        pr_cwork += clock64() - cc1;
        ++pr_stages;
      }
      if (lane == 0) mbar_arrive(&bar_empty[s]);
      if (t < 0) break;
    }
    return mx;
  };

  // gathers: columns (c, c+1) of every entry's staged row, in CSR order
  auto gath_pair = [&](int width) {
    return [width](const double* dr, const unsigned char* sls, const double* avs, int e0, int e1,
                   int c, double& a0, double& a1) {
      for (int e = e0; e < e1; ++e) {
        const double2 x = *reinterpret_cast<const double2*>(dr + int(sls[e]) * width + c);
        const double av = avs[e];
        a0 = a0 + av * x.x;
        a1 = a1 + av * x.y;
      }
    };
  };
  // CPL 4: columns (c, c+1) and (ch, ch+1) of every entry's staged row, in
  // CSR order (the second pair only where it exists: vh)
  auto gath_quad = [&](int width) {
    return [width](const double* dr, const unsigned char* sls, const double* avs, int e0, int e1,
                   int c, int ch, bool vh, double(&acc)[4]) {
      // the second pair's byte offset; a lane without one re-reads its first
      // pair (unused), so no load is predicated
      const int hb = vh ? (ch - c) * 8 : 0;
      const unsigned rb = unsigned(width) * 8u;
      const unsigned char* lo = reinterpret_cast<const unsigned char*>(dr + c);
#pragma unroll 4
      for (int e = e0; e < e1; ++e) {
        const unsigned char* xr = lo + unsigned(sls[e]) * rb;
        const double2 x = *reinterpret_cast<const double2*>(xr);
        const double2 y = *reinterpret_cast<const double2*>(xr + hb);
        const double av = avs[e];
        acc[0] = acc[0] + av * x.x;
        acc[1] = acc[1] + av * x.y;
        acc[2] = acc[2] + av * y.x;
        acc[3] = acc[3] + av * y.y;
      }
    };
  };

  // ================= init: row-major V into D0, ||Vw_1||, max|V| (phi_block.cpp:76-92)
  // D0 holds V row-major with an even stride p1e (pad column 0): its rows
  // are whole 16-byte granules, so the first S term stages them with bulk
  // copies.  Lane lg of a row's group loads V columns lg and lg + G; the
  // lanes' Vw_1 columns (V[src] * g) come by shuffle.  NB row groups per warp
  // have their loads in flight together.
  const int p1e = (p1 + 1) & ~1;
  unsigned long long m0 = 0, mv = 0;
  {
    constexpr int NB = 4;
    const int G = GS, gpw = 32 / G, g = lane / G, lg = lane % G, c = 2 * lg;
    int src[2];
    double gv[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int cc = c + e;
      const int j = cc < w ? cc / r : 0, i = cc < w ? cc - j * r : 0;
      src[e] = j == 0 ? 0 : p + 1 - j;
      gv[e] = cc < w ? __ldg(a.g + i) : 0.0;
    }
    const int nwarps = ncta * kBW, ngroups = (n + gpw - 1) / gpw;
    for (int q0 = cta * kBW + warp; q0 < ngroups; q0 += NB * nwarps) {
      double v0[NB], v1[NB];
      int rowb[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int q = q0 + b * nwarps, row = q * gpw + g;
        rowb[b] = (q < ngroups && row < n) ? row : -1;
        v0[b] = (rowb[b] >= 0 && lg < p1) ? __ldg(a.V + size_t(lg) * size_t(n) + row) : 0.0;
        v1[b] = (rowb[b] >= 0 && lg + G < p1) ? __ldg(a.V + size_t(lg + G) * size_t(n) + row) : 0.0;
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int row = rowb[b];
        if (row >= 0) {
          if (lg < p1) mv = umax64(mv, abs_bits(v0[b]));
          if (lg + G < p1) mv = umax64(mv, abs_bits(v1[b]));
          if (lg < p1e) a.D0[size_t(row) * size_t(p1e) + lg] = v0[b];
          if (lg + G < p1e) a.D0[size_t(row) * size_t(p1e) + lg + G] = v1[b];
        }
        double ax[1][2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double x0 = __shfl_sync(kFull, v0[b], g * G + (src[e] % G));
          const double x1 = __shfl_sync(kFull, v1[b], g * G + (src[e] % G));
          const double vv = src[e] < G ? x0 : x1;
          ax[0][e] = (row >= 0 && c + e < w) ? fabs(vv * gv[e]) : 0.0;
        }
        const double rsum = group_rowsum<1, 2>(ax, G, 1);
        if (row >= 0) m0 = umax64(m0, abs_bits(rsum));
      }
    }
  }
  double mD, mSn;
  sync_step(m0, mv, mD, mSn);
  if (!(mSn <= DBL_MAX_D)) {  // a non-finite entry of V (check_request, phi_block.cpp:25-26)
    finish(kStInputNonFinite, 0, 1, 0);
    return;
  }
  double c1 = INF, c2 = mD, nS = mD;
  trace(0.0, c2, nS);

  // exact ||S||_inf (canonical row sums) for an inconclusive stopping test
  // (see k_phimv_block: the bounds nSl <= ||S|| <= nSu decide every other term)
  // Paired S terms (see the S-series loop): after a skip term S holds
  // S_{k-1}; S_k = fl(S + fl(D_k / sigma_k)) is then formed on the fly from
  // D_k (Ds != nullptr) -- the same two roundings the fold applies.
  auto s_norm_exact = [&](const double* Ds, double sig) -> double {
    unsigned long long m = 0;
    const int c = 2 * (lane % GS);
    plain_rows(GS, [&](int row, bool rv, int) {
      double as[1][2] = {{0.0, 0.0}};
      if (rv && c < w) {
        double2 x = *reinterpret_cast<const double2*>(a.S + (unsigned(row) * ldb + c));
        if (Ds) {
          const double2 d = *reinterpret_cast<const double2*>(Ds + (unsigned(row) * ldb + c));
          x.x = x.x + d.x / sig;
          x.y = x.y + d.y / sig;
        }
        as[0][0] = fabs(x.x);
        as[0][1] = fabs(x.y);
      }
      const double rs = group_rowsum<1, 2>(as, GS, 1);
      if (rv) m = umax64(m, abs_bits(rs));
    });
    double mx, dmy;
    sync_step(m, m, mx, dmy);
    return mx;
  };
  const bool exact_every_term = a.trace != nullptr;
  double nSl = nS, nSu = nS;
  bool exact = true;

  // ================= S series (phi_block.cpp:93-106)
  int k = 1;
  double sigma = 1.0;
  double* Dc = a.D0;
  double* Dn = a.D1;
  int err = kStOk, err_idx = 0;
  if (c1 + c2 > a.tol * nS) {
    // the first term (k = 2), peeled: D_1 = Vw_1 = S_1 = fl(V[src] * g) from
    // the row-major V in D0; the gathered V rows are loaded a batch at a time
    ++k;
    c1 = c2;
    sigma *= k;
    int src[2], srcl[2], jj[2];
    double gg[2], kd[2], ka[2], tos[2];
    {
      const int c = 2 * (lane % GS);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = c + e;
        const bool ok = cc < w;
        const int j = ok ? cc / r : 0, i = ok ? cc - j * r : 0;
        jj[e] = j;
        src[e] = j == 0 ? 0 : p + 1 - j;
        srcl[e] = j <= 1 ? 0 : p + 2 - j;
        gg[e] = ok ? __ldg(a.g + i) : 0.0;
        kd[e] = ok ? __ldg(a.colKd + cc) : 0.0;
        ka[e] = ok ? __ldg(a.colKa + cc) : 0.0;
        tos[e] = ok ? __ldg(a.colTos + cc) : 0.0;
      }
    }
    double* const Dn1 = Dn;
    const double sig1 = sigma, rsig1 = 1.0 / sigma;
    const unsigned long long mdb = bulk_phase(
        IC<2>{}, GS, w, p1e, a.D0, 0, nullptr, nullptr,
        // acc = sum_e av_e * Vw_1[col_e] = av_e * fl(V[col_e][src] * g)
        [&](const double* dr, const unsigned char* sls, const double* avs, int e0, int e1, int,
            double& a0, double& a1) {
          for (int e = e0; e < e1; ++e) {
            const double* vr = dr + int(sls[e]) * p1e;
            const double av = avs[e];
            a0 = a0 + av * (vr[src[0]] * gg[0]);
            a1 = a1 + av * (vr[src[1]] * gg[1]);
          }
        },
        [&](bool v, bool rvalid, int row, int c, double a0, double a1, const double* self,
            const double*, const double*, int, int G) -> unsigned long long {
          double ad[1][2] = {{0.0, 0.0}};
          if (v) {
            const double acc[2] = {a0, a1};
            double vn[2], dn[2], sn[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const double vw = self[src[e]] * gg[e];  // Vw_1 = D_1 = S_1
              const double vwl = jj[e] >= 2 ? self[srcl[e]] * gg[e] : 0.0;
              double g2 = 0.0;  // Vw = Vw * Kiter (:98)
              if (jj[e] >= 2) g2 = g2 + vwl * ka[e];
              g2 = g2 + vw * kd[e];
              vn[e] = g2;
              double y = acc[e];  // D = (A - xi I) D (:99), * t_i/s, + Vw
              if (has_xi) y = y - a.xi * vw;
              y = y * tos[e];
              dn[e] = y + g2;
              sn[e] = vw + div_rcp(dn[e], sig1, rsig1);  // S += D/sigma (:105)
              ad[0][e] = fabs(dn[e]);
            }
            const unsigned o = unsigned(row) * ldb + c;
            __stcs(reinterpret_cast<double2*>(a.Vw + o), make_double2(vn[0], vn[1]));
            __stcs(reinterpret_cast<double2*>(Dn1 + o), make_double2(dn[0], dn[1]));
            __stcs(reinterpret_cast<double2*>(a.S + o), make_double2(sn[0], sn[1]));
          }
          const double rd = group_rowsum<1, 2>(ad, G, 1);
          return rvalid ? abs_bits(rd) : 0ull;
        });
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
        nS = s_norm_exact(nullptr, 0.0);
        nSl = nSu = nS;
        exact = true;
      }
      trace(1.0, c2, nS);
      double* tmp = Dc;
      Dc = Dn;
      Dn = tmp;
    }
  } else {
    // no S term at all (tol * ||S|| infinite): the phases below read S = Vw_1
    const int c = 2 * (lane % GS);
    plain_rows(GS, [&](int row, bool rv, int) {
      if (!rv || c >= w) return;
      double x[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = c + e;
        const int j = cc / r, i = cc - j * r;
        const int sc = j == 0 ? 0 : p + 1 - j;
        x[e] = a.D0[size_t(row) * size_t(p1e) + sc] * __ldg(a.g + i);
      }
      *reinterpret_cast<double2*>(a.S + (unsigned(row) * ldb + c)) = make_double2(x[0], x[1]);
    });
    double dmy1, dmy2;
    sync_step(0ull, 0ull, dmy1, dmy2);
  }
#if !PHX_CPL4
  // the lane's S-term column coefficients (fixed for the whole launch)
  int jjS[2];
  double kdS[2], kaS[2], tosS[2];
  // kaL: the lane's Vw column coefficients of block j - 1 (column c - r): the
  // fold term recomputes Vw_{k-1}[c - r] from Vw_{k-2}.
  double kaL[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int cc = 2 * (lane % GS) + e;
    const bool ok = cc < w;
    jjS[e] = ok ? cc / r : 0;
    kdS[e] = ok ? __ldg(a.colKd + cc) : 0.0;
    kaS[e] = ok ? __ldg(a.colKa + cc) : 0.0;
    tosS[e] = ok ? __ldg(a.colTos + cc) : 0.0;
    kaL[e] = (ok && cc >= r) ? __ldg(a.colKa + (cc - r)) : 0.0;
  }
#else
  // CPL 4: the block index j of the lane's columns (c, c+1, ch, ch+1), a
  // byte each; the column coefficients are read per pair (__ldg, L1-resident)
  unsigned jjq = 0;
  {
    const int GLS = GS > 1 ? GS >> 1 : 1;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int cc = 2 * (lane % GLS) + (e < 2 ? 0 : 2 * GLS) + (e & 1);
      jjq |= unsigned(cc < w ? cc / r : 0) << (8 * e);
    }
  }
#endif
  // The specialised S-term consumer (skip and fold terms of the common
  // shape: 16 < w <= 32, i.e. 8 lanes per row and 4 rows per warp pass; r
  // even; xi != 0).  The same per-element operations in the same order as the
  // general CPL-4 consumer below -- bitwise unchanged -- with what that
  // consumer decides at run time fixed at compile time: the lane's second
  // column pair sits 128 bytes after its first (immediate offsets, loaded
  // unconditionally and masked at the stores), the column coefficients come
  // from the shared table ctab (lane-constant addresses) instead of global
  // loads, a row's entries are gathered in blocks of 4 / 2 / 1 with a
  // block's loads issued before its arithmetic, and the row-sum tree has its
  // three shuffle levels unrolled.
  const bool fastS = PHX_FAST_S && PHX_CPL4 && GS == 16 && (r % 2) == 0 && w <= 32 && has_xi &&
                     (a.bulk_flags & 4) == 0;
  if (fastS) {
    if (threadIdx.x < 32) {
      const int cc = threadIdx.x;
      const bool ok = cc < w;
      // (padding columns get Kd = t/s = 1: a lane without its second pair
      // computes on the next row's values, never stores them, and must not
      // produce the exact zeros that send a warp's IEEE division through its
      // slow path on every row)
      ctab[0][cc] = ok ? __ldg(a.colKd + cc) : 1.0;
      ctab[1][cc] = ok ? __ldg(a.colKa + cc) : 0.0;
      ctab[2][cc] = ok ? __ldg(a.colTos + cc) : 1.0;
      ctab[3][cc] = (ok && cc >= r) ? __ldg(a.colKa + (cc - r)) : 0.0;
    }
    __syncthreads();
  }
  auto s_fast = [&](auto foldc, double* Dnn, double sig, double sigp) {
    constexpr bool FOLD = decltype(foldc)::value != 0;
    const int lg = lane & 7, g = lane >> 3;
    const int c = 2 * lg;              // the lane's pairs: columns (c, c+1) and (16+c, 17+c)
    const bool v1 = 16 + c < w;        // the second pair exists (the first always does: w > 16)
    const int jA = c / r, jB = v1 ? (16 + c) / r : 0;  // the pairs' block index (r even)
    const unsigned rb = unsigned(w) * 8u, cb = unsigned(c) * 8u, r8 = unsigned(r) * 8u;
    const double* const ct = &ctab[0][c];
    const double xi = a.xi;
    return [=, &a](const unsigned char* st, const BulkStage& L, int t, int TM, int M) -> unsigned long long {
      const int base = t * TM, rows = min(TM, n - base);
      const int* const rps = reinterpret_cast<const int*>(st + L.rp);
      const int e_lo = rps[0];
      // indexed by the absolute entry number
      const unsigned char* const sls = st + L.sl + ((e_lo & 15) - e_lo);
      const double* const avs = reinterpret_cast<const double*>(st + L.av) + ((e_lo & 1) - e_lo);
      const int wlo = max(row0 + base - 1, 0);
      const unsigned char* const xb = st + L.dr + cb;
      const unsigned char* const selfb = xb + unsigned(row0 + base - wlo) * rb;
      const unsigned char* const pab = st + L.sa + cb;
      const unsigned char* const pbb = st + L.sb + cb;
      unsigned long long mx = 0;
#ifdef PHX_DIAG
      if (a.bulk_flags & 16) return 0x3ff0000000000000ull;  // developer: consumers idle
#endif
      for (int r0 = warp * 4; r0 < rows; r0 += kBulkConsumers * 4) {
        const int rr = r0 + g;
        const bool rv = rr < rows;
        int e = 0, e1 = 0;
        if (rv) {
          e = rps[rr];
          e1 = rps[rr + 1];
        }
#ifdef PHX_DIAG
        if (a.bulk_flags & 8) e1 = e;  // developer: no gather
#endif
        const unsigned char* xr = xb;
        if (M > 1) xr += unsigned(max(row0 + base + (rr / kPlanT) * kPlanT - 1, 0) - wlo) * rb;
        if (PHX_CHECKS && rv) {  // every entry and slot inside its stage region
          const int dj = int((xr - xb) / rb);
          PHX_CHECK(e >= e_lo && e1 >= e && e1 - e_lo <= a.plan_emax * M);
          for (int q = e; q < e1; ++q) PHX_CHECK(int(sls[q]) + dj < (M > 1 ? TM + 2 : a.plan_rows));
          PHX_CHECK(row0 + base + rr - wlo < (M > 1 ? TM + 2 : kPlanT + 2));
        }
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        // NB entries: all loads first, then the products and sums in CSR order
#define PHX_GBLK(NB)                                                                   \
  {                                                                                    \
    unsigned sl_[NB];                                                                  \
    double av_[NB];                                                                    \
    double2 x_[NB], y_[NB];                                                            \
    _Pragma("unroll") for (int q = 0; q < NB; ++q) {                                   \
      sl_[q] = sls[e + q];                                                             \
      av_[q] = avs[e + q];                                                             \
    }                                                                                  \
    _Pragma("unroll") for (int q = 0; q < NB; ++q) {                                   \
      const unsigned char* xe = xr + sl_[q] * rb;                                      \
      x_[q] = *reinterpret_cast<const double2*>(xe);                                   \
      y_[q] = *reinterpret_cast<const double2*>(xe + 128);                             \
    }                                                                                  \
    _Pragma("unroll") for (int q = 0; q < NB; ++q) {                                   \
      acc[0] = acc[0] + av_[q] * x_[q].x;                                              \
      acc[1] = acc[1] + av_[q] * x_[q].y;                                              \
      acc[2] = acc[2] + av_[q] * y_[q].x;                                              \
      acc[3] = acc[3] + av_[q] * y_[q].y;                                              \
    }                                                                                  \
  }
        for (; e + 4 <= e1; e += 4) PHX_GBLK(4)
        if (e + 2 <= e1) {
          PHX_GBLK(2)
          e += 2;
        }
        if (e < e1) PHX_GBLK(1)
#undef PHX_GBLK
        const unsigned char* const par = pab + unsigned(rr) * rb;
        const unsigned char* const selfr = selfb + unsigned(rr) * rb;
        const unsigned o = unsigned(base + rr) * ldb + unsigned(c);
        double ad[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int off = 128 * h;
          const bool hv = rv && (h == 0 || v1);
          const int jj = h ? jB : jA;
          const double2 kd = *reinterpret_cast<const double2*>(ct + 16 * h);
          const double2 ka = *reinterpret_cast<const double2*>(ct + 32 + 16 * h);
          const double2 tos = *reinterpret_cast<const double2*>(ct + 64 + 16 * h);
          const double2 x0 = *reinterpret_cast<const double2*>(par + off);
          const double2 x1r = *reinterpret_cast<const double2*>(par + off - r8);
          const double2 ds = *reinterpret_cast<const double2*>(selfr + off);
          // Vw_k[c] = fl(fl(+0 + Vw_{k-1}[c - r] Ka) + Vw_{k-1}[c] Kd) (:98)
          auto vwb = [](double kd_, double ka_, double vw, double vl) {
            double g2 = 0.0;
            g2 = g2 + vl * ka_;
            g2 = g2 + vw * kd_;
            return g2;
          };
          // D = (A - xi I) D (:99), * t_i/s (:101), + Vw (:102)
          auto dnx = [xi](double tos_, double ac, double dsv, double g2) {
            double y = ac - xi * dsv;
            y = y * tos_;
            return y + g2;
          };
          const bool j2 = jj >= 2;
          const double2 x1 = make_double2(j2 ? x1r.x : 0.0, j2 ? x1r.y : 0.0);
          if constexpr (!FOLD) {
            // skip term: Vw_{k-1} in, D_k out
            const double d0 = dnx(tos.x, acc[2 * h], ds.x, vwb(kd.x, ka.x, x0.x, x1.x));
            const double d1 = dnx(tos.y, acc[2 * h + 1], ds.y, vwb(kd.y, ka.y, x0.y, x1.y));
            ad[2 * h] = hv ? fabs(d0) : 0.0;
            ad[2 * h + 1] = hv ? fabs(d1) : 0.0;
            if (hv) __stcs(reinterpret_cast<double2*>(Dnn + (o + 16 * h)), make_double2(d0, d1));
          } else {
            // fold term: Vw_{k-2} and S_{k-2} in; Vw_k, D_k, S_k out (ds = D_{k-1})
            const double2 kl = *reinterpret_cast<const double2*>(ct + 96 + 16 * h);
            const double2 x2r = *reinterpret_cast<const double2*>(par + off - 2 * r8);
            const double2 so = *reinterpret_cast<const double2*>(pbb + unsigned(rr) * rb + off);
            const bool j3 = jj >= 3;
            const double2 x2 = make_double2(j3 ? x2r.x : 0.0, j3 ? x2r.y : 0.0);
            double vn[2], dn[2], sn[2];
            const double kdv[2] = {kd.x, kd.y}, kav[2] = {ka.x, ka.y}, tov[2] = {tos.x, tos.y},
                         klv[2] = {kl.x, kl.y}, x0v[2] = {x0.x, x0.y}, x1v[2] = {x1.x, x1.y},
                         x1rv[2] = {x1r.x, x1r.y}, x2v[2] = {x2.x, x2.y}, sov[2] = {so.x, so.y},
                         dpv[2] = {ds.x, ds.y};
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              // Vw_{k-1}[c] and Vw_{k-1}[c - r], as the skip term formed them
              const double wc = vwb(kdv[q], kav[q], x0v[q], x1v[q]);
              double wl = 0.0;
              wl = wl + x2v[q] * klv[q];
              wl = wl + x1rv[q] * kdv[q];
              wl = j2 ? wl : 0.0;
              vn[q] = vwb(kdv[q], kav[q], wc, wl);                 // Vw_k
              dn[q] = dnx(tov[q], acc[2 * h + q], dpv[q], vn[q]);  // D_k
              const double s1 = sov[q] + dpv[q] / sigp;            // S_{k-1} (:105)
              sn[q] = s1 + dn[q] / sig;                            // S_k
              ad[2 * h + q] = hv ? fabs(dn[q]) : 0.0;
            }
            if (hv) {
              __stcs(reinterpret_cast<double2*>(a.Vw + (o + 16 * h)), make_double2(vn[0], vn[1]));
              __stcs(reinterpret_cast<double2*>(Dnn + (o + 16 * h)), make_double2(dn[0], dn[1]));
              __stcs(reinterpret_cast<double2*>(a.S + (o + 16 * h)), make_double2(sn[0], sn[1]));
            }
          }
        }
        // the canonical row sum: pairwise tree over the 32 (padded) columns
        double lo = ad[0] + ad[1], hi = ad[2] + ad[3];
#pragma unroll
        for (int m = 1; m < 8; m <<= 1) {
          lo = lo + __shfl_xor_sync(kFull, lo, m);
          hi = hi + __shfl_xor_sync(kFull, hi, m);
        }
        const double rd = lo + hi;
        if (rv) mx = umax64(mx, abs_bits(rd));
      }
      return mx;
    };
  };
  // Paired S terms (bitwise the reference's per-term data flow, 25% fewer
  // bytes): S_k = S_{k-1} + D_k / sigma_k and Vw_k = Vw_{k-1} Kiter are
  // STORED only every other term.  A skip term (odd k >= 3) reads Vw_{k-1},
  // forms Vw_k in registers and writes D_k alone; the next, fold term (k + 1)
  // reads Vw_{k-1} again, recomputes Vw_k with the same roundings, forms
  // Vw_{k+1}, and folds both S updates in the reference order,
  // S_{k+1} = fl(fl(S_{k-1} + fl(D_k / sigma_k)) + fl(D_{k+1} / sigma_{k+1}))
  // with D_k the gather source's own row (already staged in the window).
  // Per pair: D read, D' write and Vw read twice, Vw write and S read/write
  // once -- 72 w n bytes instead of 96 w n.  After a final skip term one fold
  // pass completes S for the promotion.
  bool s_stale = false;  // S (and Vw) hold term k - 1's values
  double sig_prev = sigma;
  const bool vwl_vec = (r % 2) == 0;
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
      nS = s_norm_exact(s_stale ? Dc : nullptr, sigma);
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
    sig_prev = sigma;
    sigma *= k;
    double* const Dnn = Dn;
    const double sig = sigma, sigp = sig_prev, rsig = 1.0 / sigma, rsigp = 1.0 / sig_prev;
    // Vw_k[c] = fl(fl(+0 + Vw_{k-1}[c - r] Ka) + Vw_{k-1}[c] Kd) (:98)
    auto vw_nx = [&](int jj, double kd, double ka, double vw, double vl) {
      double g2 = 0.0;
      if (jj >= 2) g2 = g2 + vl * ka;
      g2 = g2 + vw * kd;
      return g2;
    };
    // D = (A - xi I) D (:99), * t_i/s (:101), + Vw (:102)
    auto d_nx = [&](double tos, double acc, double ds, double g2) {
      double y = acc;
      if (has_xi) y = y - a.xi * ds;
      y = y * tos;
      return y + g2;
    };
#if !PHX_CPL4
    auto vw_next = [&](int e, double vw, double vl) { return vw_nx(jjS[e], kdS[e], kaS[e], vw, vl); };
    auto d_next = [&](int e, double acc, double ds, double g2) { return d_nx(tosS[e], acc, ds, g2); };
#endif
    unsigned long long mdb;
#if PHX_CPL4
    // CPL 4 (see bulk_phase): the lane's column pairs h = 0, 1 at cp = c, ch;
    // the pairs' coefficients are read per row (__ldg: L1-resident); pa / pb:
    // the row's staged stream rows.  With r even (double2 shifts) the
    // optional shifted loads are unconditional -- every such address stays
    // inside the stage -- and zeroed by select, which is bitwise the branchy
    // form: fl(+0 + 0 * Ka) = +0 for the finite Ka.
    auto jsel = [](bool on, double2 x) { return on ? x : make_double2(0.0, 0.0); };
    auto vw_b = [&](double kd, double ka, double vw, double vl) {  // vl = 0 where j < 2
      double g2 = 0.0;
      g2 = g2 + vl * ka;
      g2 = g2 + vw * kd;
      return g2;
    };
    if (fastS) {
      if (!s_stale)
        mdb = bulk_phase(IC<8>{}, GS, w, w, Dc, Dc == a.D0 ? 0 : 1, a.Vw, nullptr,
                         s_fast(IC<0>{}, Dnn, sig, sigp), 0);
      else
        mdb = bulk_phase(IC<8>{}, GS, w, w, Dc, Dc == a.D0 ? 0 : 1, a.Vw, a.S,
                         s_fast(IC<1>{}, Dnn, sig, sigp), 0);
    } else if (!s_stale) {
      // skip term: Vw_{k-1} in, D_k out
      mdb = bulk_phase(
          IC<4>{}, GS, w, w, Dc, Dc == a.D0 ? 0 : 1, a.Vw, nullptr, gath_quad(w),
          [&](bool v0, bool v1, bool rvalid, int row, int c, int ch, const double(&acc)[4],
              const double* self, const double* pa, const double*, int GL) -> unsigned long long {
            double ad[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int cp = h ? ch : c;
              if (h ? v1 : v0) {
                const unsigned jx = (jjq >> (16 * h)) & 0xffu, jy = (jjq >> (16 * h + 8)) & 0xffu;
                const double2 kd = __ldg(reinterpret_cast<const double2*>(a.colKd + cp));
                const double2 ka = __ldg(reinterpret_cast<const double2*>(a.colKa + cp));
                const double2 tos = __ldg(reinterpret_cast<const double2*>(a.colTos + cp));
                const double2 vw = *reinterpret_cast<const double2*>(pa + cp);
                double2 vl = make_double2(0.0, 0.0);
                if (vwl_vec) {
                  vl = jsel(jx >= 2, *reinterpret_cast<const double2*>(pa + cp - r));
                } else {
                  if (jx >= 2) vl.x = pa[cp - r];
                  if (jy >= 2) vl.y = pa[cp + 1 - r];
                }
                double2 ds = make_double2(0.0, 0.0);
                if (has_xi) ds = *reinterpret_cast<const double2*>(self + cp);
                const double d0 = d_nx(tos.x, acc[2 * h], ds.x, vw_b(kd.x, ka.x, vw.x, vl.x));
                const double d1 = d_nx(tos.y, acc[2 * h + 1], ds.y, vw_b(kd.y, ka.y, vw.y, vl.y));
                ad[2 * h] = fabs(d0);
                ad[2 * h + 1] = fabs(d1);
                __stcs(reinterpret_cast<double2*>(Dnn + (unsigned(row) * ldb + cp)), make_double2(d0, d1));
              }
            }
            const double rd = quad_rowsum(ad, GL);
            return rvalid ? abs_bits(rd) : 0ull;
          });
    } else {
      // fold term: Vw_{k-2} and S_{k-2} in; Vw_k, D_k, S_k out
      mdb = bulk_phase(
          IC<4>{}, GS, w, w, Dc, Dc == a.D0 ? 0 : 1, a.Vw, a.S, gath_quad(w),
          [&](bool v0, bool v1, bool rvalid, int row, int c, int ch, const double(&acc)[4],
              const double* self, const double* pa, const double* pb, int GL) -> unsigned long long {
            double ad[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int cp = h ? ch : c;
              if (h ? v1 : v0) {
                const unsigned jx = (jjq >> (16 * h)) & 0xffu, jy = (jjq >> (16 * h + 8)) & 0xffu;
                const double2 kd2 = __ldg(reinterpret_cast<const double2*>(a.colKd + cp));
                const double2 ka2 = __ldg(reinterpret_cast<const double2*>(a.colKa + cp));
                const double2 tos2 = __ldg(reinterpret_cast<const double2*>(a.colTos + cp));
                // Vw_{k-2}[c], [c - r], [c - 2r] (zeros where the block has none)
                const double2 x0 = *reinterpret_cast<const double2*>(pa + cp);
                double2 x1 = make_double2(0.0, 0.0), x2 = make_double2(0.0, 0.0);
                if (vwl_vec) {
                  x1 = jsel(jx >= 1, *reinterpret_cast<const double2*>(pa + cp - r));
                  x2 = jsel(jx >= 2, *reinterpret_cast<const double2*>(pa + cp - 2 * r));
                } else {
                  if (jx >= 1) x1.x = pa[cp - r];
                  if (jy >= 1) x1.y = pa[cp + 1 - r];
                  if (jx >= 2) x2.x = pa[cp - 2 * r];
                  if (jy >= 2) x2.y = pa[cp + 1 - 2 * r];
                }
                const double2 so = *reinterpret_cast<const double2*>(pb + cp);
                const double2 dp = *reinterpret_cast<const double2*>(self + cp);  // D_{k-1}
                const double v0v[2] = {x0.x, x0.y}, v1v[2] = {x1.x, x1.y}, v2v[2] = {x2.x, x2.y},
                             sov[2] = {so.x, so.y}, dpv[2] = {dp.x, dp.y};
                const unsigned jjv[2] = {jx, jy};
                const double kdv[2] = {kd2.x, kd2.y}, kav[2] = {ka2.x, ka2.y}, tov[2] = {tos2.x, tos2.y};
                double vn[2], dn[2], sn[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                  // Vw_{k-1}[c] (x1 = 0 where j < 2) and Vw_{k-1}[c - r] (j >= 2:
                  // fl(fl(+0 + Vw[c - 2r] Ka(c - r)) + Vw[c - r] Kd), x2 = 0 where j < 3)
                  const double wc = vw_b(kdv[q], kav[q], v0v[q], jjv[q] >= 2 ? v1v[q] : 0.0);
                  double wl = 0.0;
                  if (jjv[q] >= 2) {
                    const double kl = __ldg(a.colKa + (cp + q - r));  // Ka of column c - r
                    wl = 0.0;
                    wl = wl + (jjv[q] >= 3 ? v2v[q] : 0.0) * kl;
                    wl = wl + v1v[q] * kdv[q];
                  }
                  vn[q] = vw_b(kdv[q], kav[q], wc, wl);                // Vw_k
                  dn[q] = d_nx(tov[q], acc[2 * h + q], dpv[q], vn[q]);  // D_k (ds = D_{k-1} row)
                  const double s1 = sov[q] + div_rcp(dpv[q], sigp, rsigp);  // S_{k-1} (:105)
                  sn[q] = s1 + div_rcp(dn[q], sig, rsig);                   // S_k
                  ad[2 * h + q] = fabs(dn[q]);
                }
                const unsigned o = unsigned(row) * ldb + cp;
                __stcs(reinterpret_cast<double2*>(a.Vw + o), make_double2(vn[0], vn[1]));
                __stcs(reinterpret_cast<double2*>(Dnn + o), make_double2(dn[0], dn[1]));
                __stcs(reinterpret_cast<double2*>(a.S + o), make_double2(sn[0], sn[1]));
              }
            }
            const double rd = quad_rowsum(ad, GL);
            return rvalid ? abs_bits(rd) : 0ull;
          });
    }
#else
    if (!s_stale) {
      // skip term: Vw_{k-1} in, D_k out
      mdb = bulk_phase(
          IC<2>{}, GS, w, w, Dc, Dc == a.D0 ? 0 : 1, a.Vw, nullptr, gath_pair(w),
          [&](bool v, bool rvalid, int row, int c, double a0, double a1, const double* self,
              const double* pa, const double*, int, int G) -> unsigned long long {
            double ad[1][2] = {{0.0, 0.0}};
            if (v) {
              const double2 vw = *reinterpret_cast<const double2*>(pa);
              double2 vl = make_double2(0.0, 0.0);
              if (vwl_vec) {
                if (jjS[0] >= 2) vl = *reinterpret_cast<const double2*>(pa - r);
              } else {
                if (jjS[0] >= 2) vl.x = pa[-r];
                if (jjS[1] >= 2) vl.y = pa[1 - r];
              }
              double2 ds = make_double2(0.0, 0.0);
              if (has_xi) ds = *reinterpret_cast<const double2*>(self + c);
              const double d0 = d_next(0, a0, ds.x, vw_next(0, vw.x, vl.x));
              const double d1 = d_next(1, a1, ds.y, vw_next(1, vw.y, vl.y));
              ad[0][0] = fabs(d0);
              ad[0][1] = fabs(d1);
              __stcs(reinterpret_cast<double2*>(Dnn + (unsigned(row) * ldb + c)), make_double2(d0, d1));
            }
            const double rd = group_rowsum<1, 2>(ad, G, 1);
            return rvalid ? abs_bits(rd) : 0ull;
          });
    } else {
      // fold term: Vw_{k-2} and S_{k-2} in; Vw_k, D_k, S_k out
      mdb = bulk_phase(
          IC<2>{}, GS, w, w, Dc, Dc == a.D0 ? 0 : 1, a.Vw, a.S, gath_pair(w),
          [&](bool v, bool rvalid, int row, int c, double a0, double a1, const double* self,
              const double* pa, const double* pb, int, int G) -> unsigned long long {
            double ad[1][2] = {{0.0, 0.0}};
            if (v) {
              // Vw_{k-2}[c], [c - r], [c - 2r] (zeros where the block has none)
              const double2 v0 = *reinterpret_cast<const double2*>(pa);
              double2 v1 = make_double2(0.0, 0.0), v2 = make_double2(0.0, 0.0);
              if (vwl_vec) {
                if (jjS[0] >= 1) v1 = *reinterpret_cast<const double2*>(pa - r);
                if (jjS[0] >= 2) v2 = *reinterpret_cast<const double2*>(pa - 2 * r);
              } else {
                if (jjS[0] >= 1) v1.x = pa[-r];
                if (jjS[1] >= 1) v1.y = pa[1 - r];
                if (jjS[0] >= 2) v2.x = pa[-2 * r];
                if (jjS[1] >= 2) v2.y = pa[1 - 2 * r];
              }
              const double2 so = *reinterpret_cast<const double2*>(pb);
              const double2 dp = *reinterpret_cast<const double2*>(self + c);  // D_{k-1}
              const double v0v[2] = {v0.x, v0.y}, v1v[2] = {v1.x, v1.y}, v2v[2] = {v2.x, v2.y},
                           sov[2] = {so.x, so.y}, dpv[2] = {dp.x, dp.y}, acc[2] = {a0, a1};
              double vn[2], dn[2], sn[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                // Vw_{k-1}[c] and Vw_{k-1}[c - r], as the skip term formed them
                const double wc = vw_next(e, v0v[e], v1v[e]);
                double wl = 0.0;
                if (jjS[e] >= 2) {  // column c - r, block j - 1 >= 1
                  wl = 0.0;
                  if (jjS[e] >= 3) wl = wl + v2v[e] * kaL[e];
                  wl = wl + v1v[e] * kdS[e];
                }
                vn[e] = vw_next(e, wc, wl);            // Vw_k
                dn[e] = d_next(e, acc[e], dpv[e], vn[e]);  // D_k (ds = D_{k-1} row)
                const double s1 = sov[e] + div_rcp(dpv[e], sigp, rsigp);  // S_{k-1} (:105)
                sn[e] = s1 + div_rcp(dn[e], sig, rsig);                   // S_k
                ad[0][e] = fabs(dn[e]);
              }
              const unsigned o = unsigned(row) * ldb + c;
              __stcs(reinterpret_cast<double2*>(a.Vw + o), make_double2(vn[0], vn[1]));
              __stcs(reinterpret_cast<double2*>(Dnn + o), make_double2(dn[0], dn[1]));
              __stcs(reinterpret_cast<double2*>(a.S + o), make_double2(sn[0], sn[1]));
            }
            const double rd = group_rowsum<1, 2>(ad, G, 1);
            return rvalid ? abs_bits(rd) : 0ull;
          });
    }
#endif
    s_stale = !s_stale;
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
    double* tmp = Dc;
    Dc = Dn;
    Dn = tmp;
    if (exact_every_term) {
      nS = s_norm_exact(s_stale ? Dc : nullptr, sigma);
      nSl = nSu = nS;
      exact = true;
    }
    trace(1.0, c2, nS);
  }
  if (err == kStOk && s_stale) {
    // the series ended on a skip term: S_L = fl(S_{L-1} + fl(D_L / sigma_L)).
    // Row groups strided over all warps, NB groups per warp in flight (the
    // pass is a pure stream; one group at a time left it latency-bound).
    constexpr int NB = 4;
    const int gpw = 32 / GS, g = lane / GS, c = 2 * (lane % GS);
    const int nwarps = ncta * kBW, units = (n + gpw - 1) / gpw;
    for (int u0 = cta * kBW + warp; u0 < units; u0 += NB * nwarps) {
      double2 x[NB], d[NB];
      unsigned o[NB];
      bool v[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int u = u0 + b * nwarps, row = u * gpw + g;
        v[b] = u < units && row < n && c < w;
        o[b] = unsigned(row) * ldb + unsigned(c);
        if (v[b]) {
          x[b] = __ldcs(reinterpret_cast<const double2*>(a.S + o[b]));
          d[b] = __ldcs(reinterpret_cast<const double2*>(Dc + o[b]));
        }
      }
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (v[b]) {
          x[b].x = x[b].x + d[b].x / sigma;
          x[b].y = x[b].y + d[b].y / sigma;
          *reinterpret_cast<double2*>(a.S + o[b]) = x[b];
        }
    }
    double dmy1, dmy2;
    sync_step(0ull, 0ull, dmy1, dmy2);
    s_stale = false;
  }
  const int L_S = k;
  if (err != kStOk) {
    finish(err, err_idx, L_S, 0);
    return;
  }

  // ================= promotion (phi_block.cpp:109-120)
  // F_L = fl(fl(A S_L * t_i) + v0) (unshifted A), F_R = S block p
  double* Fc = a.F0;
  double* Fn = a.F1;
  const bool sweeps = SW && a.s_eff > 1;
  const unsigned long long mf = bulk_phase(
      IC<2>{}, GF, fc, w, a.S, 2, nullptr, nullptr,
      // gathers S block-0 columns (left F columns live at the same column
      // index in S); a pair straddling the left/right split gathers one extra
      // column, unused
      [&](const double* dr, const unsigned char* sls, const double* avs, int e0, int e1, int c,
          double& a0, double& a1) {
        if (c >= r) return;
        for (int e = e0; e < e1; ++e) {
          const double2 x = *reinterpret_cast<const double2*>(dr + int(sls[e]) * w + c);
          const double av = avs[e];
          a0 = a0 + av * x.x;
          a1 = a1 + av * x.y;
        }
      },
      [&](bool v, bool rvalid, int row, int c, double a0, double a1, const double* self,
          const double*, const double*, int, int G) -> unsigned long long {
        double f[2] = {0.0, 0.0}, af[1][2] = {{0.0, 0.0}};
        if (v) {
          const double acc[2] = {a0, a1};
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cc = c + e;
            const int i = cc < r ? cc : cc - r;
            const double* srow = self + size_t(p) * size_t(r);  // S block p of the row
            if (cc < r) {
              const double sc = acc[e] * __ldg(a.t + i);
              f[e] = sc + __ldg(a.V + row);
            } else {
              f[e] = srow[i];
            }
            if (!sweeps && cc < r) {
              // assembly W = F_L + fl(F_R * alpha) (:148-154)
              double wv = f[e];
              double fr = 0.0;
              if (p > 0) {
                fr = srow[i];
                wv = wv + fr * __ldg(a.alpha + i);
              }
              a.W[size_t(i) * size_t(n) + row] = wv;
              if (a.FLo) a.FLo[size_t(i) * size_t(n) + row] = f[e];
              if (a.FRo) a.FRo[size_t(i) * size_t(n) + row] = fr;
            }
            af[0][e] = fabs(f[e]);
          }
          if (sweeps) {
            const unsigned o = unsigned(row) * ldf + c;
            *reinterpret_cast<double2*>(Fc + o) = make_double2(f[0], f[1]);
            *reinterpret_cast<double2*>(a.E + o) = make_double2(f[0], f[1]);
          }
        }
        if (!sweeps) return 0ull;
        const double rf = group_rowsum<1, 2>(af, G, 1);
        return rvalid ? abs_bits(rf) : 0ull;
      });
  if (!sweeps) {
    finish(kStOk, 0, L_S, 1);
    return;
  }
  if constexpr (!SW) {
    return;  // (unreachable: s_eff = 1 launches finish above)
  } else {
  double fnorm, dummy;
  sync_step(mf, mf, fnorm, dummy);

  auto e_norm_exact = [&]() -> double {
    unsigned long long m = 0;
    const int c = 2 * (lane % GF);
    plain_rows(GF, [&](int row, bool rv, int) {
      double ae[1][2] = {{0.0, 0.0}};
      if (rv && c < fc) {
        const double2 x = *reinterpret_cast<const double2*>(a.E + (unsigned(row) * ldf + c));
        ae[0][0] = fabs(x.x);
        ae[0][1] = fabs(x.y);
      }
      const double rs = group_rowsum<1, 2>(ae, GF, 1);
      if (rv) m = umax64(m, abs_bits(rs));
    });
    double mx, dmy;
    sync_step(m, m, mx, dmy);
    return mx;
  };

  // the lane's recovery column scale t_i / s
  double tosF[2];
  {
    const int c = 2 * (lane % GF);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int cc = c + e;
      const int i = cc < r ? cc : cc - r;
      tosF[e] = cc < fc ? __ldg(a.colTos + i) : 0.0;
    }
  }

  // The specialised recovery-term consumer (8 < fc <= 16: 4 lanes per row
  // with 4 columns each, 8 rows per warp pass; block variant; xi != 0): the
  // general consumer's per-element operations in the same order -- bitwise
  // unchanged -- at half the lanes per row, so the per-entry slot / value /
  // address work, the row bookkeeping and the row-sum shuffles are shared by
  // twice the columns.  Odd rows take their two column pairs in the opposite
  // order, so a quarter-warp's 16-byte loads (two rows of 128 bytes) cover
  // all 32 banks.
  // (window-only plans: their merged stages hold >= 64 rows, so all consumer
  // warps have a pass; a 32-row stage would leave half of them idle)
  const bool fastF = PHX_FAST_S && GF == 8 && !a.single_variant && has_xi && a.plan_merge != 0 &&
                     (a.bulk_flags & 4) == 0;
  auto r_fast = [&](double* Fnn, double dkk) {
    const int lg = lane & 3, g = lane >> 2;
    const int cA = 2 * lg + ((g & 1) ? 8 : 0), cB = 2 * lg + ((g & 1) ? 0 : 8);  // the lane's pairs
    const bool vA = cA < fc, vB = cB < fc;
    const unsigned rb = unsigned(fc) * 8u, offA = unsigned(cA) * 8u;
    const int dAB = (cB - cA) * 8;
    double tA[2], tB[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int ca = cA + e, cb_ = cB + e;
      tA[e] = ca < fc ? __ldg(a.colTos + (ca < r ? ca : ca - r)) : 0.0;
      tB[e] = cb_ < fc ? __ldg(a.colTos + (cb_ < r ? cb_ : cb_ - r)) : 0.0;
    }
    const double tA0 = tA[0], tA1 = tA[1], tB0 = tB[0], tB1 = tB[1];
    const double xi = a.xi;
    return [=, &a](const unsigned char* st, const BulkStage& L, int t, int TM, int M) -> unsigned long long {
      const int base = t * TM, rows = min(TM, n - base);
      const int* const rps = reinterpret_cast<const int*>(st + L.rp);
      const int e_lo = rps[0];
      const unsigned char* const sls = st + L.sl + ((e_lo & 15) - e_lo);
      const double* const avs = reinterpret_cast<const double*>(st + L.av) + ((e_lo & 1) - e_lo);
      const int wlo = max(row0 + base - 1, 0);
      const unsigned char* const xb = st + L.dr + offA;
      const unsigned char* const selfb = xb + unsigned(row0 + base - wlo) * rb;
      const unsigned char* const pab = st + L.sa + offA;
      unsigned long long mx = 0;
      for (int r0 = warp * 8; r0 < rows; r0 += kBulkConsumers * 8) {
        const int rr = r0 + g;
        const bool rv = rr < rows;
        int e = 0, e1 = 0;
        if (rv) {
          e = rps[rr];
          e1 = rps[rr + 1];
        }
        const unsigned char* xr = xb;
        if (M > 1) xr += unsigned(max(row0 + base + (rr / kPlanT) * kPlanT - 1, 0) - wlo) * rb;
        if (PHX_CHECKS && rv) {  // every entry and slot inside its stage region
          const int dj = int((xr - xb) / rb);
          PHX_CHECK(e >= e_lo && e1 >= e && e1 - e_lo <= a.plan_emax * M);
          for (int q = e; q < e1; ++q) PHX_CHECK(int(sls[q]) + dj < (M > 1 ? TM + 2 : a.plan_rows));
          PHX_CHECK(row0 + base + rr - wlo < (M > 1 ? TM + 2 : kPlanT + 2));
        }
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#define PHX_GBLK(NB)                                                                   \
  {                                                                                    \
    unsigned sl_[NB];                                                                  \
    double av_[NB];                                                                    \
    double2 x_[NB], y_[NB];                                                            \
    _Pragma("unroll") for (int q = 0; q < NB; ++q) {                                   \
      sl_[q] = sls[e + q];                                                             \
      av_[q] = avs[e + q];                                                             \
    }                                                                                  \
    _Pragma("unroll") for (int q = 0; q < NB; ++q) {                                   \
      const unsigned char* xe = xr + sl_[q] * rb;                                      \
      x_[q] = *reinterpret_cast<const double2*>(xe);                                   \
      y_[q] = *reinterpret_cast<const double2*>(xe + dAB);                             \
    }                                                                                  \
    _Pragma("unroll") for (int q = 0; q < NB; ++q) {                                   \
      acc[0] = acc[0] + av_[q] * x_[q].x;                                              \
      acc[1] = acc[1] + av_[q] * x_[q].y;                                              \
      acc[2] = acc[2] + av_[q] * y_[q].x;                                              \
      acc[3] = acc[3] + av_[q] * y_[q].y;                                              \
    }                                                                                  \
  }
        for (; e + 4 <= e1; e += 4) PHX_GBLK(4)
        if (e + 2 <= e1) {
          PHX_GBLK(2)
          e += 2;
        }
        if (e < e1) PHX_GBLK(1)
#undef PHX_GBLK
        const unsigned char* const par = pab + unsigned(rr) * rb;
        const unsigned char* const selfr = selfb + unsigned(rr) * rb;
        const double2 eoA = *reinterpret_cast<const double2*>(par);
        const double2 eoB = *reinterpret_cast<const double2*>(par + dAB);
        const double2 fsA = *reinterpret_cast<const double2*>(selfr);
        const double2 fsB = *reinterpret_cast<const double2*>(selfr + dAB);
        // y = ((A - xi I) F) / kk (:132) * t_i/s (:134-135); E += F (:138)
        auto term = [xi, dkk](double ac, double fs, double tos_) {
          double yv = ac - xi * fs;
          yv = yv / dkk;
          return yv * tos_;
        };
        const double yA0 = term(acc[0], fsA.x, tA0), yA1 = term(acc[1], fsA.y, tA1);
        const double yB0 = term(acc[2], fsB.x, tB0), yB1 = term(acc[3], fsB.y, tB1);
        const bool hA = rv && vA, hB = rv && vB;
        const unsigned o = unsigned(base + rr) * ldf;
        if (hA) {
          __stcs(reinterpret_cast<double2*>(Fnn + (o + unsigned(cA))), make_double2(yA0, yA1));
          __stcs(reinterpret_cast<double2*>(a.E + (o + unsigned(cA))), make_double2(eoA.x + yA0, eoA.y + yA1));
        }
        if (hB) {
          __stcs(reinterpret_cast<double2*>(Fnn + (o + unsigned(cB))), make_double2(yB0, yB1));
          __stcs(reinterpret_cast<double2*>(a.E + (o + unsigned(cB))), make_double2(eoB.x + yB0, eoB.y + yB1));
        }
        // the canonical row sum: pairwise tree over the 16 (padded) columns
        double sA = (hA ? fabs(yA0) : 0.0) + (hA ? fabs(yA1) : 0.0);
        double sB = (hB ? fabs(yB0) : 0.0) + (hB ? fabs(yB1) : 0.0);
#pragma unroll
        for (int m = 1; m < 4; m <<= 1) {
          sA = sA + __shfl_xor_sync(kFull, sA, m);
          sB = sB + __shfl_xor_sync(kFull, sB, m);
        }
        const double rd = sA + sB;
        if (rv) mx = umax64(mx, abs_bits(rd));
      }
      return mx;
    };
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
      const double dkk = double(kk), rkk = 1.0 / dkk;
      double* const Fnn = Fn;
      const unsigned long long mfb = fastF ? bulk_phase(IC<8>{}, GF, fc, fc, Fc, Fc == a.F0 ? 3 : 4, a.E,
                                                        nullptr, r_fast(Fnn, dkk), 0)
                                           : bulk_phase(
          IC<2>{}, GF, fc, fc, Fc, Fc == a.F0 ? 3 : 4, a.E, nullptr, gath_pair(fc),
          [&](bool v, bool rvalid, int row, int c, double a0, double a1, const double* self,
              const double* pa, const double*, int, int G) -> unsigned long long {
            double ay[1][2] = {{0.0, 0.0}};
            if (v) {
              const double2 eo = *reinterpret_cast<const double2*>(pa);
              double2 fs = make_double2(0.0, 0.0);
              if (has_xi) fs = *reinterpret_cast<const double2*>(self + c);
              const double eov[2] = {eo.x, eo.y}, fsv[2] = {fs.x, fs.y}, acc[2] = {a0, a1};
              double y[2], en[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                double yv = acc[e];
                if (has_xi) yv = yv - a.xi * fsv[e];
                if (a.single_variant) {
                  yv = fac * yv;  // phi_single.cpp:106
                } else {
                  yv = div_rcp(yv, dkk, rkk);  // phi_block.cpp:132
                  yv = yv * tosF[e];  // :134-135
                }
                y[e] = yv;
                en[e] = eov[e] + yv;  // E += F (:138)
                ay[0][e] = fabs(yv);
              }
              const unsigned o = unsigned(row) * ldf + c;
              __stcs(reinterpret_cast<double2*>(Fnn + o), make_double2(y[0], y[1]));
              __stcs(reinterpret_cast<double2*>(a.E + o), make_double2(en[0], en[1]));
            }
            const double ry = group_rowsum<1, 2>(ay, G, 1);
            return rvalid ? abs_bits(ry) : 0ull;
          });
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
    }
    if (err != kStOk) break;
    if (lead) a.lensF[sweep - 1] = kk;

    // ---- sweep end (:141-145): E *= mu; Sadv = Sadv*Jexp; F refresh
    // phase A (S layout): Sadv blocks 1..p in place, ascending source column
    {
      const int c = 2 * (lane % GS);
      plain_rows(GS, [&](int row, bool rv, int) {
        double nv[2];
        bool wq[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cc = c + e;
          const int j = cc < w ? cc / r : 0, i = cc - j * r;
          wq[e] = rv && cc < w && j >= 1;
          nv[e] = 0.0;
          if (wq[e]) {
            const double* srow = a.S + size_t(row) * ldb;
            const double* cj = a.jc + size_t(i) * size_t(p + 1);
            double accv = 0.0;
            for (int l = 1; l <= j; ++l) accv = accv + srow[l * r + i] * __ldg(cj + (j - l));
            nv[e] = accv;
          }
        }
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (wq[e]) a.S[size_t(row) * ldb + c + e] = nv[e];
      });
    }
    __syncthreads();
    // phase B (F layout): F_L = E_L*mu, F_R = E_R*mu + Sadv_p; E = F
    const bool last = sweep == a.s_eff - 1;
    unsigned long long mfe = 0;
    {
      const int c = 2 * (lane % GF);
      plain_rows(GF, [&](int row, bool rv, int) {
        double f[2], af[1][2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          f[e] = 0.0;
          const int cc = c + e;
          if (rv && c < fc) {
            const int i = cc < r ? cc : cc - r;
            const size_t srow = size_t(row) * ldb + size_t(p) * size_t(r);
            const double en = a.E[size_t(row) * ldf + cc] * __ldg(a.mu + i);
            double fv = en;
            if (cc >= r) fv = en + a.S[srow + i];
            f[e] = fv;
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
          af[0][e] = (rv && c < fc) ? fabs(f[e]) : 0.0;
        }
        if (!last) {
          __syncwarp();
          if (rv && c < fc) {
            const unsigned o = unsigned(row) * ldf + c;
            *reinterpret_cast<double2*>(Fc + o) = make_double2(f[0], f[1]);
            *reinterpret_cast<double2*>(a.E + o) = make_double2(f[0], f[1]);
          }
          const double rf = group_rowsum<1, 2>(af, GF, 1);
          if (rv) mfe = umax64(mfe, abs_bits(rf));
        }
      });
    }
    if (!last) {
      double dmy;
      sync_step(mfe, mfe, fnorm, dmy);
    }
  }
  finish(err, err_idx, L_S, 0);
  }
}

}  // namespace

cudaError_t bulk_occupancy(size_t smem, int* per_sm, bool part) {
  // both instantiations (with / without recovery code) of the variant must
  // fit: the launch picks one of them by s_eff
  const void* fs[2] = {part ? reinterpret_cast<const void*>(k_phimv_bulk<true, true>)
                            : reinterpret_cast<const void*>(k_phimv_bulk<false, true>),
                       part ? reinterpret_cast<const void*>(k_phimv_bulk<true, false>)
                            : reinterpret_cast<const void*>(k_phimv_bulk<false, false>)};
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  int per = 1 << 30;
  for (const void* f : fs) {
    // the opt-in limit covers the kernel's static shared memory too: a ring
    // that leaves no room for it does not fit (0 CTAs), which is not an error
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return e;
    if (smem + fa.sharedSizeBytes > size_t(optin)) {
      *per_sm = 0;
      return cudaSuccess;
    }
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    int p1 = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p1, f, kBulkThreads, smem);
    if (e != cudaSuccess) return e;
    per = p1 < per ? p1 : per;
  }
  *per_sm = per;
  return cudaSuccess;
}

cudaError_t launch_phimv_bulk(const BlockArgs& a, int grid, cudaStream_t st) {
  BlockArgs copy = a;
  void* args[] = {&copy};
  const size_t smem = size_t(a.bulk_ns) * size_t(a.bulk_stage_bytes);
  const void* f = a.s_eff > 1 ? reinterpret_cast<const void*>(k_phimv_bulk<false, true>)
                              : reinterpret_cast<const void*>(k_phimv_bulk<false, false>);
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaLaunchCooperativeKernel(f, grid, kBulkThreads, args, smem, st);
}

cudaError_t launch_phimv_bulk_parts(const BulkPartArgs& pa, int grid, cudaStream_t st) {
  void* args[] = {const_cast<BulkPartArgs*>(&pa)};
  const BlockArgs& a = pa.pa[pa.pa[0].plo];
  const size_t smem = size_t(a.bulk_ns) * size_t(a.bulk_stage_bytes);
  const void* f = a.s_eff > 1 ? reinterpret_cast<const void*>(k_phimv_bulk<true, true>)
                              : reinterpret_cast<const void*>(k_phimv_bulk<true, false>);
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaLaunchCooperativeKernel(f, grid, kBulkThreads, args, smem, st);
}

}  // namespace phx
