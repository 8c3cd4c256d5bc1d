// Shared declarations between the host orchestration (phx_host.cpp) and the
// sm_100a kernels (phx_kernels.cu).  No torch, no Eigen: plain device
// pointers.
#pragma once
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

namespace phx {

constexpr int kChunk = 4096;       // stableNorm block (Eigen blocking)
constexpr int kNormThreads = 256;  // canonical lane count of a chunk

constexpr int kMaxParts = 16;
constexpr int kCtaStampBase = 4096;  // diagnostics layout of BlockArgs::tstamp  // row parts of a partitioned operator

// Cross-part step mailbox: part p's leader writes (a, b) then gen into slot
// p of every part's mailbox array (peer memory in a multi-GPU run).
struct MailBox {
  unsigned gen;
  unsigned pad;
  unsigned long long a, b;
};

// One row part of a partitioned operator: its CSR rows with
// encoded columns (owner part << 27 | row within the owner), its block
// buffers (part-local rows), its step slots, arrival counters and mailboxes.
struct PartTab {
  const int32_t* rp;
  const int32_t* ci;
  const double* av;
  const double* V;
  double* Vw;
  double* D0;
  double* D1;
  double* S;
  double* F0;
  double* F1;
  double* E;
  double* W;
  unsigned long long* slots;  // [3][4]
  unsigned* arrive;           // [3]
  MailBox* mbox;              // [2 step parities][nparts]
  int32_t row0, nrows;
  // the part's tile plan (bulk kernel; phx_plan.cpp with row0 / ntot)
  const int32_t* plan_desc;
  const uint8_t* plan_slot;
  const int32_t* plan_sgl;
};

// Per-call parameters of the persistent phimv_block kernel.
struct BlockArgs {
  // operator (CSR, int32 indices)
  int32_t n;
  const int32_t* rp;
  const int32_t* ci;
  const double* av;
  // shape
  int32_t p, r, w, fcols;
  int32_t GS, QS;  // S-layout: lanes per row (pow2 <= 32), columns per lane
  int32_t GF, QF;  // F-layout
  int32_t QT;      // template width: pow2 >= max(QS, QF), in {1,2,4,8}
  int32_t vec;     // adjacent columns per lane (2 when both widths are even)
  int32_t R;       // rows per lane group per warp tile (1 or 2; 2 only when QT == 1)
  int32_t tile;    // rows per tile (row -> CTA mapping, independent of layout)
  int32_t dyn;          // 1: dynamic-tail kernel (always for partitioned runs)
  int32_t bsmall;       // 1: the short-gather-batch variant (rows fit it)
  int32_t lat;          // 1: the latency-mode variant (fewer tiles than SMs)
  float gather_keep;    // L2 evict_last fraction for gather loads (0 or 1)
  int32_t cl_rows;      // cluster mode: rows per part allocated in shared memory
  int32_t cl_nnz;       // cluster mode: CSR entries per part allocated in shared memory
  double static_frac;  // DYN kernels: share of a phase's CTA tiles assigned statically
  // scalars
  double xi, tol;
  int32_t s_eff;
  int32_t single_variant;  // recovery op order of phi_single.cpp:106
  double t_single;         // t (single variant only)
  // per-column / per-abscissa coefficients (device)
  const double* colKd;   // [w]   Kiter diagonal
  const double* colKa;   // [w]   Kiter superdiagonal (0 for blocks 0,1)
  const double* colTos;  // [w]   t_i / s
  const double* t;       // [r]
  const double* alpha;   // [r]
  const double* mu;      // [r]
  const double* g;       // [r]   mu_i / s
  const double* jc;      // [r*(p+1)] Jexp chain c_d per abscissa
  // buffers (row-interleaved blocks, row stride ldb / ldf doubles)
  const double* V;  // n x (p+1) column-major, ld n
  double* Vw;
  double* D0;
  double* D1;
  double* S;
  int32_t ldb;
  double* F0;
  double* F1;
  double* E;
  int32_t ldf;
  double* W;    // n x r column-major, ld n
  double* FLo;  // optional n x r exp_v0 (single variant), ld n
  double* FRo;  // optional n x r tail, ld n
  // control
  unsigned long long* slots;  // [3][4] ring: row-sum maxima A, B, tile counter, pad
  int32_t* status;            // [8]: code, index, L_S, sweeps done, steps
  int32_t* lensF;             // [s_eff-1]
  double* trace;              // optional (kind, a, b) triples
  int32_t trace_cap;
  // partitioned operator (nparts > 1): this launch handles parts
  // plo .. plo+pcount-1; ptab (device, nparts entries) describes all parts
  int32_t nparts, plo, pcount;
  const PartTab* ptab;
  // tile plan of the bulk-copy evaluator (k_phimv_bulk, phx_bulk.cu): per
  // kPlanT-row tile a descriptor of its contiguous gather copies, a one-byte
  // slot per CSR entry (its row in the stage's gathered-row array) and the
  // single rows; the stage layout (rows, entries) and ring depth
  const int32_t* plan_desc;
  const uint8_t* plan_slot;
  const int32_t* plan_sgl;
  int32_t plan_rows;     // gathered rows per stage: window (T+2) + singles + groups
  int32_t plan_sgl_cap;  // single rows per stage (groups start after them)
  int32_t plan_emax;     // CSR entries per tile (max over the tiles, even)
  int32_t plan_merge;    // 1: window-only plan (no groups, no singles): tiles may be merged
  int32_t bulk_ns;       // stages in the ring
  int32_t bulk_stage_bytes;
  int32_t bulk_flags;    // bit 0: gather copies evict_last (else evict_normal); bit 1: try_wait
                         // with a suspend-time hint (waiting warps sleep instead of spinning);
                         // bit 2: general consumers only (no specialised S-term / recovery-term
                         // consumer: the A/B and test switch, PHX_BULK_FLAGS)
  // diagnostics (PHX_STEP_TIMES): %globaltimer after each grid step barrier
  // at [step]; CTA arrivals (time mod 2^48 | smid << 48) at
  // [kCtaStampBase + step * ncta + cta]
  unsigned long long* tstamp;
  int32_t tstamp_cap;
};

// status codes written by the kernel
enum : int32_t {
  kStOk = 0,
  kStSeriesCap = 1,
  kStSeriesDiverged = 2,
  kStRecoveryCap = 3,
  kStRecoveryDiverged = 4,
  kStInputNonFinite = 5,  // V has a non-finite entry (detected in the init pass)
};

// ---------------------------------------------------------------------------
// Tile plan of the bulk-copy evaluator (built once
// per operator by build_tile_plan, phx_plan.cpp).  A tile is kPlanT
// consecutive rows.  Its gather sources are staged in shared memory by
// cp.async.bulk copies of CONTIGUOUS row ranges: the window [base-1,
// base+T+1) (the tile's own rows and every column inside it), up to
// kPlanGroups "offset groups" (the entries whose column - row offset is shared
// by many rows of the tile: rows [base+off, base+off+T) in one copy) and a few
// single rows.  Descriptor (kPlanDesc int32 per tile):
//   [0] groups  [1] singles  [2] first single in plan_sgl  [3] e_lo  [4] e_hi
//   [5] the tile   [8+g] group g's first source row   [12+g] rows | (stage row << 16)
// stored in the plan's processing order (phx_plan.cpp tile_order).
#ifndef PHX_PLAN_T
#define PHX_PLAN_T 32
#endif
constexpr int kPlanT = PHX_PLAN_T;  // rows per tile
constexpr int kPlanGroups = 4;
constexpr int kPlanDesc = 16;
constexpr int kPlanMaxSingles = 32;
constexpr int kPlanMaxEntries = 1024;  // per tile (stage capacity)
#ifndef PHX_BULK_CONS
#define PHX_BULK_CONS 8
#endif
constexpr int kBulkConsumers = PHX_BULK_CONS;  // consumer warps per CTA (+ 1 producer warp)
constexpr int kBulkThreads = (kBulkConsumers + 1) * 32;
constexpr int kBulkMaxStages = 8;

struct TilePlan {
  std::vector<int32_t> desc;
  std::vector<uint8_t> slot;  // nnz + 16 (padded for 16-byte copy granules)
  std::vector<int32_t> sgl;   // + 1
  int32_t rows = 0, sgl_cap = 0, emax = 0;
  bool ok = false;
  bool blocked = false;  // y-blocked lattice order (else natural)
};
// false (plan.ok == false) when some tile needs more than the stage holds
// A part's plan (row-partitioned operators): its n rows start at global row
// row0 of an operator of ntot rows; row_ptr points at the part's first entry
// of the whole row_ptr, col_idx is the whole column array (global columns).
// Tiles and entry slots are part-local; window, group and single source rows
// are global (the kernel resolves them to the owning part's buffer).
bool build_tile_plan(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, TilePlan* plan,
                     int64_t row0 = 0, int64_t ntot = -1);

// byte layout of one stage of the bulk ring (host and device agree)
struct BulkStage {
  int32_t dr, sa, sb, av, sl, rp, hdr, bytes;
};
__host__ __device__ inline BulkStage bulk_stage(int32_t rows, int32_t emax, int32_t width,
                                                int32_t streams, int32_t T = kPlanT) {
  BulkStage L;
  int32_t o = 0;
  L.dr = o;  // gathered rows (width even: 16-byte multiples)
  o += rows * width * 8;
  L.sa = o;  // stream A tile (Vw | E)
  o += streams >= 1 ? T * width * 8 : 0;
  L.sb = o;  // stream B tile (S)
  o += streams >= 2 ? T * width * 8 : 0;
  L.av = o;  // CSR values (copied from a 16-byte granule)
  o += (emax + 2) * 8;
  L.sl = o;  // slots
  o += (emax + 32 + 15) / 16 * 16;
  L.rp = o;  // row_ptr slice
  o += (T + 4 + 3) / 4 * 16;
  L.hdr = o;  // tile id
  o += 16;
  L.bytes = (o + 127) / 128 * 128;
  return L;
}

cudaError_t launch_phimv_bulk(const BlockArgs& a, int grid, cudaStream_t st);
// every part's arguments (pa[q] for the launch's parts plo .. plo+pcount-1;
// pa[0] also carries the fields common to all parts: nparts, plo, pcount,
// ptab) -- the kernel parameter of the partitioned bulk kernel
struct BulkPartArgs {
  BlockArgs pa[kMaxParts];
};
cudaError_t launch_phimv_bulk_parts(const BulkPartArgs& pa, int grid, cudaStream_t st);
// co-resident CTAs per SM of k_phimv_bulk at the given dynamic shared memory
cudaError_t bulk_occupancy(size_t smem, int* per_sm, bool part = false);

// launch wrappers (phx_kernels.cu)
cudaError_t launch_phimv_block(const BlockArgs& a, int grid, int block, cudaStream_t st);
int eval_block_size();     // threads per CTA of k_phimv_block
// cluster mode (one thread-block cluster, one CTA per part, blocks in shared
// memory): dynamic shared memory per CTA, and the launch (nparts CTAs)
size_t eval_cluster_smem(int32_t cl_rows, int32_t cl_nnz, int32_t tile, int32_t ldb, int32_t ldf);

cudaError_t launch_phimv_block_cluster(const BlockArgs& a, int nparts, int block, cudaStream_t st);
size_t eval_pipe_bytes();  // its dynamic shared memory per CTA
cudaError_t coop_grid_size(int QT, int V, int R, bool part, bool dyn, bool small, int block,
                           int* max_blocks, bool lat = false);

// one instantiated kernel variant and its occupancy query
struct EvalKernel {
  const void* fn;
  cudaError_t (*occ)(int block, int* per_sm);
  size_t smem;  // dynamic shared memory per CTA (the variant's pipes)
};
// per-file variant tables (phx_eval_q*.cu): true when the file holds the
// variant (QT, V, R, partitioned, dynamic tail, short gather batch)
bool eval_kernels_q1v1(int QT, int V, int R, bool part, bool dyn, bool small, bool cluster, EvalKernel* out);
bool eval_kernels_q1v2a(int QT, int V, int R, bool part, bool dyn, bool small, bool cluster, EvalKernel* out);
bool eval_kernels_q1v2b(int QT, int V, int R, bool part, bool dyn, bool small, bool cluster, EvalKernel* out);
bool eval_kernels_q2(int QT, int V, int R, bool part, bool dyn, bool small, bool cluster, EvalKernel* out);
bool eval_kernels_q4(int QT, int V, int R, bool part, bool dyn, bool small, bool cluster, EvalKernel* out);
bool eval_kernels_q8(int QT, int V, int R, bool part, bool dyn, bool small, bool cluster, EvalKernel* out);
// the cluster variants (phx_eval_cl.cu) and their CTA size
bool eval_kernels_cl(int QT, int V, int R, bool small, EvalKernel* out);
// latency-mode variants (phx_eval_lat.cu): unpartitioned, static, 1 CTA/SM
bool eval_kernels_lat(int QT, int V, int R, bool small, EvalKernel* out);
int eval_cl_block();

// y = f(A x) with mode 0: A x, 1: A x - fl(xi x), 2: (A x) / div ; fused
// per-chunk max|y| into chunkmax (bit patterns) when chunkmax != nullptr
cudaError_t launch_spmv(int32_t n, const int32_t* rp, const int32_t* ci, const double* av,
                        const double* x, double* y, int mode, double xi, double div,
                        unsigned long long* chunkmax, cudaStream_t st);
// y = B c (B column-major n x ncol, ld n), canonical sequential order; fused
// chunk max
cudaError_t launch_gemv(int32_t n, int32_t ncol, const double* B, const double* c, double* y,
                        unsigned long long* chunkmax, cudaStream_t st);
cudaError_t launch_chunkmax(int32_t n, const double* x, unsigned long long* chunkmax,
                            cudaStream_t st);
// partial[b] = canonical sum over chunk b of fl(fl(x*inv[b])^2)
cudaError_t launch_chunk_ssq(int32_t n, const double* x, const double* inv, double* partial,
                             cudaStream_t st);
// x = x * s (mode 0) or x / s (mode 1)
cudaError_t launch_scale(int32_t n, double* x, double s, int mode, cudaStream_t st);
// stableNorm's per-chunk invScale from the chunk maxima, on the device (the
// host then needs one read-back: the maxima and the scaled partial sums)
cudaError_t launch_stable_inv(int32_t nch, const unsigned long long* chunkmax, double* inv,
                              cudaStream_t st);
// host col-major block (device copy, ld n) <-> nothing else needed; apply on
// k columns: Y = A X (mode 0) or (A - xi I) X (mode 1), column-major, ld n
cudaError_t launch_spmm_cols(int32_t n, int32_t k, const int32_t* rp, const int32_t* ci,
                             const double* av, const double* X, double* Y, int mode, double xi,
                             cudaStream_t st);

// expRK4s6 stage kernel arguments (phx_kernels.cu k_rk_stage).  mode 0: f_n
// (CSR A u + reaction) -> g_n, hf, V2; 1: stage 2 -> V34; 2: stage pair
// (ca, cb) -> next V; 3: u_next = u + W with a non-finite flag.
struct RkStageArgs {
  int mode;
  int64_t n;
  const int32_t* rp;
  const int32_t* ci;
  const double* av;
  const double* u;
  const double* W;  // n x (1 or 2), ld n
  double* gn;
  double* hf;
  double* V;  // n x (p+1), ld n
  double* out;
  int* flag;
  double gamma, h;
  double s0, s1, s2, s3;  // per-mode stage scalars (computed on the host)
  double ca, cb;
};
cudaError_t launch_rk_stage(const RkStageArgs& a, cudaStream_t st);

// block_series_direct term (phx_kernels.cu k_series_term); r <= kSeriesMaxR
constexpr int kSeriesMaxR = 64;
constexpr int kOccCacheDevices = 64;  // devices whose kernel occupancy is cached
cudaError_t launch_series_term(int32_t n, int32_t p1, int32_t r, const double* X, const double* M,
                               const double* tpow, double* G, unsigned long long* slots,
                               cudaStream_t st);

int64_t kernel_launch_count();
void count_launch();

}  // namespace phx
