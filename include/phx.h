/*
 * phx.h — C ABI of the B200-native phi-combination engine (libphx.so).
 *
 * This is the drop-in boundary for the hot path of arXiv 2509.26475
 * ("phiact"): parameter selection (Alg. 1) and the block evaluator (Alg. 3).
 * Each entry point names the reference C++ interface it replaces
 * (paths relative to the reference's proj/ directory).  Plain pointers and
 * sizes only; host buffers are column-major like the reference's Eigen
 * matrices (include/phiact/linop.hpp:12).  The C++ wrapper in
 * include/phx/phiact.hpp restores the reference names and exception types on
 * top of this header.
 *
 * Every compute entry point runs on an NVIDIA B200 (sm_100a).  There is no CPU
 * fallback: without a usable device every call returns PHX_ECUDA.
 *
 * Error model: functions return a phx_status; on failure phx_last_error()
 * returns the thread-local message.  The codes map onto the reference's
 * exception types (include/phiact headers):
 *   PHX_EINVAL  -> std::invalid_argument (bad input)
 *   PHX_ENUMERIC-> std::runtime_error    (divergence, non-convergence,
 *                                          mu overflow, rejected operator)
 *   PHX_ELOGIC  -> std::logic_error      (empty operator, shape)
 *   PHX_ECUDA   -> CUDA / device failure (no reference analogue)
 * Messages reproduce the reference's text where one exists.
 */
#ifndef PHX_H
#define PHX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PHX_OK = 0,
  PHX_EINVAL = 1,
  PHX_ENUMERIC = 2,
  PHX_ELOGIC = 3,
  PHX_ECUDA = 4,
  PHX_ENOMEM = 5
} phx_status;

/* Opaque handles. */
typedef struct phx_op_s* phx_op;       /* device-resident CSR operator      */
typedef struct phx_basis_s* phx_basis; /* device-resident power basis       */

/* ScalingShift (include/phiact/params.hpp:34-41).  Same fields, same meaning:
 * s = real scaling, xi = spectral shift, s0 = preliminary scale, f_min =
 * padded objective value, m = Taylor degree, r = accepted power count. */
typedef struct {
  double s;
  double xi;
  double s0;
  double f_min;
  int32_t m;
  int32_t r;
} phx_scaling_shift;

/* RunRecord (include/phiact/phi_single.hpp:16-21).  series_lens_F is a
 * caller-owned array of lens_capacity ints; n_sweeps = s_effective - 1 is the
 * number of entries the evaluation produced (entries beyond the capacity are
 * dropped, n_sweeps still reports the full count). */
typedef struct {
  int64_t s_effective;
  int32_t series_len_S;
  int32_t n_sweeps;
  int32_t* series_lens_F;
  int64_t lens_capacity;
  int64_t matvecs;
} phx_run_record;

/* ---------------------------------------------------------------------------
 * Operator (replaces LinearOperator, include/phiact/linop.hpp:19-37, for CSR
 * operators; the reference's ApplyFn is an opaque host callback that cannot
 * cross to the device, so the operator is a CSR descriptor instead).
 * row_ptr has n+1 entries, col_idx/vals have row_ptr[n] entries; column
 * indices are used in storage order (the product accumulates each row in that
 * order).  The handle owns device copies; the host arrays may be freed after
 * the call.  Immutable after creation; concurrent calls on one handle are
 * serialised internally.  device < 0 selects the current device.
 * Rejects n < 1, nnz >= 2^31, out-of-range indices, non-finite values
 * (dense_operator's checks, linop.cpp:26-38).
 * ------------------------------------------------------------------------- */
phx_status phx_op_create_csr(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                             const double* vals, int32_t device, phx_op* out);
phx_status phx_op_destroy(phx_op op);
/* Row-partitioned operator: rows split into nparts
 * contiguous parts, part q resident on devices[q] (NULL or -1: the current
 * device).  phx_phimv_block on it evaluates every part's rows on its device,
 * reading other parts' block rows over NVLink peer memory and combining the
 * per-term stopping norms across parts; the result is bitwise the
 * unpartitioned one.  Parts that share a device run as one launch (single-GPU
 * emulation).  Parameter selection and apply need an unpartitioned operator:
 * select on the whole operator and reuse the ScalingShift.  nparts <= 16,
 * each part < 2^27 rows. */
phx_status phx_op_create_csr_partitioned(int64_t n, const int64_t* row_ptr,
                                         const int32_t* col_idx, const double* vals,
                                         int32_t nparts, const int32_t* devices, phx_op* out);
int32_t phx_op_nparts(phx_op op);
int64_t phx_op_dim(phx_op op);
int64_t phx_op_nnz(phx_op op);
/* The CUDA stream (cudaStream_t) every call on this operator runs on; lets a
 * caller bracket calls with its own CUDA events. */
void* phx_op_stream(phx_op op);

/* Y = A*X (LinearOperator::apply, linop.cpp:10-24) and (A - xi I) X
 * (shifted_apply, linop.cpp:40-49) on host column-major blocks of k columns
 * with leading dimensions ldx/ldy >= n. */
phx_status phx_apply(phx_op op, const double* X, int64_t ldx, int64_t k, double* Y, int64_t ldy);
phx_status phx_shifted_apply(phx_op op, double xi, const double* X, int64_t ldx, int64_t k,
                             double* Y, int64_t ldy);

/* ---------------------------------------------------------------------------
 * Parameter selection (include/phiact/params.hpp:50-77).
 * ------------------------------------------------------------------------- */
/* select_parameters(op, m = 61, tol = -1 (2^-53), delta = 0.8)
 * (params.hpp:75-77, params.cpp:241-247). */
phx_status phx_select_parameters(phx_op op, int32_t m, double tol, double delta,
                                 phx_scaling_shift* out);

/* build_power_basis (params.hpp:50-51, params.cpp:81-154).  The basis lives
 * on the device, column-major n x (m+1). */
phx_status phx_basis_build(phx_op op, int32_t m, double delta, phx_basis* out);
phx_status phx_basis_destroy(phx_basis b);
/* r, m, s0; logs (r entries) and log_binom (m+1 entries) may be NULL;
 * columns (n*(m+1), column-major) may be NULL — copying it is a D2H. */
phx_status phx_basis_info(phx_basis b, int32_t* r, int32_t* m, double* s0, double* logs,
                          double* log_binom, double* columns);
/* objective(basis, xi) (params.hpp:56, params.cpp:156-170). */
phx_status phx_objective(phx_basis b, double xi, double* f);
/* minimize_shift(basis) (params.hpp:61, params.cpp:172-189).  path (may be
 * NULL) receives the Brent trial points as (u, f(u)) pairs. */
phx_status phx_minimize_shift(phx_basis b, double* xi, double* f_min, double* path,
                              int64_t path_capacity, int64_t* path_len);
/* parameters_for_shift(op, basis, xi, tol) (params.hpp:70-72,
 * params.cpp:213-239). */
phx_status phx_parameters_for_shift(phx_op op, phx_basis b, double xi, double tol,
                                    phx_scaling_shift* out);

/* ---------------------------------------------------------------------------
 * Block evaluator: phimv_block(op, BlockPhiRequest) (phi_block.hpp:30-31,
 * phi_block.cpp:48-157).  w_i = sum_j alpha_i^j phi_j(t_i A) v_j, i < r.
 *   t, alpha : r values each (BlockPhiRequest::t / ::alpha)
 *   V        : n x (p+1) column-major host block [v_0 .. v_p], leading dim ldv
 *   tol      : <= 0 means 2^-53
 *   params   : from phx_select_parameters (or any ScalingShift)
 *   W        : n x r column-major host output, leading dim ldw
 *   rec      : may be NULL
 * ------------------------------------------------------------------------- */
phx_status phx_phimv_block(phx_op op, int32_t r, const double* t, const double* alpha, int32_t p,
                           const double* V, int64_t ldv, double tol,
                           const phx_scaling_shift* params, double* W, int64_t ldw,
                           phx_run_record* rec);

/* Same evaluation on device-resident data: d_V is a device n x (p+1)
 * column-major block (leading dim n), d_W a device n x r column-major output
 * (leading dim n).  Runs on the operator's stream; returns after the result
 * and the record are complete.  Used to time the evaluation without host
 * copies. */
phx_status phx_phimv_block_device(phx_op op, int32_t r, const double* t, const double* alpha,
                                  int32_t p, const double* d_V, double tol,
                                  const phx_scaling_shift* params, double* d_W,
                                  phx_run_record* rec);

/* Row parts of a (partitioned) operator: part q holds rows
 * [row0, row0 + nrows) on `device`, evaluated on `stream`.  An unpartitioned
 * operator is one part.  Any output pointer may be null. */
phx_status phx_op_part_info(phx_op op, int32_t q, int64_t* row0, int64_t* nrows, int32_t* device,
                            void** stream);

/* The distributed device-resident form of phx_phimv_block_device: part q's
 * rows of V (nrows_q x (p+1)) and of W (nrows_q x r) live on part q's device,
 * column-major with leading dimension nrows_q (phx_op_part_info).  No copies:
 * every part reads its V slice and writes its W slice in place.  (On a
 * partitioned operator phx_phimv_block_device scatters V's rows from, and
 * gathers W's rows to, the operator's first device with peer copies.) */
phx_status phx_phimv_block_device_parts(phx_op op, int32_t r, const double* t, const double* alpha,
                                        int32_t p, const double* const* d_V_parts, double tol,
                                        const phx_scaling_shift* params, double* const* d_W_parts,
                                        phx_run_record* rec);

/* Single-combination evaluator phimv (phi_single.hpp:44, phi_single.cpp:38-127):
 * w = sum_j alpha^j phi_j(tA) v_j with the single variant's operation order.
 * exp_v0 / tail (n values each) may be NULL. */
phx_status phx_phimv(phx_op op, double t, double alpha, int32_t p, const double* V, int64_t ldv,
                     double tol, const phx_scaling_shift* params, double* w, double* exp_v0,
                     double* tail, phx_run_record* rec);

/* block_series_direct (phi_block.hpp:33-47, phi_block.cpp:158-212): the
 * direct power series G = sum_j A^j V D_j Gamma T^j (D_j = diag(a_0j..a_pj),
 * Gamma = [alpha_k^i]), the reference's cross-check of the scaled evaluator;
 * converges only while the t_k A are small.  coeffs: NULL for
 * phi_series_coeffs (a_ij = 1/(i+j)!), else a (p+1) x ncoef column-major
 * table of a_ij.  G: n x r host output (leading dim ldg).  r <= 64.  Errors
 * as phimv_block ("direct series did not converge within 500 terms",
 * "direct series produced a non-finite term at index j"). */
phx_status phx_block_series_direct(phx_op op, int32_t r, const double* t, const double* alpha,
                                  int32_t p, const double* V, int64_t ldv, double tol,
                                  const double* coeffs, int64_t ncoef, double* G, int64_t ldg);

/* ---------------------------------------------------------------------------
 * Sparse Matrix Market ingestion.  The reference's
 * read_matrix_market (matrix_market.hpp:10-16, matrix_market.cpp:37-100)
 * accepts the same files but reads them dense; these read CSR (structural
 * entries, columns ascending, duplicates summed in file order from +0, so
 * values equal the reference's dense entries bit for bit).  Failures return
 * PHX_ENUMERIC (std::runtime_error) with the reference's message text
 * "matrix market: <path>: <what>".  Host-only.
 */

/* Reads the file; always sets *n and *nnz.  Copies the CSR (row_ptr n+1,
 * col_idx / vals nnz) only when all three buffers are given and
 * cap_nnz >= nnz -- call once with NULL buffers to size them. */
phx_status phx_mm_read_csr(const char* path, int64_t* n, int64_t* nnz, int64_t* row_ptr,
                           int32_t* col_idx, double* vals, int64_t cap_nnz);
/* Writes CSR as `coordinate real general` with 17 significant digits
 * (round-trips bit for bit, like write_matrix_market's %.17g). */
phx_status phx_mm_write_csr(const char* path, int64_t n, const int64_t* row_ptr,
                            const int32_t* col_idx, const double* vals);
/* phx_op_create_csr from a Matrix Market file in one call. */
phx_status phx_op_create_mm(const char* path, int32_t device, phx_op* out);

/* ---------------------------------------------------------------------------
 * The evaluator's consumer: the fourth-order six-stage
 * exponential Runge-Kutta integrator on the 2D advection-diffusion-reaction
 * problem.
 */

/* adr_build (problems.hpp:46-70, problems.cpp:184-250) as CSR: n = nx*ny
 * rows, at most 5n entries (row_ptr n+1, col_idx / vals nnz = row_ptr[n]),
 * columns ascending; u0 (n) is the reference's initial condition bit for bit.
 * Any output pointer may be NULL.  PHX_EINVAL when nx < 8 or ny < 8
 * ("adr_build: grid must be at least 8x8").  Host-only (no device work). */
phx_status phx_adr_csr(int32_t nx, int32_t ny, double eps, double alpha_adv, int64_t* row_ptr,
                       int32_t* col_idx, double* vals, double* u0);

/* exprk4s6_step (integrator.hpp:36-38, integrator.cpp:29-105): one step of
 * size h from u (host, n) with reaction gamma*u*(u-1/2)*(1-u); four block
 * evaluations {U2}, {U3,U4}, {U5,U6}, {u_next} sharing params.  recs: NULL or
 * 4 records (one per evaluator call, StepRecord::calls).  Single-device
 * operators only. */
phx_status phx_exprk4s6_step(phx_op op, double gamma, const double* u, double h, double tol,
                             const phx_scaling_shift* params, double* u_next,
                             phx_run_record* recs);

/* integrate (integrator.hpp:47-49, integrator.cpp:107-134): fixed-step
 * integration from t = 0 to t_end with the state resident on the device.
 * u_out (n) receives the final state (the last finite one on failure);
 * t_out the time reached; n_steps_out the step count; recs NULL or
 * recs_cap records, 4 per step in step order.  Errors: PHX_EINVAL "integrate:
 * h must be positive" / "step count out of range" / "t_end is not a multiple
 * of h"; PHX_ENUMERIC "integrate: state left the finite range at t = ...". */
phx_status phx_integrate(phx_op op, double gamma, const double* u0, double h, double t_end,
                         double tol, const phx_scaling_shift* params, double* u_out,
                         double* t_out, int64_t* n_steps_out, phx_run_record* recs,
                         int64_t recs_cap);

/* ---------------------------------------------------------------------------
 * Introspection.
 * ------------------------------------------------------------------------- */
const char* phx_last_error(void);
/* Number of device kernels this process has launched through libphx. */
int64_t phx_kernel_launches(void);
/* How the last evaluation was launched (diagnostics): 0 one grid-wide
 * cooperative launch, 1 a partitioned operator's cooperative launches, 2 a
 * partitioned operator as ONE thread-block cluster with every part's blocks
 * in shared memory (opt-in: environment PHX_CLUSTER=1, all parts on one
 * device, 2..16 parts that fit). */
int32_t phx_last_eval_mode(void);

/* The kernel variant of the last single-device evaluation (diagnostics):
 * out[0..7] = column chunks per lane Q, columns per lane V, rows per lane
 * group R, tile scheduling (0 static, 1 dynamic tail, 2 the bulk-copy kernel
 * k_phimv_bulk), latency mode (0/1), short-row gather batch (0/1), grid size,
 * CTA size.  The bulk-copy kernel runs when the operator has a tile plan and
 * both block widths are even and <= 64; environment PHX_BULK=0 disables it,
 * PHX_BULK=1 forces it for every eligible operator (read on every call). */
phx_status phx_last_eval_variant(int32_t* out8);

/* The tile plan of the bulk-copy evaluator for a host CSR matrix, built on
 * the host exactly as phx_op_create_csr builds it (no device needed; for
 * diagnostics and tests).  The plan covers every kPlanT-row tile's
 * gathered rows with contiguous copies -- the window [base-1, base+T+1), up to
 * 4 offset groups (rows [base+off, base+off+T)) and single rows -- and gives
 * every CSR entry a one-byte slot (its row in the stage: window rows first,
 * then singles, then groups).  info[0..6] = ok (0/1), tiles, stage rows,
 * single rows per stage, max entries per tile (even), total single rows,
 * rows per tile.
 * When non-null, desc (tiles x 16 int32, in the kernel's processing order --
 * natural, or y-blocked for a 3D lattice operator: groups, singles, first
 * single, e_lo, e_hi, the tile, -, -, group source rows[4], group rows |
 * stage row << 16 [4]), slot (nnz + 16 bytes) and sgl (total single rows + 1)
 * are filled. */
phx_status phx_tile_plan(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int32_t* info6,
                         int32_t* desc, uint8_t* slot, int32_t* sgl);
/* The tile plan of one row part [row0, row0 + nrows) of an n-row operator
 * (row-partitioned operators, phx_op_create_csr_partitioned): tiles and entry
 * slots part-local, window / group / single source rows global.
 * phx_tile_plan(n, ...) is phx_tile_plan_part(n, ..., 0, n, ...). */
phx_status phx_tile_plan_part(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                              int64_t row0, int64_t nrows, int32_t* info7, int32_t* desc,
                              uint8_t* slot, int32_t* sgl);

/* Device-event time (ms) of the last phimv_block evaluation kernel, and the
 * number of grid-wide steps it executed (S terms + promotion + recovery
 * terms + sweep ends). */
phx_status phx_last_eval_stats(double* kernel_ms, int64_t* steps);
/* Set a device-side trace buffer capacity (0 disables).  When enabled,
 * phimv_block records (kind, a, b) triples per grid step: kind 0 = initial
 * S norms, 1 = S term (c2, ||S||), 2 = sweep start (||F||, ||E||), 3 = recovery
 * term (d2, ||E||) — the same records the oracle emits. */
phx_status phx_set_trace(int64_t capacity);
phx_status phx_get_trace(double* out, int64_t capacity, int64_t* len);

#ifdef __cplusplus
}
#endif

#endif /* PHX_H */
