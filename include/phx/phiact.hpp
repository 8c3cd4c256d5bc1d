// phx/phiact.hpp — the reference's C++ interface for the hot path, restored
// on top of the C ABI of libphx.so (include/phx.h).
//
// A caller of the reference (arXiv 2509.26475 "phiact", proj/include/phiact)
// switches by including this header instead of phiact/params.hpp +
// phiact/phi_block.hpp + phiact/phi_single.hpp and linking libphx.so:
//
//   reference                                  here
//   phiact::LinearOperator (linop.hpp:19-37)   phiact::LinearOperator built by
//                                              phiact::csr_operator(...)
//   phiact::ScalingShift (params.hpp:34-41)    same fields
//   phiact::select_parameters (params.hpp:75)  same signature
//   phiact::BlockPhiRequest / BlockPhiResult   same fields (Matrix/Vector are
//     (phi_block.hpp:14-25)                    the small column-major types below)
//   phiact::phimv_block (phi_block.hpp:30)     same signature
//   phiact::PhiRequest/PhiResult/phimv         same
//   phiact::RunRecord (phi_single.hpp:16-21)   same fields
//   exceptions std::invalid_argument / std::runtime_error / std::logic_error
//
// Differences: the operator is a CSR matrix held on the device (the
// reference's ApplyFn is an opaque host callback that cannot run on a GPU);
// phiact::dense_operator (linop.cpp:26-38) stores every entry as CSR.
// Matrix / Vector are Eigen::MatrixXd / Eigen::VectorXd -- the reference's own
// types (linop.hpp:12) -- whenever <Eigen/Dense> is available (or
// PHX_WITH_EIGEN is defined), so reference call sites compile unchanged;
// without Eigen they are minimal column-major containers with the same
// members (rows, cols, size, data, operator()).  Evaluations on one operator
// may run concurrently from several threads (each takes its own device
// workspace), as the reference's re-entrant operator allows (linop.hpp:16-18).
// Header-only.
#pragma once

#include <algorithm>
#include <cstdint>
#include <initializer_list>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../phx.h"

#if !defined(PHX_WITH_EIGEN) && !defined(PHX_NO_EIGEN) && defined(__has_include)
#if __has_include(<Eigen/Dense>)
#define PHX_WITH_EIGEN 1
#endif
#endif
#ifdef PHX_WITH_EIGEN
#include <Eigen/Dense>
#endif

namespace phiact {

using Index = std::int64_t;

#ifdef PHX_WITH_EIGEN
// the reference's types (linop.hpp:12): column-major, contiguous
using Matrix = Eigen::MatrixXd;
using Vector = Eigen::VectorXd;
#else
// Column-major dense block (the reference's Eigen::MatrixXd layout).
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols) : rows_(rows), cols_(cols), a_(size_t(rows * cols), 0.0) {}
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  double& operator()(Index i, Index j) { return a_[size_t(i + j * rows_)]; }
  double operator()(Index i, Index j) const { return a_[size_t(i + j * rows_)]; }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }
  double* col(Index j) { return a_.data() + j * rows_; }
  const double* col(Index j) const { return a_.data() + j * rows_; }

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<double> a_;
};

class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n, double v = 0.0) : a_(size_t(n), v) {}
  Vector(std::initializer_list<double> l) : a_(l) {}
  Index size() const { return Index(a_.size()); }
  double& operator()(Index i) { return a_[size_t(i)]; }
  double operator()(Index i) const { return a_[size_t(i)]; }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }

 private:
  std::vector<double> a_;
};
#endif

inline constexpr int kDefaultDegree = 61;               // params.hpp:12
inline constexpr double kDefaultGuardFraction = 0.8;    // params.hpp:13
inline constexpr double kScalingFloor = 9.5367431640625e-7;  // params.hpp:14

namespace detail {
[[noreturn]] inline void raise(phx_status st) {
  const std::string msg = phx_last_error();
  switch (st) {
    case PHX_EINVAL: throw std::invalid_argument(msg);
    case PHX_ENUMERIC: throw std::runtime_error(msg);
    case PHX_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error("phx device error: " + msg);
  }
}
inline void check(phx_status st) {
  if (st != PHX_OK) raise(st);
}
}  // namespace detail

// LinearOperator (linop.hpp:19-37) for a device-resident CSR matrix.
// Immutable after construction; copies share the device handle.
class LinearOperator {
 public:
  LinearOperator() = default;
  Index dim() const { return h_ ? phx_op_dim(h_.get()) : 0; }
  const std::string& label() const { return label_; }
  // A*X (linop.cpp:10-24)
  Matrix apply(const Matrix& X) const {
    if (!h_) throw std::logic_error("LinearOperator::apply: operator is empty");
    if (X.rows() != dim())
      throw std::invalid_argument("LinearOperator::apply: block has " + std::to_string(X.rows()) +
                                  " rows, operator dimension is " + std::to_string(dim()));
    Matrix Y(X.rows(), X.cols());
    detail::check(phx_apply(h_.get(), X.data(), X.rows(), X.cols(), Y.data(), Y.rows()));
    return Y;
  }
  phx_op handle() const { return h_.get(); }

 private:
  friend LinearOperator csr_operator(Index, const std::vector<std::int64_t>&,
                                     const std::vector<std::int32_t>&, const std::vector<double>&,
                                     std::string, int);
  std::shared_ptr<phx_op_s> h_;
  std::string label_;
};

// CSR factory (the entry point for sparse operators; the reference has only
// dense_operator and user ApplyFns, linop.cpp:26-38).
inline LinearOperator csr_operator(Index n, const std::vector<std::int64_t>& row_ptr,
                                   const std::vector<std::int32_t>& col_idx,
                                   const std::vector<double>& vals, std::string label = {},
                                   int device = -1) {
  if (Index(row_ptr.size()) != n + 1) throw std::invalid_argument("csr_operator: row_ptr size");
  phx_op h = nullptr;
  detail::check(phx_op_create_csr(n, row_ptr.data(), col_idx.data(), vals.data(), device, &h));
  LinearOperator op;
  op.h_ = std::shared_ptr<phx_op_s>(h, [](phx_op p) { phx_op_destroy(p); });
  op.label_ = std::move(label);
  return op;
}

// dense_operator (linop.cpp:26-38): square, finite, every entry stored (as
// CSR, rows in natural column order -- the reference's dense product sums a
// row in the same order); the same checks and messages.
inline LinearOperator dense_operator(const Matrix& A, std::string label = "dense",
                                     int device = -1) {
  if (A.rows() != A.cols()) throw std::invalid_argument("dense_operator: matrix must be square");
  const Index n = A.rows();
  if (n == 0) throw std::invalid_argument("dense_operator: matrix must be non-empty");
  std::vector<std::int64_t> rp(size_t(n + 1));
  std::vector<std::int32_t> ci(size_t(n * n));
  std::vector<double> av(size_t(n * n));
  for (Index i = 0; i < n; ++i) {
    rp[size_t(i)] = i * n;
    for (Index j = 0; j < n; ++j) {
      const double x = A(i, j);
      if (!(x - x == 0.0)) throw std::invalid_argument("dense_operator: matrix has non-finite entries");
      ci[size_t(i * n + j)] = std::int32_t(j);
      av[size_t(i * n + j)] = x;
    }
  }
  rp[size_t(n)] = n * n;
  return csr_operator(n, rp, ci, av, std::move(label), device);
}

// (A - xi I) X (linop.cpp:40-49)
inline Matrix shifted_apply(const LinearOperator& op, double xi, const Matrix& X) {
  Matrix Y(X.rows(), X.cols());
  detail::check(phx_shifted_apply(op.handle(), xi, X.data(), X.rows(), X.cols(), Y.data(), Y.rows()));
  return Y;
}

struct ScalingShift {  // params.hpp:34-41
  double s = 1.0;
  double xi = 0.0;
  double s0 = 1.0;
  double f_min = 0.0;
  int m = kDefaultDegree;
  int r = 0;
};

struct RunRecord {  // phi_single.hpp:16-21
  long s_effective = 1;
  int series_len_S = 0;
  std::vector<int> series_lens_F;
  long matvecs = 0;
};

namespace detail {
// recovery sweeps of an evaluation, s_eff - 1 with s_eff = max(1,
// ceil(s * max|t|)) (phi_block.cpp:57-59): the size of the run record's
// series_lens_F buffer
inline std::size_t sweeps_of(double s, const double* t, Index r) {
  double tmax = 0.0;
  for (Index i = 0; i < r; ++i) tmax = std::max(tmax, t[i] < 0 ? -t[i] : t[i]);
  const double prod = s * tmax;
  if (!(prod < 2147483647.0)) return 1;  // the evaluator rejects it with the reference's error
  const double c = prod <= 1.0 ? 1.0 : double(std::int64_t(prod) + (double(std::int64_t(prod)) < prod));
  return std::size_t(std::max(1.0, c - 1.0));
}
inline phx_scaling_shift to_c(const ScalingShift& s) {
  return phx_scaling_shift{s.s, s.xi, s.s0, s.f_min, s.m, s.r};
}
inline ScalingShift from_c(const phx_scaling_shift& c) {
  return ScalingShift{c.s, c.xi, c.s0, c.f_min, c.m, c.r};
}
}  // namespace detail

// select_parameters (params.hpp:75-77)
inline ScalingShift select_parameters(const LinearOperator& op, int m = kDefaultDegree,
                                      double tol = -1.0,
                                      double delta = kDefaultGuardFraction) {
  phx_scaling_shift out{};
  detail::check(phx_select_parameters(op.handle(), m, tol, delta, &out));
  return detail::from_c(out);
}

struct BlockPhiRequest {  // phi_block.hpp:14-20
  Vector t;
  Vector alpha;
  Matrix V;
  double tol = -1.0;
  ScalingShift params;
};

struct BlockPhiResult {  // phi_block.hpp:22-25
  Matrix W;
  RunRecord stats;
};

// phimv_block (phi_block.hpp:30-31)
inline BlockPhiResult phimv_block(const LinearOperator& op, const BlockPhiRequest& req) {
  if (req.t.size() == 0) throw std::invalid_argument("phimv_block: at least one abscissa required");
  if (req.alpha.size() != req.t.size())
    throw std::invalid_argument("phimv_block: t and alpha lengths differ");
  if (req.V.cols() < 1) throw std::invalid_argument("phimv_block: V must have at least one column");
  if (req.V.rows() != op.dim())
    throw std::invalid_argument("phimv_block: V row count does not match operator");
  BlockPhiResult out;
  out.W = Matrix(req.V.rows(), req.t.size());
  const phx_scaling_shift ss = detail::to_c(req.params);
  std::vector<int32_t> lens(detail::sweeps_of(req.params.s, req.t.data(), req.t.size()));
  phx_run_record rec{0, 0, 0, lens.data(), int64_t(lens.size()), 0};
  detail::check(phx_phimv_block(op.handle(), int32_t(req.t.size()), req.t.data(), req.alpha.data(),
                                int32_t(req.V.cols() - 1), req.V.data(), req.V.rows(), req.tol, &ss,
                                out.W.data(), out.W.rows(), &rec));
  out.stats.s_effective = rec.s_effective;
  out.stats.series_len_S = rec.series_len_S;
  out.stats.series_lens_F.assign(lens.begin(), lens.begin() + std::min<int64_t>(rec.n_sweeps, int64_t(lens.size())));
  out.stats.matvecs = rec.matvecs;
  return out;
}

struct PhiRequest {  // phi_single.hpp:26-32
  double t = 1.0;
  double alpha = 1.0;
  Matrix V;
  double tol = -1.0;
  ScalingShift params;
};

struct PhiResult {  // phi_single.hpp:34-39
  Vector w;
  Vector exp_v0;
  Vector tail;
  RunRecord stats;
};

// phimv (phi_single.hpp:44)
inline PhiResult phimv(const LinearOperator& op, const PhiRequest& req) {
  const Index n = op.dim();
  if (req.V.cols() < 1) throw std::invalid_argument("phimv: V must have at least one column");
  if (req.V.rows() != n) throw std::invalid_argument("phimv: V row count does not match operator");
  PhiResult out;
  out.w = Vector(n);
  out.exp_v0 = Vector(n);
  out.tail = Vector(n);
  const phx_scaling_shift ss = detail::to_c(req.params);
  std::vector<int32_t> lens(detail::sweeps_of(req.params.s, &req.t, 1));
  phx_run_record rec{0, 0, 0, lens.data(), int64_t(lens.size()), 0};
  detail::check(phx_phimv(op.handle(), req.t, req.alpha, int32_t(req.V.cols() - 1), req.V.data(),
                          req.V.rows(), req.tol, &ss, out.w.data(), out.exp_v0.data(),
                          out.tail.data(), &rec));
  out.stats.s_effective = rec.s_effective;
  out.stats.series_len_S = rec.series_len_S;
  out.stats.series_lens_F.assign(lens.begin(), lens.begin() + std::min<int64_t>(rec.n_sweeps, int64_t(lens.size())));
  out.stats.matvecs = rec.matvecs;
  return out;
}

// ---------------------------------------------------------------------------
// The evaluator's consumer (integrator.hpp, problems.hpp:46-70)
struct ExpRK4s6Coefficients {  // integrator.hpp:13-19
  static constexpr double c2 = 0.5;
  static constexpr double c3 = 0.5;
  static constexpr double c4 = 1.0 / 3.0;
  static constexpr double c5 = 5.0 / 6.0;
  static constexpr double c6 = 1.0 / 3.0;
};

// ADRProblem (problems.hpp:46-66) with the operator stored as CSR.
struct ADRProblem {
  int nx = 0;
  int ny = 0;
  double eps = 1e-3;
  double alpha_adv = -0.5;
  double gamma = 1000.0;
  LinearOperator op;
  Vector u0;
  double t_end = 0.5;
  // gamma u (u - 1/2)(1 - u) (problems.cpp:180-182)
  Vector reaction(const Vector& u) const {
    Vector g(u.size());
    for (Index i = 0; i < u.size(); ++i) g(i) = gamma * u(i) * (u(i) - 0.5) * (1.0 - u(i));
    return g;
  }
};

inline ADRProblem adr_build(int nx, int ny, double eps = 1e-3, double alpha_adv = -0.5,
                            double gamma = 1000.0, int device = -1) {
  if (nx < 8 || ny < 8) throw std::invalid_argument("adr_build: grid must be at least 8x8");
  const Index n = Index(nx) * Index(ny);
  std::vector<std::int64_t> rp(size_t(n + 1));
  std::vector<std::int32_t> ci(size_t(5 * n));
  std::vector<double> av(size_t(5 * n));
  ADRProblem prob;
  prob.u0 = Vector(n);
  detail::check(phx_adr_csr(nx, ny, eps, alpha_adv, rp.data(), ci.data(), av.data(),
                            prob.u0.data()));
  ci.resize(size_t(rp[size_t(n)]));
  av.resize(size_t(rp[size_t(n)]));
  prob.nx = nx;
  prob.ny = ny;
  prob.eps = eps;
  prob.alpha_adv = alpha_adv;
  prob.gamma = gamma;
  prob.op = csr_operator(n, rp, ci, av, "adr", device);
  return prob;
}

struct StepState {  // integrator.hpp:21-25
  double t = 0.0;
  Vector u;
  double h = 0.0;
};

struct StepRecord {  // integrator.hpp:27-30
  double t = 0.0;
  RunRecord calls[4];
};

namespace detail {
inline RunRecord from_rec(const phx_run_record& r, const std::vector<int32_t>& lens) {
  RunRecord o;
  o.s_effective = r.s_effective;
  o.series_len_S = r.series_len_S;
  o.series_lens_F.assign(lens.begin(),
                         lens.begin() + std::min<int64_t>(r.n_sweeps, int64_t(lens.size())));
  o.matvecs = r.matvecs;
  return o;
}
}  // namespace detail

// exprk4s6_step (integrator.hpp:36-38)
inline Vector exprk4s6_step(const ADRProblem& problem, const StepState& state, double tol,
                            const ScalingShift& params, StepRecord* record = nullptr) {
  Vector out(state.u.size());
  const phx_scaling_shift ss = detail::to_c(params);
  // every stage's abscissae are <= h: at most sweeps_of(s, h) sweeps each
  const std::size_t cap = detail::sweeps_of(params.s, &state.h, 1);
  std::vector<std::vector<int32_t>> lens(4, std::vector<int32_t>(cap));
  phx_run_record recs[4];
  for (int k = 0; k < 4; ++k)
    recs[k] = phx_run_record{0, 0, 0, lens[size_t(k)].data(), int64_t(cap), 0};
  detail::check(phx_exprk4s6_step(problem.op.handle(), problem.gamma, state.u.data(), state.h,
                                  tol, &ss, out.data(), record ? recs : nullptr));
  if (record) {
    record->t = state.t;
    for (int k = 0; k < 4; ++k) record->calls[k] = detail::from_rec(recs[k], lens[size_t(k)]);
  }
  return out;
}

struct IntegrateResult {  // integrator.hpp:40-44
  Vector u;
  double t = 0.0;
  std::vector<StepRecord> steps;
};

// integrate (integrator.hpp:47-49)
inline IntegrateResult integrate(const ADRProblem& problem, double h, double t_end, double tol,
                                 const ScalingShift& params, bool keep_records = true) {
  IntegrateResult out;
  out.u = Vector(problem.u0.size());
  const phx_scaling_shift ss = detail::to_c(params);
  int64_t nrec = 0;
  if (keep_records && h > 0.0) {
    const double q = t_end / h;
    if (q >= 0.5 && q < 1.0e6 + 0.5) nrec = 4 * int64_t(std::llround(q));
  }
  // per record: the sweeps of an evaluation with abscissae <= h
  const int64_t kLens = int64_t(detail::sweeps_of(params.s, &h, 1));
  std::vector<int32_t> lens(size_t(std::max<int64_t>(1, nrec) * kLens));
  std::vector<phx_run_record> recs(size_t(std::max<int64_t>(1, nrec)));
  for (int64_t k = 0; k < nrec; ++k)
    recs[size_t(k)] = phx_run_record{0, 0, 0, lens.data() + k * kLens, kLens, 0};
  int64_t nsteps = 0;
  detail::check(phx_integrate(problem.op.handle(), problem.gamma, problem.u0.data(), h, t_end,
                              tol, &ss, out.u.data(), &out.t, &nsteps,
                              nrec ? recs.data() : nullptr, nrec));
  for (int64_t s = 0; s < nsteps && 4 * s + 3 < nrec; ++s) {
    StepRecord st;
    st.t = double(s) * h;
    for (int k = 0; k < 4; ++k) {
      const phx_run_record& r = recs[size_t(4 * s + k)];
      const std::vector<int32_t> l(r.series_lens_F, r.series_lens_F + kLens);
      st.calls[k] = detail::from_rec(r, l);
    }
    out.steps.push_back(std::move(st));
  }
  return out;
}

}  // namespace phiact
