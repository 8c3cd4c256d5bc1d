// ============================================================================
//  phx ORACLE — TEST INFRASTRUCTURE ONLY.
//
//  A plain C++ CPU restatement of the reference hot path (arXiv 2509.26475,
//  "phiact"): parameter selection (Alg. 1) and the block phi evaluator
//  (Alg. 3), plus the single-combination evaluator (Alg. 2) and the
//  long-double augmented-matrix references used as the high-precision check.
//
//  It is the CHECKER for the CUDA product in paper_2509_26475_b200/: only
//  tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
//  arm load it.  The product never links or calls it.
//
//  The reference library itself cannot be compiled here (it needs Eigen3,
//  which is absent from the image, plus an un-shipped vendor/ tree), so this
//  file restates the algorithm.  Every function cites the reference file:line
//  it follows (paths relative to the reference's proj/ directory).
//
//  Numerical contract (see DESIGN.md §3 and SURVEY.md Appendix A):
//   * every operation is an individually rounded IEEE double op in the same
//     order as the reference statement it restates; built -ffp-contract=off;
//   * where the reference delegates the ORDER of a reduction to Eigen
//     (row-sum redux, squaredNorm, GEMV), the order is unpinnable here and is
//     FIXED by this file ("canonical order"), identically in the CUDA
//     kernels:
//       - matrix inf-norm row sums: pairwise tree over the columns in natural
//         order, padded with zeros to the next power of two;
//       - sums of squares: 4096-element chunks (Eigen stableNorm blocking),
//         256 lanes per chunk, lane l sums elements l, l+256, ... in order,
//         lanes combined by a pairwise tree;
//       - CSR products and GEMVs: sequential accumulation from +0 in storage
//         order;
//       - structured GEMMs (Vw*Kiter, Sadv*Jexp): ascending source column,
//         accumulated from +0; the zero products Eigen would add are exact
//         no-ops for finite data and are skipped.
// ============================================================================
#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cerrno>
#include <cstdio>
#include <functional>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

namespace orc {

using Vec = std::vector<double>;

// Column-major dense matrix (the reference's Eigen::MatrixXd layout,
// linop.hpp:12).
struct Mat {
  long rows = 0, cols = 0;
  Vec a;
  Mat() = default;
  Mat(long r, long c) : rows(r), cols(c), a(size_t(r) * size_t(c), 0.0) {}
  double* col(long j) { return a.data() + size_t(j) * size_t(rows); }
  const double* col(long j) const { return a.data() + size_t(j) * size_t(rows); }
  double& operator()(long i, long j) { return a[size_t(i) + size_t(j) * size_t(rows)]; }
  double operator()(long i, long j) const { return a[size_t(i) + size_t(j) * size_t(rows)]; }
};

// CSR view.  The reference has no CSR type; CSR operators enter through its
// only extension point, LinearOperator's ApplyFn (linop.hpp:19-37).  This is
// the ApplyFn: Y(i,c) = sum over the row's entries in storage order,
// accumulated sequentially from +0 (Eigen's row-major sparse*dense kernel
// has the same shape).
struct Op {
  long n = 0;
  const int64_t* rp = nullptr;
  const int32_t* ci = nullptr;
  const double* v = nullptr;
};

// Row-parallel loops for the CPU timing arms (bench.py): orc_set_threads(T)
// splits every n-sized loop of phimv_block into T contiguous row ranges.
// Rows are independent and the maxima order-free, so results are bitwise
// those of one thread (the reference itself is single-threaded; T = 1 is
// its configuration and the default).
static int g_threads = 1;
template <class F>
static void pfor(long n, F&& f) {
  const long T = (n < 65536) ? 1 : long(g_threads);
  if (T <= 1) {
    f(0L, n);
    return;
  }
  const long chunk = (n + T - 1) / T;
  std::vector<std::thread> th;
  for (long q = 1; q < T; ++q) {
    const long lo = q * chunk, hi = std::min(n, lo + chunk);
    if (lo < hi) th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  f(0L, std::min(n, chunk));
  for (auto& x : th) x.join();
}

// LinearOperator::apply (linop.cpp:10-24) for a CSR ApplyFn.
static void apply_into(const Op& op, const double* X, long ldx, long k, double* Y,
                       long ldy) {
  for (long c = 0; c < k; ++c) {
    const double* x = X + size_t(c) * size_t(ldx);
    double* y = Y + size_t(c) * size_t(ldy);
    pfor(op.n, [&](long lo, long hi) {
      for (long i = lo; i < hi; ++i) {
        double acc = 0.0;
        for (int64_t e = op.rp[i]; e < op.rp[i + 1]; ++e) acc = acc + op.v[e] * x[op.ci[e]];
        y[i] = acc;
      }
    });
  }
}

static Mat apply(const Op& op, const Mat& X) {
  if (X.rows != op.n)
    throw std::invalid_argument("LinearOperator::apply: block has " +
                                std::to_string(X.rows) +
                                " rows, operator dimension is " + std::to_string(op.n));
  Mat Y(X.rows, X.cols);
  apply_into(op, X.a.data(), X.rows, X.cols, Y.a.data(), Y.rows);
  return Y;
}

// shifted_apply (linop.cpp:40-49): exactly apply() when xi == 0, else
// Y(i) - fl(xi * X(i)).
static Mat shifted_apply(const Op& op, double xi, const Mat& X) {
  if (!std::isfinite(xi)) throw std::invalid_argument("shifted_apply: shift must be finite");
  Mat Y = apply(op, X);
  if (xi == 0.0) return Y;
  for (size_t q = 0; q < Y.a.size(); ++q) Y.a[q] = Y.a[q] - xi * X.a[q];
  return Y;
}

// ---------------------------------------------------------------------------
// Canonical reductions
// ---------------------------------------------------------------------------
static inline double nan_max(double m, double v) {
  // max that lets a NaN through and keeps it (the device path takes the max
  // of the IEEE bit patterns with the sign cleared, where NaN > inf)
  if (std::isnan(m)) return m;
  if (std::isnan(v)) return v;
  return v > m ? v : m;
}

static long pow2ceil(long w) {
  long p = 1;
  while (p < w) p <<= 1;
  return p;
}

// pairwise tree over |x_c|, natural column order padded to a power of two
static double tree_abs(const double* x, long lo, long len, long w) {
  if (len == 1) return lo < w ? std::fabs(x[lo]) : 0.0;
  const long h = len / 2;
  const double a = tree_abs(x, lo, h, w);
  const double b = tree_abs(x, lo + h, h, w);
  return a + b;
}

// Alternative row-sum orders, for the robustness test only
// (tests/test_oracle_port.py::test_rowsum_order_*): the reference's
// `cwiseAbs().rowwise().sum()` (linop.cpp:53) leaves the order to Eigen, whose
// version is not pinned.  Restated from Eigen's published
// sources: 1 = the 4-unrolled packet-wise partial redux of Eigen 3.4
// (p = c0; p += ((c1 + c2) + (c3 + c4)); ...; then the remaining columns one by
// one); 2 = the scalar redux (c0 + c1 + c2 + ..., Eigen 3.3, and 3.4's rows
// outside a full packet); 3 = order 1 for the rows in full 2-row packets
// (SSE2) and order 2 for a last odd row.  0 = the canonical pairwise tree that
// the product implements.  The test shows that every discrete outcome
// (series lengths, sweeps) and hence W is the same under all of them on the
// BASELINE configs.
static int g_rowsum_order = 0;
static double rowsum_abs(const double* row, long cols, long len, long i, long rows) {
  int order = g_rowsum_order;
  if (order == 3) order = (i < (rows & ~1L)) ? 1 : 2;
  if (order == 1) {
    const long size4 = (cols - 1) & ~3L;
    double p = std::fabs(row[0]);
    long c = 1;
    for (; c < size4; c += 4)
      p = p + ((std::fabs(row[c]) + std::fabs(row[c + 1])) + (std::fabs(row[c + 2]) + std::fabs(row[c + 3])));
    for (; c < cols; ++c) p = p + std::fabs(row[c]);
    return p;
  }
  if (order == 2) {
    double p = std::fabs(row[0]);
    for (long c = 1; c < cols; ++c) p = p + std::fabs(row[c]);
    return p;
  }
  return tree_abs(row, 0, len, cols);
}

// inf_norm (linop.cpp:51-54): max_i sum_c |X_ic|; 0 for an empty matrix.
static double inf_norm(const double* X, long rows, long cols, long ld) {
  if (rows == 0 || cols == 0) return 0.0;
  const long len = pow2ceil(cols);
  std::vector<double> part(size_t(std::max(1, g_threads)) + 1, 0.0);
  std::vector<long> starts;
  pfor(rows, [&](long lo, long hi) {
    std::vector<double> row(static_cast<size_t>(cols));
    double m = 0.0;
    for (long i = lo; i < hi; ++i) {
      for (long c = 0; c < cols; ++c) row[size_t(c)] = X[size_t(i) + size_t(c) * size_t(ld)];
      m = nan_max(m, rowsum_abs(row.data(), cols, len, i, rows));
    }
    const long chunk = rows < 65536 ? rows : (rows + g_threads - 1) / g_threads;
    part[size_t(lo / std::max(1L, chunk))] = m;
  });
  double m = 0.0;
  for (double x : part) m = nan_max(m, x);
  return m;
}
static double inf_norm(const Mat& X) { return inf_norm(X.a.data(), X.rows, X.cols, X.rows); }

constexpr long kChunk = 4096;  // Eigen stableNorm block size
constexpr int kLanes = 256;

// sum of fl(fl(x*mul)^2) over one chunk in canonical order
static double chunk_sumsq(const double* x, long len, double mul) {
  double lane[kLanes];
  for (int l = 0; l < kLanes; ++l) {
    double s = 0.0;
    for (long q = l; q < len; q += kLanes) {
      const double y = x[q] * mul;
      s = s + y * y;
    }
    lane[l] = s;
  }
  for (int h = 1; h < kLanes; h *= 2)
    for (int l = 0; l < kLanes; l += 2 * h) lane[l] = lane[l] + lane[l + h];
  return lane[0];
}

// Eigen's plain norm() = sqrt(squaredNorm()); chunks folded sequentially.
static double norm2(const double* x, long n) {
  double ssq = 0.0;
  for (long b = 0; b < n; b += kChunk) ssq = ssq + chunk_sumsq(x + b, std::min(kChunk, n - b), 1.0);
  return std::sqrt(ssq);
}

// Eigen's stableNorm(): blocked scaled sum of squares (Eigen's published
// stable_norm_impl / stable_norm_kernel), restated.  Alignment-peeled head
// blocks are an Eigen memory-layout artifact and are not reproduced: blocks
// start at index 0.
static double stable_norm(const double* x, long n) {
  if (n == 1) return std::fabs(x[0]);
  double scale = 0.0, inv_scale = 1.0, ssq = 0.0;
  for (long b = 0; b < n; b += kChunk) {
    const long len = std::min(kChunk, n - b);
    double maxc = 0.0;
    for (long q = 0; q < len; ++q) maxc = nan_max(maxc, std::fabs(x[b + q]));
    if (maxc > scale) {
      const double ratio = scale / maxc;
      ssq = ssq * (ratio * ratio);
      const double tmp = 1.0 / maxc;
      if (tmp > DBL_MAX) {
        inv_scale = DBL_MAX;
        scale = 1.0 / inv_scale;
      } else if (maxc > DBL_MAX) {
        inv_scale = 1.0;
        scale = maxc;
      } else {
        scale = maxc;
        inv_scale = tmp;
      }
    } else if (maxc != maxc) {
      scale = maxc;
    }
    if (scale > 0.0) ssq = ssq + chunk_sumsq(x + b, len, inv_scale);
  }
  return scale * std::sqrt(ssq);
}

static bool all_finite(const double* x, size_t n) {
  for (size_t q = 0; q < n; ++q)
    if (!std::isfinite(x[q])) return false;
  return true;
}

// ---------------------------------------------------------------------------
// Rng (rng.hpp:15-62): mt19937_64 + Box-Muller with a spare, column-major
// fills.
// ---------------------------------------------------------------------------
class Rng {
 public:
  explicit Rng(uint64_t seed) : gen_(seed) {}
  double uniform() { return double(gen_() >> 11) * 0x1.0p-53; }
  double normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    double u1 = 0.0;
    do {
      u1 = uniform();
    } while (u1 == 0.0);
    const double u2 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * M_PI * u2;
    spare_ = radius * std::sin(angle);
    have_spare_ = true;
    return radius * std::cos(angle);
  }
  Mat matrix(long rows, long cols) {
    Mat out(rows, cols);
    for (long j = 0; j < cols; ++j)
      for (long i = 0; i < rows; ++i) out(i, j) = normal();
    return out;
  }
  Vec vector(long n) {
    Vec out(static_cast<size_t>(n));
    for (long i = 0; i < n; ++i) out[size_t(i)] = normal();
    return out;
  }
  Vec unit_vector(long n) {
    Vec v = vector(n);
    const double nrm = norm2(v.data(), n);
    for (auto& x : v) x = x / nrm;
    return v;
  }

 private:
  std::mt19937_64 gen_;
  bool have_spare_ = false;
  double spare_ = 0.0;
};

// ---------------------------------------------------------------------------
// Parameter selection (params.hpp:12-77, params.cpp)
// ---------------------------------------------------------------------------
constexpr int kDefaultDegree = 61;                 // params.hpp:12
constexpr double kDefaultGuardFraction = 0.8;      // params.hpp:13
constexpr double kScalingFloor = 9.5367431640625e-7;  // 2^-20, params.hpp:14
static double default_tolerance() { return std::ldexp(1.0, -53); }  // params.hpp:15
constexpr uint64_t kFallbackSeed = 0x9e3779b97f4a7c15ull;  // params.cpp:13
constexpr int kSeriesCap = 500;    // phi_single.hpp:11
constexpr int kRecoveryCap = 300;  // phi_single.hpp:12

struct PowerBasis {
  Mat columns;
  Vec logs;
  Vec log_binom;
  int r = 0;
  int m = 0;
  double s0 = 1.0;
};

}  // namespace orc

extern "C" {
typedef struct {
  double s, xi, s0, f_min;
  int32_t m, r;
} orc_scaling_shift;
}

namespace orc {

using ScalingShift = orc_scaling_shift;

static double log_binomial(int m, int j) {  // params.cpp:15-17
  return std::lgamma(m + 1.0) - std::lgamma(j + 1.0) - std::lgamma(m - j + 1.0);
}

// Brent's derivative-free minimizer (golden section + successive parabolic
// interpolation, absolute x tolerance), restated from params.cpp:21-77.  The
// arithmetic order of every update matches the reference statement.
static double brent_minimize(const std::function<double(double)>& f, double a, double b,
                             double tol_x, int max_iter, std::vector<double>* path) {
  const double golden = 0.3819660112501051;
  double x = a + golden * (b - a);
  double w = x, v = x;
  double fx = f(x), fw = fx, fv = fx;
  if (path) { path->push_back(x); path->push_back(fx); }
  double d = 0.0, e = 0.0;
  for (int it = 0; it < max_iter; ++it) {
    const double mid = 0.5 * (a + b);
    const double tol1 = tol_x;
    const double tol2 = 2.0 * tol1;
    if (std::fabs(x - mid) <= tol2 - 0.5 * (b - a)) break;
    bool golden_step = true;
    if (std::fabs(e) > tol1) {
      const double r = (x - w) * (fx - fv);
      double q = (x - v) * (fx - fw);
      double p = (x - v) * q - (x - w) * r;
      q = 2.0 * (q - r);
      if (q > 0.0) p = -p;
      q = std::fabs(q);
      const double e_prev = e;
      e = d;
      if (std::fabs(p) < std::fabs(0.5 * q * e_prev) && p > q * (a - x) && p < q * (b - x)) {
        d = p / q;
        const double u = x + d;
        if (u - a < tol2 || b - u < tol2) d = (x < mid) ? tol1 : -tol1;
        golden_step = false;
      }
    }
    if (golden_step) {
      e = (x < mid) ? b - x : a - x;
      d = golden * e;
    }
    const double u = (std::fabs(d) >= tol1) ? x + d : x + ((d > 0) ? tol1 : -tol1);
    const double fu = f(u);
    if (path) { path->push_back(u); path->push_back(fu); }
    if (fu <= fx) {
      if (u < x) b = x; else a = x;
      v = w; fv = fw;
      w = x; fw = fx;
      x = u; fx = fu;
    } else {
      if (u < x) a = u; else b = u;
      if (fu <= fw || w == x) {
        v = w; fv = fw;
        w = u; fw = fu;
      } else if (fu <= fv || v == x || v == w) {
        v = u; fv = fu;
      }
    }
  }
  return x;
}

// build_power_basis (params.cpp:81-154)
static PowerBasis build_power_basis(const Op& op, int m, double delta) {
  if (m < 1) throw std::invalid_argument("build_power_basis: m must be >= 1");
  if (!(delta > 0.0 && delta <= 1.0))
    throw std::invalid_argument("build_power_basis: delta must be in (0, 1]");
  const long n = op.n;
  const double g_max = delta * std::log(std::numeric_limits<double>::max());
  const double g_min = delta * std::log(std::numeric_limits<double>::min());

  PowerBasis basis;
  basis.m = m;
  basis.log_binom.resize(size_t(m) + 1);
  double ell_max = 0.0;
  for (int j = 0; j <= m; ++j) {
    basis.log_binom[size_t(j)] = log_binomial(m, j);
    ell_max = std::max(ell_max, basis.log_binom[size_t(j)]);
  }

  Rng rng(kFallbackSeed);
  Vec v = rng.unit_vector(n);
  Vec w(static_cast<size_t>(n));
  apply_into(op, v.data(), n, 1, w.data(), n);
  if (!all_finite(w.data(), w.size()))
    throw std::runtime_error("build_power_basis: A*v is not finite; operator rejected");
  if (stable_norm(w.data(), n) == 0.0) {
    v = rng.unit_vector(n);
    apply_into(op, v.data(), n, 1, w.data(), n);
    if (!all_finite(w.data(), w.size()))
      throw std::runtime_error("build_power_basis: A*v is not finite; operator rejected");
  }
  const double first_norm = stable_norm(w.data(), n);
  basis.columns = Mat(n, m + 1);
  std::copy(v.begin(), v.end(), basis.columns.col(0));

  int r = 0;
  for (int k = 1; k <= m; ++k) {
    if (k > 1) apply_into(op, basis.columns.col(k - 1), n, 1, w.data(), n);
    const double norm_w = stable_norm(w.data(), n);
    const double L = norm_w > 0.0 ? std::log(norm_w) : -std::numeric_limits<double>::infinity();
    if (!(L + 0.5 * std::log(k + 1.0) + ell_max <= g_max) || L < g_min) break;
    std::copy(w.begin(), w.end(), basis.columns.col(k));
    basis.logs.push_back(L);
    r = k;
  }
  basis.r = r;
  if (r >= 3) {
    const int j_r = std::max(2, r - 5);
    basis.s0 = std::exp((basis.logs[size_t(r - 1)] - basis.logs[size_t(j_r - 1)]) / (r - j_r));
  } else {
    basis.s0 = std::max(first_norm, 1.0);
  }
  if (!(basis.s0 > 0.0) || !std::isfinite(basis.s0)) basis.s0 = 1.0;

  double scale = 1.0;
  for (int j = 1; j <= r; ++j) {
    scale /= basis.s0;
    double* c = basis.columns.col(j);
    for (long i = 0; i < n; ++i) c[i] = c[i] * scale;
  }
  for (int k = r + 1; k <= m; ++k) {
    double* c = basis.columns.col(k);
    apply_into(op, basis.columns.col(k - 1), n, 1, c, n);
    for (long i = 0; i < n; ++i) c[i] = c[i] / basis.s0;
  }
  return basis;
}

// objective (params.cpp:156-170); GEMV in canonical order
static double objective(const PowerBasis& basis, double xi) {
  if (!std::isfinite(xi)) throw std::invalid_argument("objective: shift must be finite");
  const int m = basis.m;
  const double z = -xi / basis.s0;
  Vec coeff(static_cast<size_t>(m) + 1);
  double zp = 1.0;
  for (int j = m; j >= 0; --j) {
    coeff[size_t(j)] = std::exp(basis.log_binom[size_t(j)]) * zp;
    zp *= z;
  }
  const long n = basis.columns.rows;
  Vec y(static_cast<size_t>(n));
  for (long i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int j = 0; j <= m; ++j) acc = acc + basis.columns(i, j) * coeff[size_t(j)];
    y[size_t(i)] = acc;
  }
  const double norm = stable_norm(y.data(), n);
  return norm > 0.0 ? std::exp(std::log(norm) / m) : 0.0;
}

// minimize_shift (params.cpp:172-189)
static std::pair<double, double> minimize_shift(const PowerBasis& basis,
                                                std::vector<double>* path) {
  const double n = double(basis.columns.rows);
  const double half_width = std::sqrt(n) * basis.s0;
  const auto f = [&basis](double xi) { return objective(basis, xi); };
  const double tol_x = 1e-8 * (1.0 + basis.s0);
  double xi_star = brent_minimize(f, -half_width, half_width, tol_x, 200, path);
  double f_min = f(xi_star);
  const double f0 = f(0.0);
  if (f0 <= f_min) {
    xi_star = 0.0;
    f_min = f0;
  }
  for (const double edge : {-half_width, half_width}) {
    const double fe = f(edge);
    if (fe < f_min) {
      xi_star = edge;
      f_min = fe;
    }
  }
  return {xi_star, f_min};
}

// log_shifted_power (params.cpp:195-209)
static double log_shifted_power(const Op& op, const double* v, double xi, int m) {
  Mat w(op.n, 1);
  std::copy(v, v + op.n, w.col(0));
  double acc = 0.0;
  for (int k = 0; k < m; ++k) {
    w = shifted_apply(op, xi, w);
    const double nw = stable_norm(w.col(0), op.n);
    if (!(nw > 0.0) || !std::isfinite(nw))
      return nw == 0.0 ? -std::numeric_limits<double>::infinity()
                       : std::numeric_limits<double>::infinity();
    acc += std::log(nw);
    for (long i = 0; i < op.n; ++i) w.a[size_t(i)] = w.a[size_t(i)] / nw;
  }
  return acc;
}

// parameters_for_shift (params.cpp:213-239)
static ScalingShift parameters_for_shift(const Op& op, const PowerBasis& basis, double xi,
                                         double tol) {
  if (!(tol > 0.0)) throw std::invalid_argument("parameters_for_shift: tol must be positive");
  const int m = basis.m;
  const double f_basis = objective(basis, xi);
  const double log_nu = log_shifted_power(op, basis.columns.col(0), xi, m);
  const double f_direct = std::isfinite(log_nu) ? std::exp(log_nu / m) / basis.s0 : 0.0;
  const double f_val = std::max(f_basis, f_direct) * (1.0 + 1e-6);
  ScalingShift out{};
  out.xi = xi;
  out.s0 = basis.s0;
  out.f_min = f_val;
  out.m = m;
  out.r = basis.r;
  const double denom = std::exp((std::log(tol) + std::lgamma(m + 1.0)) / m);
  out.s = f_val > 0.0 ? basis.s0 * f_val / denom : 0.0;
  out.s = std::max(out.s, kScalingFloor);
  if (!std::isfinite(out.s)) throw std::runtime_error("parameters_for_shift: scaling is not finite");
  return out;
}

// select_parameters (params.cpp:241-247)
static ScalingShift select_parameters(const Op& op, int m, double tol, double delta) {
  if (tol <= 0.0) tol = default_tolerance();
  const PowerBasis basis = build_power_basis(op, m, delta);
  const double xi_star = minimize_shift(basis, nullptr).first;
  return parameters_for_shift(op, basis, xi_star, tol);
}

// ---------------------------------------------------------------------------
// Block evaluator (phi_block.cpp:48-157)
// ---------------------------------------------------------------------------
struct RunRecord {
  long s_effective = 1;
  int series_len_S = 0;
  std::vector<int> series_lens_F;
  long matvecs = 0;
};

struct Trace {  // per-term stopping-test norms, for term-by-term parity
  std::vector<double>* out = nullptr;
  void add(double kind, double a, double b) {
    if (!out) return;
    out->push_back(kind);
    out->push_back(a);
    out->push_back(b);
  }
};

[[noreturn]] static void diverged(const char* who, const char* where, int k) {
  throw std::runtime_error(std::string(who) + ": " + where +
                           " produced a non-finite term at index " + std::to_string(k));
}
[[noreturn]] static void no_convergence(const char* who, const char* where, int cap) {
  throw std::runtime_error(std::string(who) + ": " + where + " did not converge within " +
                           std::to_string(cap) + " terms");
}

// Jexp chain of exp(J (x) Delta / s) (nilpotent.cpp:12-21, 38-52): entry
// (l*r+k, j*r+k), 1 <= l <= j <= p, equals c_{j-l} with c_0 = 1 and
// c_d = fl(fl(c_{d-1} * fl(alpha_k / s)) / d); block 0 is the identity.
static std::vector<double> jexp_chain(double alpha, double s, int p) {
  std::vector<double> c(static_cast<size_t>(p) + 1, 0.0);
  c[0] = 1.0;
  const double ka = alpha / s;
  for (int d = 1; d <= p; ++d) c[size_t(d)] = (c[size_t(d - 1)] * ka) / double(d);
  return c;
}

struct BlockResult {
  Mat W;
  RunRecord rec;
};

// phases (timing arms only): [setup, S terms, S terms run, promotion,
// sweeps, sweeps run, assembly, first S term, first sweep] seconds / counts.  max_s_terms / max_sweeps
// > 0 stop the S series / the recovery after that many (a timing SAMPLE:
// W is then not the evaluation's result).
static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static BlockResult phimv_block(const Op& op, const Vec& t, const Vec& alpha, const Mat& V,
                               double req_tol, const ScalingShift& params, Trace tr,
                               int max_s_terms = 0, int max_sweeps = 0,
                               double* phases = nullptr, double* term_times = nullptr) {
  double tp = now_s();
  auto lap = [&](int slot) {
    const double x = now_s();
    if (phases) phases[slot] += x - tp;
    tp = x;
  };
  // check_request (phi_block.cpp:15-27)
  if (t.empty()) throw std::invalid_argument("phimv_block: at least one abscissa required");
  if (alpha.size() != t.size()) throw std::invalid_argument("phimv_block: t and alpha lengths differ");
  if (V.cols < 1) throw std::invalid_argument("phimv_block: V must have at least one column");
  if (V.rows != op.n) throw std::invalid_argument("phimv_block: V row count does not match operator");
  if (!all_finite(t.data(), t.size()) || !all_finite(alpha.data(), alpha.size()) ||
      !all_finite(V.a.data(), V.a.size()))
    throw std::invalid_argument("phimv_block: inputs must be finite");

  const double tol = req_tol > 0.0 ? req_tol : default_tolerance();
  const long r = long(t.size());
  const int p = int(V.cols) - 1;
  const double xi = params.xi;
  const long n = op.n;
  const long w = (p + 1) * r;

  RunRecord rec;
  double tmax = 0.0;
  for (double ti : t) tmax = std::max(tmax, std::fabs(ti));
  const long s = std::max<long>(1, long(std::ceil(params.s * tmax)));  // :58-59
  rec.s_effective = s;

  Vec mu(static_cast<size_t>(r));
  for (long i = 0; i < r; ++i) {  // :62-68
    mu[size_t(i)] = std::exp(xi * t[size_t(i)] / double(s));
    if (!std::isfinite(mu[size_t(i)]))
      throw std::runtime_error("phimv_block: shift undo factor e^{t xi / s} overflows");
  }

  // Kiter = kron_shifted(J, alpha, t, xi)/s (nilpotent.cpp:54-71, :74):
  // diagonal fl(-fl(xi t_i)/s), superdiagonal blocks (j-1 -> j, 2<=j<=p)
  // fl(alpha_i/s).
  Vec Kd(static_cast<size_t>(r)), Ka(static_cast<size_t>(r)), tos(static_cast<size_t>(r));
  std::vector<std::vector<double>> jc(static_cast<size_t>(r));
  for (long i = 0; i < r; ++i) {
    Kd[size_t(i)] = (0.0 - xi * t[size_t(i)]) / double(s);
    Ka[size_t(i)] = (1.0 * alpha[size_t(i)]) / double(s);
    tos[size_t(i)] = t[size_t(i)] / double(s);  // :85
    jc[size_t(i)] = jexp_chain(alpha[size_t(i)], double(s), p);
  }

  // Vw: block j holds v_src(j) * fl(mu_i / s), src 0 -> 0, j -> p+1-j (:76-83)
  Mat Vw(n, w);
  for (int j = 0; j <= p; ++j) {
    const long src = j == 0 ? 0 : p + 1 - j;
    for (long i = 0; i < r; ++i) {
      const double g = mu[size_t(i)] / double(s);
      const double* vs = V.col(src);
      double* dst = Vw.col(j * r + i);
      pfor(n, [&](long lo, long hi) {
        for (long q = lo; q < hi; ++q) dst[q] = vs[q] * g;
      });
    }
  }
  const size_t nw = size_t(n) * size_t(w);
  // elementwise pass over a whole block, row-parallel
  auto each = [&](auto&& f) {
    pfor(long(nw), [&](long lo, long hi) {
      for (long q = lo; q < hi; ++q) f(size_t(q));
    });
  };

  Mat S = Vw, D = Vw;
  int k = 1;
  double sigma = 1.0;
  double c1 = std::numeric_limits<double>::infinity();
  double c2 = inf_norm(D);
  double nS = inf_norm(S);
  tr.add(0, c2, nS);
  Mat Vn(n, w), Dn(n, w);
  lap(0);
  while (c1 + c2 > tol * nS) {  // :93
    if (max_s_terms > 0 && k - 1 >= max_s_terms) break;  // timing sample only
    if (k >= kSeriesCap) no_convergence("phimv_block", "series", kSeriesCap);
    const double t_term = now_s();
    ++k;
    c1 = c2;
    sigma *= k;
    // Vw = Vw * Kiter (:98): ascending source column, from +0
    for (int j = 0; j <= p; ++j)
      for (long i = 0; i < r; ++i) {
        const long c = j * r + i;
        const double* self = Vw.col(c);
        double* out = Vn.col(c);
        const double ka = Ka[size_t(i)], kd = Kd[size_t(i)];
        if (j >= 2) {
          const double* lw = Vw.col(c - r);
          pfor(n, [&](long lo, long hi) {
            for (long q = lo; q < hi; ++q) {
              double acc = 0.0;
              acc = acc + lw[q] * ka;
              acc = acc + self[q] * kd;
              out[q] = acc;
            }
          });
        } else {
          pfor(n, [&](long lo, long hi) {
            for (long q = lo; q < hi; ++q) {
              double acc = 0.0;
              acc = acc + self[q] * kd;
              out[q] = acc;
            }
          });
        }
      }
    std::swap(Vw, Vn);
    // D = shifted_apply(op, xi, D) (:99; linop.cpp:40-49), into a second block
    apply_into(op, D.a.data(), n, w, Dn.a.data(), n);
    if (xi != 0.0) each([&](size_t q) { Dn.a[q] = Dn.a[q] - xi * D.a[q]; });
    std::swap(D, Dn);
    rec.matvecs += (p + 1) * r;
    for (int j = 0; j <= p; ++j)  // :101
      for (long i = 0; i < r; ++i) {
        double* dc = D.col(j * r + i);
        const double ts = tos[size_t(i)];
        pfor(n, [&](long lo, long hi) {
          for (long q = lo; q < hi; ++q) dc[q] = dc[q] * ts;
        });
      }
    each([&](size_t q) { D.a[q] = D.a[q] + Vw.a[q]; });  // :102
    c2 = inf_norm(D) / sigma;                            // :103
    if (!std::isfinite(c2)) diverged("phimv_block", "series", k);
    each([&](size_t q) { S.a[q] = S.a[q] + D.a[q] / sigma; });  // :105
    nS = inf_norm(S);
    tr.add(1, c2, nS);
    if (phases) {
      phases[2] += 1.0;
      if (phases[2] == 1.0) phases[7] = now_s() - tp;  // the first S term alone
    }
    if (term_times) term_times[k - 2] = now_s() - t_term;
  }
  rec.series_len_S = k;
  lap(1);

  // promotion (:109-120)
  const long fcols = p == 0 ? r : 2 * r;
  Mat F(n, fcols);
  std::copy(S.col(0), S.col(0) + size_t(n) * size_t(r), F.col(0));
  if (p > 0) std::copy(S.col(p * r), S.col(p * r) + size_t(n) * size_t(r), F.col(r));
  {
    Mat FL(n, r);
    std::copy(F.col(0), F.col(0) + size_t(n) * size_t(r), FL.col(0));
    Mat AF(n, r);
    apply_into(op, FL.a.data(), n, r, AF.a.data(), n);
    rec.matvecs += r;
    for (long i = 0; i < r; ++i) {
      double* a = AF.col(i);
      double* f = F.col(i);
      const double* v0 = V.col(0);
      for (long q = 0; q < n; ++q) {
        const double sc = a[q] * t[size_t(i)];
        f[q] = sc + v0[q];
      }
    }
  }

  lap(3);
  // recovery sweeps (:122-146)
  Mat& Sadv = S;
  Mat E(n, fcols), Fn(n, fcols);
  const size_t nf = size_t(n) * size_t(fcols);
  auto eachf = [&](auto&& f) {
    pfor(long(nf), [&](long lo, long hi) {
      for (long q = lo; q < hi; ++q) f(size_t(q));
    });
  };
  for (long sweep = 1; sweep < s; ++sweep) {
    if (max_sweeps > 0 && sweep > max_sweeps) break;  // timing sample only
    if (phases) phases[5] += 1.0;
    E = F;
    int kk = 0;
    double d1 = std::numeric_limits<double>::infinity();
    double d2 = inf_norm(F);
    double nE = inf_norm(E);
    tr.add(2, d2, nE);
    while (d1 + d2 > tol * nE) {
      if (kk >= kRecoveryCap) no_convergence("phimv_block", "recovery sweep", kRecoveryCap);
      ++kk;
      d1 = d2;
      // F = shifted_apply(op, xi, F) (linop.cpp:40-49), into a second block
      apply_into(op, F.a.data(), n, fcols, Fn.a.data(), n);
      if (xi != 0.0) eachf([&](size_t q) { Fn.a[q] = Fn.a[q] - xi * F.a[q]; });
      std::swap(F, Fn);
      const double dkk = double(kk);
      eachf([&](size_t q) { F.a[q] = F.a[q] / dkk; });
      rec.matvecs += fcols;
      for (long c = 0; c < fcols; ++c) {
        const double sc = tos[size_t(c % r)];
        double* fc = F.col(c);
        pfor(n, [&](long lo, long hi) {
          for (long q = lo; q < hi; ++q) fc[q] = fc[q] * sc;
        });
      }
      d2 = inf_norm(F);
      if (!std::isfinite(d2)) diverged("phimv_block", "recovery sweep", kk);
      eachf([&](size_t q) { E.a[q] = E.a[q] + F.a[q]; });
      nE = inf_norm(E);
      tr.add(3, d2, nE);
    }
    rec.series_lens_F.push_back(kk);
    if (phases && phases[5] == 1.0) phases[8] = -1.0;  // marker: first sweep's end below
    for (long c = 0; c < fcols; ++c) {  // :141-142
      const double sc = mu[size_t(c % r)];
      double* ec = E.col(c);
      for (long q = 0; q < n; ++q) ec[q] = ec[q] * sc;
    }
    // Sadv = Sadv * Jexp (:143), blocks p..1 in place (block j reads 1..j)
    for (int j = p; j >= 1; --j)
      for (long i = 0; i < r; ++i) {
        const std::vector<double>& cc = jc[size_t(i)];
        double* out = Sadv.col(j * r + i);
        for (long q = 0; q < n; ++q) {
          double acc = 0.0;
          for (int l = 1; l <= j; ++l) acc = acc + Sadv(q, l * r + i) * cc[size_t(j - l)];
          out[q] = acc;
        }
      }
    if (p > 0)  // :144
      for (long i = 0; i < r; ++i) {
        double* fr = F.col(r + i);
        const double* er = E.col(r + i);
        const double* sp = Sadv.col(p * r + i);
        for (long q = 0; q < n; ++q) fr[q] = er[q] + sp[q];
      }
    std::copy(E.col(0), E.col(0) + size_t(n) * size_t(r), F.col(0));  // :145
    if (phases && phases[8] == -1.0) phases[8] = now_s() - tp;  // the first sweep alone
  }
  lap(4);

  BlockResult out;  // :148-154
  out.W = Mat(n, r);
  for (long i = 0; i < r; ++i)
    for (long q = 0; q < n; ++q) {
      double wv = F(q, i);
      if (p > 0) wv = wv + F(q, r + i) * alpha[size_t(i)];
      out.W(q, i) = wv;
    }
  out.rec = std::move(rec);
  lap(6);
  return out;
}

// ---------------------------------------------------------------------------
// Single-combination evaluator (phi_single.cpp:38-127); r = 1 with the
// single variant's operation order (D = fl(t/s) Y + Vw, F = fl(t/(s kk)) Y).
// ---------------------------------------------------------------------------
struct SingleResult {
  Vec w, exp_v0, tail;
  RunRecord rec;
};

static SingleResult phimv(const Op& op, double t, double alpha, const Mat& V, double req_tol,
                          const ScalingShift& params) {
  if (V.cols < 1) throw std::invalid_argument("phimv: V must have at least one column");
  if (V.rows != op.n) throw std::invalid_argument("phimv: V row count does not match operator");
  if (!all_finite(V.a.data(), V.a.size()))
    throw std::invalid_argument("phimv: V has non-finite entries");
  if (!std::isfinite(t) || !std::isfinite(alpha))
    throw std::invalid_argument("phimv: t and alpha must be finite");
  const double tol = req_tol > 0.0 ? req_tol : default_tolerance();
  const int p = int(V.cols) - 1;
  const double xi = params.xi;
  const long n = op.n;
  RunRecord rec;
  const long s = std::max<long>(1, long(std::ceil(std::fabs(t) * params.s)));
  rec.s_effective = s;
  const double mu = std::exp(t * xi / double(s));
  if (!std::isfinite(mu)) throw std::runtime_error("phimv: shift undo factor e^{t xi / s} overflows");
  const std::vector<double> jc = jexp_chain(alpha, double(s), p);
  // Jiter = (alpha J - t xi I)/s: superdiag fl(alpha/s), diag fl(-fl(t xi)/s)
  const double jd = (0.0 - t * xi) / double(s);
  const double ja = (alpha * 1.0 - t * xi * 0.0) / double(s);
  Mat Vw(n, p + 1);
  std::copy(V.col(0), V.col(0) + n, Vw.col(0));
  for (int j = 1; j <= p; ++j) std::copy(V.col(p + 1 - j), V.col(p + 1 - j) + n, Vw.col(j));
  const double g = mu / double(s);
  for (auto& x : Vw.a) x = x * g;
  Mat S = Vw, D = Vw, Vn(n, p + 1);
  int k = 1;
  double sigma = 1.0;
  double c1 = std::numeric_limits<double>::infinity();
  double c2 = inf_norm(D);
  const double tos = t / double(s);
  while (c1 + c2 > tol * inf_norm(S)) {
    if (k >= kSeriesCap) no_convergence("phimv", "series", kSeriesCap);
    ++k;
    c1 = c2;
    sigma *= k;
    for (int j = 0; j <= p; ++j)
      for (long q = 0; q < n; ++q) {
        double acc = 0.0;
        if (j >= 2) acc = acc + Vw(q, j - 1) * ja;
        acc = acc + Vw(q, j) * jd;
        Vn(q, j) = acc;
      }
    std::swap(Vw, Vn);
    Mat Y = shifted_apply(op, xi, D);
    for (size_t q = 0; q < D.a.size(); ++q) D.a[q] = tos * Y.a[q] + Vw.a[q];
    rec.matvecs += p + 1;
    c2 = inf_norm(D) / sigma;
    if (!std::isfinite(c2)) diverged("phimv", "series", k);
    for (size_t q = 0; q < S.a.size(); ++q) S.a[q] = S.a[q] + D.a[q] / sigma;
  }
  rec.series_len_S = k;
  const int ncols = p == 0 ? 1 : 2;
  Mat F(n, ncols);
  std::copy(S.col(0), S.col(0) + n, F.col(0));
  if (p > 0) std::copy(S.col(p), S.col(p) + n, F.col(1));
  {
    Mat F0(n, 1);
    std::copy(F.col(0), F.col(0) + n, F0.col(0));
    Mat AF = apply(op, F0);
    for (long q = 0; q < n; ++q) F(q, 0) = t * AF.a[size_t(q)] + V(q, 0);
    rec.matvecs += 1;
  }
  Mat& Sadv = S;
  for (long sweep = 1; sweep < s; ++sweep) {
    Mat E = F;
    int kk = 0;
    double d1 = std::numeric_limits<double>::infinity();
    double d2 = inf_norm(F);
    while (d1 + d2 > tol * inf_norm(E)) {
      if (kk >= kRecoveryCap) no_convergence("phimv", "recovery sweep", kRecoveryCap);
      ++kk;
      d1 = d2;
      const double fac = t / (double(s) * kk);
      Mat Y = shifted_apply(op, xi, F);
      for (size_t q = 0; q < F.a.size(); ++q) F.a[q] = fac * Y.a[q];
      rec.matvecs += ncols;
      d2 = inf_norm(F);
      if (!std::isfinite(d2)) diverged("phimv", "recovery sweep", kk);
      for (size_t q = 0; q < E.a.size(); ++q) E.a[q] = E.a[q] + F.a[q];
    }
    rec.series_lens_F.push_back(kk);
    for (auto& x : E.a) x = x * mu;
    for (int j = p; j >= 1; --j)
      for (long q = 0; q < n; ++q) {
        double acc = 0.0;
        for (int l = 1; l <= j; ++l) acc = acc + Sadv(q, l) * jc[size_t(j - l)];
        Sadv(q, j) = acc;
      }
    if (p > 0)
      for (long q = 0; q < n; ++q) F(q, 1) = E(q, 1) + Sadv(q, p);
    for (long q = 0; q < n; ++q) F(q, 0) = E(q, 0);
  }
  SingleResult out;
  out.exp_v0.assign(F.col(0), F.col(0) + n);
  out.tail = p > 0 ? Vec(F.col(1), F.col(1) + n) : Vec(size_t(n), 0.0);
  out.w.resize(size_t(n));
  for (long q = 0; q < n; ++q) out.w[size_t(q)] = out.exp_v0[size_t(q)] + alpha * out.tail[size_t(q)];
  out.rec = std::move(rec);
  return out;
}

// ---------------------------------------------------------------------------
// High-precision references (oracle.cpp:15-116), long double, dense.
// ---------------------------------------------------------------------------
using LD = long double;
struct LMat {
  long n = 0;
  std::vector<LD> a;  // column-major n x n
  explicit LMat(long n_ = 0) : n(n_), a(size_t(n_) * size_t(n_), 0.0L) {}
  LD& operator()(long i, long j) { return a[size_t(i) + size_t(j) * size_t(n)]; }
  LD operator()(long i, long j) const { return a[size_t(i) + size_t(j) * size_t(n)]; }
};

// C = A B; output columns are split across host threads (each column is
// computed by one thread in a fixed order, so the result is thread-count
// independent).
static LMat lmul(const LMat& A, const LMat& B) {
  const long n = A.n;
  LMat C(n);
  auto cols = [&](long j0, long j1) {
    for (long j = j0; j < j1; ++j)
      for (long k = 0; k < n; ++k) {
        const LD b = B(k, j);
        if (b == 0.0L) continue;
        const LD* ak = &A.a[size_t(k) * size_t(n)];
        LD* cj = &C.a[size_t(j) * size_t(n)];
        for (long i = 0; i < n; ++i) cj[i] += ak[i] * b;
      }
  };
  const long nt = n >= 128 ? std::max(1u, std::thread::hardware_concurrency()) : 1;
  if (nt <= 1) {
    cols(0, n);
    return C;
  }
  std::vector<std::thread> ts;
  for (long q = 0; q < nt; ++q) ts.emplace_back(cols, n * q / nt, n * (q + 1) / nt);
  for (auto& t : ts) t.join();
  return C;
}

// expm_core (oracle.cpp:15-34): Taylor-30 on A/2^sigma with compensated
// summation, then sigma squarings.
static LMat expm_core(const LMat& A) {
  const long d = A.n;
  LD norm1 = 0.0L;
  for (long j = 0; j < d; ++j) {
    LD cs = 0.0L;
    for (long i = 0; i < d; ++i) cs += std::fabs(A(i, j));
    norm1 = std::max(norm1, cs);
  }
  int sg = 0;
  if (norm1 > 0.25L) sg = int(std::ceil(std::log2(double(norm1 / 0.25L))));
  LMat X(d);
  const LD div = std::exp2l(LD(sg));
  for (size_t q = 0; q < X.a.size(); ++q) X.a[q] = A.a[q] / div;
  LMat sum(d), comp(d), term(d);
  for (long i = 0; i < d; ++i) sum(i, i) = term(i, i) = 1.0L;
  for (int k = 1; k <= 30; ++k) {
    term = lmul(term, X);
    for (auto& x : term.a) x /= LD(k);
    for (size_t q = 0; q < sum.a.size(); ++q) {
      const LD y = term.a[q] - comp.a[q];
      const LD tt = sum.a[q] + y;
      comp.a[q] = (tt - sum.a[q]) - y;
      sum.a[q] = tt;
    }
  }
  for (int q = 0; q < sg; ++q) sum = lmul(sum, sum);
  return sum;
}

// reference_w (oracle.cpp:53-91)
static Vec reference_w(const Mat& A, const Mat& V, double t, double alpha) {
  const long n = A.rows;
  if (A.rows != A.cols) throw std::invalid_argument("reference_w: A must be square");
  if (V.rows != n) throw std::invalid_argument("reference_w: V row count mismatch");
  const int p = int(V.cols) - 1;
  if (p < 0) throw std::invalid_argument("reference_w: V is empty");
  if (n + p > 2000) throw std::invalid_argument("reference_w: augmented dimension above 2000");
  Vec w(static_cast<size_t>(n));
  if (p == 0) {
    LMat B(n);
    for (long j = 0; j < n; ++j)
      for (long i = 0; i < n; ++i) B(i, j) = LD(t * A(i, j));
    const LMat E = expm_core(B);
    for (long i = 0; i < n; ++i) {
      LD acc = 0.0L;
      for (long j = 0; j < n; ++j) acc += E(i, j) * LD(V(j, 0));
      w[size_t(i)] = double(acc);
    }
  } else {
    const long d = n + p;
    LMat B(d);
    for (long j = 0; j < n; ++j)
      for (long i = 0; i < n; ++i) B(i, j) = LD(t * A(i, j));
    double apow = alpha;
    for (int j = 1; j <= p; ++j) {
      for (long i = 0; i < n; ++i) B(i, n + p - j) = LD(apow * V(i, j));
      apow *= alpha;
    }
    for (int i = 0; i < p - 1; ++i) B(n + i, n + i + 1) = 1.0L;
    std::vector<LD> tail(static_cast<size_t>(d), 0.0L);
    for (long i = 0; i < n; ++i) tail[size_t(i)] = LD(V(i, 0));
    tail[size_t(d - 1)] = 1.0L;
    const LMat E = expm_core(B);
    for (long i = 0; i < n; ++i) {
      LD acc = 0.0L;
      for (long j = 0; j < d; ++j) acc += E(i, j) * tail[size_t(j)];
      w[size_t(i)] = double(acc);
    }
  }
  if (!all_finite(w.data(), w.size())) throw std::runtime_error("reference_w: exponential overflowed");
  return w;
}

// dense_phi (oracle.cpp:93-116): phi_0..phi_jmax of t*M from one
// exponential of the block-bidiagonal embedding.
static std::vector<Mat> dense_phi(const Mat& M, double t, int jmax) {
  const long d = M.rows;
  if (M.rows != M.cols) throw std::invalid_argument("dense_phi: matrix must be square");
  if (d > 50) throw std::invalid_argument("dense_phi: dimension above 50");
  if (jmax < 0) throw std::invalid_argument("dense_phi: jmax must be >= 0");
  const long dim = d * (jmax + 1);
  LMat K(dim);
  for (long j = 0; j < d; ++j)
    for (long i = 0; i < d; ++i) K(i, j) = LD(t * M(i, j));
  for (int b = 0; b + 1 <= jmax; ++b)
    for (long i = 0; i < d; ++i) K(b * d + i, (b + 1) * d + i) = 1.0L;
  const LMat E = expm_core(K);
  std::vector<Mat> phis;
  for (int k = 0; k <= jmax; ++k) {
    Mat P(d, d);
    for (long j = 0; j < d; ++j)
      for (long i = 0; i < d; ++i) P(i, j) = double(E(i, k * d + j));
    if (!all_finite(P.a.data(), P.a.size())) throw std::runtime_error("dense_phi: exponential overflowed");
    phis.push_back(std::move(P));
  }
  return phis;
}

}  // namespace orc

// ============================================================================
// C ABI for the test harness (ctypes).  Errors: return value 0 = ok,
// 1 = std::invalid_argument, 2 = std::runtime_error, 3 = std::logic_error,
// 9 = other; message via orc_last_error().
// ============================================================================
namespace orc {

// ---------------------------------------------------------------------------
// block_series_direct (phi_block.cpp:158-212): the
// direct power series G = sum_j A^j V D_j Gamma T^j, a cross-check of the
// scaled evaluator.  Canonical orders (the reference delegates them to
// Eigen): term(:,k) = sum_{i=0..p} X(:,i) * M(i,k) accumulated from +0 in
// ascending i (M = diag(d_j) Gamma formed first), then * tpow_k, then
// G += term; inf-norms as everywhere else.
// phi_series_coeffs (:158-169): a_ij = 1/(i+j)! on the chain f_k = f_{k-1}/k.
static std::vector<double> phi_inv_factorials(int upto) {
  std::vector<double> t{1.0};
  while (int(t.size()) <= upto) t.push_back(t.back() / double(t.size()));
  return t;
}

// coeff(i, j): the series coefficients; nullptr = phi_series_coeffs
static Mat block_series_direct(const Op& op, const Vec& t, const Vec& alpha, const Mat& V,
                               double req_tol,
                               const std::function<double(int, int)>* coeff = nullptr) {
  // check_request (phi_block.cpp:15-27)
  if (t.empty()) throw std::invalid_argument("phimv_block: at least one abscissa required");
  if (alpha.size() != t.size()) throw std::invalid_argument("phimv_block: t and alpha lengths differ");
  if (V.cols < 1) throw std::invalid_argument("phimv_block: V must have at least one column");
  if (V.rows != op.n) throw std::invalid_argument("phimv_block: V row count does not match operator");
  if (!all_finite(t.data(), t.size()) || !all_finite(alpha.data(), alpha.size()) ||
      !all_finite(V.a.data(), V.a.size()))
    throw std::invalid_argument("phimv_block: inputs must be finite");
  const double tol = req_tol > 0.0 ? req_tol : default_tolerance();
  const long r = long(t.size());
  const int p = int(V.cols) - 1;
  const long n = op.n;
  std::vector<double> inv_fact = phi_inv_factorials(p);
  auto a = [&](int i, int j) -> double {
    if (coeff) return (*coeff)(i, j);
    while (int(inv_fact.size()) <= i + j) inv_fact.push_back(inv_fact.back() / double(inv_fact.size()));
    return inv_fact[size_t(i + j)];
  };
  Mat gamma(p + 1, r);  // Gamma = [alpha_k^i]
  for (long k = 0; k < r; ++k) {
    double power = 1.0;
    for (int i = 0; i <= p; ++i) {
      gamma(i, k) = power;
      power *= alpha[size_t(k)];
    }
  }
  Mat X = V;
  Vec tpow(static_cast<size_t>(r), 1.0);
  Mat G(n, r);
  Mat term(n, r);
  double c1 = std::numeric_limits<double>::infinity(), c2 = 0.0;
  for (int j = 0;; ++j) {
    if (j >= kSeriesCap)
      throw std::runtime_error("phimv_block: direct series did not converge within " +
                               std::to_string(kSeriesCap) + " terms");
    if (j > 0) {
      X = apply(op, X);
      for (long k = 0; k < r; ++k) tpow[size_t(k)] = tpow[size_t(k)] * t[size_t(k)];
    }
    Mat M(p + 1, r);
    for (long k = 0; k < r; ++k)
      for (int i = 0; i <= p; ++i) M(i, k) = a(i, j) * gamma(i, k);
    for (long k = 0; k < r; ++k)
      for (long q = 0; q < n; ++q) {
        double acc = 0.0;
        for (int i = 0; i <= p; ++i) acc = acc + X(q, i) * M(i, k);
        acc = acc * tpow[size_t(k)];
        term(q, k) = acc;
        G(q, k) = G(q, k) + acc;
      }
    c1 = c2;
    c2 = inf_norm(term);
    if (!std::isfinite(c2))
      throw std::runtime_error("phimv_block: direct series produced a non-finite term at index " +
                               std::to_string(j));
    if (j >= 1 && c1 + c2 <= tol * inf_norm(G)) break;
  }
  return G;
}

// ---------------------------------------------------------------------------
// The evaluator's consumer
// ---------------------------------------------------------------------------

// ADRProblem::reaction (problems.cpp:180-182): gamma * u * (u - 1/2) * (1 - u),
// left-associative like the Eigen array expression.
static double adr_reaction(double gamma, double u) { return gamma * u * (u - 0.5) * (1.0 - u); }

// adr_build's matrix-free apply (problems.cpp:184-231), restated verbatim:
// mirror ghosts at x = 0 / y = 0, eliminated Dirichlet edges at x = 1 / y = 1.
static void adr_apply_stencil(int nx, int ny, double eps, double alpha_adv, const double* u,
                              double* y) {
  const double hx = 1.0 / nx, hy = 1.0 / ny;
  const double dxx = eps / (hx * hx), dyy = eps / (hy * hy);
  const double ax = alpha_adv / (2.0 * hx), ay = alpha_adv / (2.0 * hy);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const long idx = long(j) * nx + i;
      const double uc = u[idx];
      const double uw = i > 0 ? u[idx - 1] : u[idx + 1];
      const double ue = i < nx - 1 ? u[idx + 1] : 0.0;
      const double us = j > 0 ? u[idx - nx] : u[idx + nx];
      const double un = j < ny - 1 ? u[idx + nx] : 0.0;
      const double lap = dxx * (uw - 2.0 * uc + ue) + dyy * (us - 2.0 * uc + un);
      const double adv = ax * (ue - uw) + ay * (un - us);
      y[idx] = lap - adv;
    }
}

// adr_build's initial condition (problems.cpp:239-246)
static void adr_u0(int nx, int ny, double* u0) {
  const double hx = 1.0 / nx, hy = 1.0 / ny;
  for (int j = 0; j < ny; ++j) {
    const double y = j * hy;
    for (int i = 0; i < nx; ++i) {
      const double x = i * hx;
      u0[long(j) * nx + i] = 256.0 * x * x * y * y * (1.0 - x) * (1.0 - x) * (1.0 - y) * (1.0 - y);
    }
  }
}

// ExpRK4s6Coefficients (integrator.hpp:13-19)
constexpr double kC2 = 0.5, kC3 = 0.5, kC4 = 1.0 / 3.0, kC5 = 5.0 / 6.0, kC6 = 1.0 / 3.0;

// exprk4s6_step (integrator.cpp:29-105) on a CSR operator with reaction gamma
static Vec exprk4s6_step(const Op& op, double gamma, const Vec& u, double h, double tol,
                         const ScalingShift& params, RunRecord* recs) {
  const long n = long(u.size());
  Vec g_n(static_cast<size_t>(n)), hf(static_cast<size_t>(n));
  {
    Mat U(n, 1);
    std::copy(u.begin(), u.end(), U.col(0));
    const Mat AU = apply(op, U);
    for (long i = 0; i < n; ++i) {
      g_n[size_t(i)] = adr_reaction(gamma, u[size_t(i)]);
      const double f = AU(i, 0) + g_n[size_t(i)];  // op.apply(u) + g_n
      hf[size_t(i)] = h * f;
    }
  }
  auto stage_call = [&](const Vec& t, const Vec& alpha, const Mat& V, RunRecord* rec) {
    Trace trc;
    BlockResult res = phimv_block(op, t, alpha, V, tol, params, trc);
    if (rec) *rec = res.rec;
    return res.W;
  };
  auto react_diff = [&](const double* W) {
    Vec d(static_cast<size_t>(n));
    for (long i = 0; i < n; ++i)
      d[size_t(i)] = adr_reaction(gamma, u[size_t(i)] + W[i]) - g_n[size_t(i)];
    return d;
  };
  // stage 2 alone
  Mat V2(n, 2);
  for (long i = 0; i < n; ++i) V2(i, 1) = kC2 * hf[size_t(i)];
  const Mat U2 = stage_call({kC2 * h}, {1.0}, V2, recs ? recs + 0 : nullptr);
  const Vec d2 = react_diff(U2.col(0));
  // stages 3 and 4, alpha_i = c_i
  Mat V34(n, 3);
  const double s34 = h / kC2;
  for (long i = 0; i < n; ++i) {
    V34(i, 1) = hf[size_t(i)];
    V34(i, 2) = s34 * d2[size_t(i)];
  }
  const Mat U34 = stage_call({kC3 * h, kC4 * h}, {kC3, kC4}, V34, recs ? recs + 1 : nullptr);
  const Vec d3 = react_diff(U34.col(0)), d4 = react_diff(U34.col(1));
  // stages 5 and 6
  const double c34 = kC3 - kC4;
  Mat V56(n, 4);
  {
    const double A = h / c34, B = -(kC4 / kC3), C = kC3 / kC4, D = 2.0 * h / c34;
    for (long i = 0; i < n; ++i) {
      V56(i, 1) = hf[size_t(i)];
      V56(i, 2) = A * (B * d3[size_t(i)] + C * d4[size_t(i)]);
      V56(i, 3) = D * (d3[size_t(i)] / kC3 - d4[size_t(i)] / kC4);
    }
  }
  const Mat U56 = stage_call({kC5 * h, kC6 * h}, {kC5, kC6}, V56, recs ? recs + 2 : nullptr);
  const Vec d5 = react_diff(U56.col(0)), d6 = react_diff(U56.col(1));
  // the update, alpha = 1
  const double c56 = kC5 - kC6;
  Mat Vn(n, 4);
  {
    const double A = h / c56, B = -(kC6 / kC5), C = kC5 / kC6, D = 2.0 * h / c56;
    for (long i = 0; i < n; ++i) {
      Vn(i, 1) = hf[size_t(i)];
      Vn(i, 2) = A * (B * d5[size_t(i)] + C * d6[size_t(i)]);
      Vn(i, 3) = D * (d5[size_t(i)] / kC5 - d6[size_t(i)] / kC6);
    }
  }
  const Mat Un = stage_call({h}, {1.0}, Vn, recs ? recs + 3 : nullptr);
  Vec out(static_cast<size_t>(n));
  for (long i = 0; i < n; ++i) out[size_t(i)] = u[size_t(i)] + Un(i, 0);
  return out;
}

// read_matrix_market (matrix_market.cpp:37-100), restated: the reference's
// dense reader, for pinning the product's CSR reader.
// Lines come from getline(3) instead of std::getline, and `stream >> x` is
// restated as libstdc++'s classic-locale num_get: collect the decimal
// grammar ([sign] digits [. digits] [(e|E) [sign] digits] for double,
// [sign] digits for long), convert with strtod / strtol, fail when the
// conversion stops early or overflows.  (No iostreams: the oracle is loaded
// into processes with another libstdc++.)
static std::string mm_lower(std::string s) {
  for (char& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
  return s;
}
[[noreturn]] static void mm_fail(const std::string& path, const std::string& what) {
  throw std::runtime_error("matrix market: " + path + ": " + what);
}
struct MmIn {
  FILE* f = nullptr;
  ~MmIn() {
    if (f) std::fclose(f);
  }
  bool getline(std::string& line) {  // std::getline: up to '\n', '\n' dropped
    line.clear();
    int c;
    bool any = false;
    while ((c = std::fgetc(f)) != EOF) {
      any = true;
      if (c == '\n') return true;
      line.push_back(char(c));
    }
    return any;
  }
};
static bool mm_next_data_line(MmIn& in, std::string& line) {
  while (in.getline(line)) {
    while (!line.empty() && (line.back() == '\r' || line.back() == '\n')) line.pop_back();
    if (line.empty() || line[0] == '%') continue;
    if (line.find_first_not_of(" \t") == std::string::npos) continue;
    return true;
  }
  return false;
}
struct MmStream {  // istringstream >> long / double / string, classic locale
  const std::string& s;
  size_t i = 0;
  bool ok = true;
  explicit MmStream(const std::string& str) : s(str) {}
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  MmStream& operator>>(std::string& w) {
    w.clear();
    if (!ok) return *this;
    ws();
    while (i < s.size() && !std::isspace(static_cast<unsigned char>(s[i]))) w.push_back(s[i++]);
    if (w.empty()) ok = false;
    return *this;
  }
  MmStream& operator>>(long& v) {
    if (!ok) return *this;
    ws();
    const size_t b = i;
    if (i < s.size() && (s[i] == '+' || s[i] == '-')) ++i;
    while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) ++i;
    const std::string tok = s.substr(b, i - b);
    char* end = nullptr;
    errno = 0;
    v = std::strtol(tok.c_str(), &end, 10);
    if (tok.empty() || *end != '\0' || errno == ERANGE) ok = false;
    return *this;
  }
  MmStream& operator>>(double& v) {
    if (!ok) return *this;
    ws();
    const size_t b = i;
    bool mant = false;
    if (i < s.size() && (s[i] == '+' || s[i] == '-')) ++i;
    while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) ++i, mant = true;
    if (i < s.size() && s[i] == '.') {
      ++i;
      while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) ++i, mant = true;
    }
    if (mant && i < s.size() && (s[i] == 'e' || s[i] == 'E')) {
      ++i;
      if (i < s.size() && (s[i] == '+' || s[i] == '-')) ++i;
      while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) ++i;
    }
    const std::string tok = s.substr(b, i - b);
    char* end = nullptr;
    v = std::strtod(tok.c_str(), &end);
    if (tok.empty() || *end != '\0' || std::isinf(v)) ok = false;
    return *this;
  }
  explicit operator bool() const { return ok; }
};
static Mat read_matrix_market(const std::string& path) {
  MmIn in;
  in.f = std::fopen(path.c_str(), "rb");
  if (!in.f) mm_fail(path, "cannot open file");
  std::string header;
  if (!in.getline(header)) mm_fail(path, "empty file");
  while (!header.empty() && (header.back() == '\r' || header.back() == '\n')) header.pop_back();
  MmStream hs(header);
  std::string banner, object, format, field, symmetry;
  hs >> banner >> object >> format >> field >> symmetry;
  if (mm_lower(banner) != "%%matrixmarket" || mm_lower(object) != "matrix")
    mm_fail(path, "malformed header line");
  format = mm_lower(format);
  field = mm_lower(field);
  symmetry = mm_lower(symmetry);
  if (format != "array" && format != "coordinate") mm_fail(path, "unsupported format '" + format + "'");
  if (field != "real" && field != "integer") mm_fail(path, "non-real field '" + field + "'");
  if (symmetry != "general" && symmetry != "symmetric")
    mm_fail(path, "unsupported symmetry '" + symmetry + "'");
  const bool symmetric = symmetry == "symmetric";
  std::string line;
  if (!mm_next_data_line(in, line)) mm_fail(path, "missing size line");
  MmStream ss(line);
  long rows = 0, cols = 0, nnz = 0;
  if (!(ss >> rows >> cols)) mm_fail(path, "malformed size line");
  if (format == "coordinate" && !(ss >> nnz)) mm_fail(path, "missing entry count");
  if (rows <= 0 || cols <= 0) mm_fail(path, "non-positive dimensions");
  if (rows != cols)
    mm_fail(path, "matrix is " + std::to_string(rows) + "x" + std::to_string(cols) + ", expected square");
  Mat A(rows, cols);
  if (format == "array") {
    for (long j = 0; j < cols; ++j)
      for (long i = symmetric ? j : 0; i < rows; ++i) {
        if (!mm_next_data_line(in, line)) mm_fail(path, "truncated array data");
        MmStream es(line);
        double value = 0.0;
        if (!(es >> value)) mm_fail(path, "malformed entry");
        A(i, j) = value;
        if (symmetric) A(j, i) = value;
      }
  } else {
    for (long k = 0; k < nnz; ++k) {
      if (!mm_next_data_line(in, line)) mm_fail(path, "truncated coordinate data");
      MmStream es(line);
      long i = 0, j = 0;
      double value = 0.0;
      if (!(es >> i >> j >> value)) mm_fail(path, "malformed entry");
      if (i < 1 || i > rows || j < 1 || j > cols) mm_fail(path, "entry index out of range");
      A(i - 1, j - 1) += value;
      if (symmetric && i != j) A(j - 1, i - 1) += value;
    }
  }
  if (!all_finite(A.a.data(), A.a.size())) mm_fail(path, "non-finite entries");
  return A;
}

struct IntegrateResult {
  Vec u;
  double t = 0.0;
  std::vector<RunRecord> recs;  // 4 per step
};

// integrate (integrator.cpp:107-134)
static IntegrateResult integrate(const Op& op, double gamma, const Vec& u0, double h, double t_end,
                                 double tol, const ScalingShift& params, bool keep_records) {
  if (!(h > 0.0)) throw std::invalid_argument("integrate: h must be positive");
  const double span = t_end;
  const long n_steps = std::lround(span / h);
  if (n_steps < 1 || n_steps > 1000000)
    throw std::invalid_argument("integrate: step count out of range");
  if (std::abs(n_steps * h - span) > 1e-9 * std::max(1.0, span))
    throw std::invalid_argument("integrate: t_end is not a multiple of h");
  IntegrateResult out;
  out.u = u0;
  out.t = 0.0;
  for (long step = 0; step < n_steps; ++step) {
    RunRecord rec[4];
    Vec next = exprk4s6_step(op, gamma, out.u, h, tol, params, keep_records ? rec : nullptr);
    if (!all_finite(next.data(), next.size()))
      throw std::runtime_error("integrate: state left the finite range at t = " +
                               std::to_string(out.t));
    out.u = std::move(next);
    out.t = (step + 1) * h;
    if (keep_records)
      for (auto& r : rec) out.recs.push_back(r);
  }
  return out;
}

}  // namespace orc

namespace {
thread_local std::string g_err;
template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}
orc::Op make_op(int64_t n, const int64_t* rp, const int32_t* ci, const double* v) {
  orc::Op op;
  op.n = n;
  op.rp = rp;
  op.ci = ci;
  op.v = v;
  return op;
}
orc::Mat wrap(const double* X, int64_t rows, int64_t cols, int64_t ld) {
  orc::Mat M(rows, cols);
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i) M(i, j) = X[i + j * ld];
  return M;
}
void fill_rec(const orc::RunRecord& rec, int64_t* rec4, int32_t* lens, int64_t cap) {
  if (rec4) {
    rec4[0] = rec.s_effective;
    rec4[1] = rec.series_len_S;
    rec4[2] = int64_t(rec.series_lens_F.size());
    rec4[3] = rec.matvecs;
  }
  if (lens)
    for (size_t q = 0; q < rec.series_lens_F.size() && int64_t(q) < cap; ++q)
      lens[q] = rec.series_lens_F[q];
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_rng_matrix(uint64_t seed, int64_t rows, int64_t cols, double* out) {
  return guarded([&] {
    orc::Rng rng(seed);
    orc::Mat M = rng.matrix(rows, cols);
    std::memcpy(out, M.a.data(), M.a.size() * sizeof(double));
  });
}

// generic stream access: kinds 0 = uniform, 1 = normal, 2 = matrix-then-
// uniform draws (one Rng threaded through `count` draws of mixed kinds)
int orc_rng_draws(uint64_t seed, int64_t count, const int32_t* kinds, double* out) {
  return guarded([&] {
    orc::Rng rng(seed);
    for (int64_t q = 0; q < count; ++q) out[q] = kinds[q] == 0 ? rng.uniform() : rng.normal();
  });
}

int orc_unit_vector(uint64_t seed, int64_t n, double* out) {
  return guarded([&] {
    orc::Rng rng(seed);
    orc::Vec v = rng.unit_vector(n);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}

// stateful stream (one Rng threaded through a test's draws, like the
// reference tests' `Rng rng(seed); A = rng.matrix(..); V = rng.matrix(..)`)
void* orc_rng_new(uint64_t seed) { return new orc::Rng(seed); }
void orc_rng_free(void* h) { delete static_cast<orc::Rng*>(h); }
void orc_rng_normals(void* h, int64_t count, double* out) {
  auto* g = static_cast<orc::Rng*>(h);
  for (int64_t q = 0; q < count; ++q) out[q] = g->normal();
}
void orc_rng_uniforms(void* h, int64_t count, double* out) {
  auto* g = static_cast<orc::Rng*>(h);
  for (int64_t q = 0; q < count; ++q) out[q] = g->uniform();
}

double orc_stable_norm(const double* x, int64_t n) { return orc::stable_norm(x, n); }
double orc_norm2(const double* x, int64_t n) { return orc::norm2(x, n); }
double orc_inf_norm(const double* X, int64_t rows, int64_t cols, int64_t ld) {
  return orc::inf_norm(X, rows, cols, ld);
}

int orc_apply(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, const double* X,
              int64_t k, double* Y) {
  return guarded([&] { orc::apply_into(make_op(n, rp, ci, v), X, n, k, Y, n); });
}

// shifted_apply (linop.cpp:40-49)
int orc_shifted_apply(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, double xi,
                      const double* X, int64_t k, double* Y) {
  return guarded([&] {
    orc::Mat Xm = wrap(X, n, k, n);
    orc::Mat Ym = orc::shifted_apply(make_op(n, rp, ci, v), xi, Xm);
    std::copy(Ym.a.begin(), Ym.a.end(), Y);
  });
}

// --- power basis handle (params.hpp:22-29, 50-71) ---
void* orc_basis_build(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, int32_t m,
                      double delta, int32_t* err) {
  orc::PowerBasis* out = nullptr;
  *err = guarded([&] { out = new orc::PowerBasis(orc::build_power_basis(make_op(n, rp, ci, v), m, delta)); });
  return out;
}
void orc_basis_free(void* h) { delete static_cast<orc::PowerBasis*>(h); }
int orc_basis_info(void* h, int32_t* r, int32_t* m, double* s0, double* logs, double* columns,
                   double* log_binom) {
  const auto* b = static_cast<const orc::PowerBasis*>(h);
  *r = b->r;
  *m = b->m;
  *s0 = b->s0;
  if (logs) std::copy(b->logs.begin(), b->logs.end(), logs);
  if (columns) std::copy(b->columns.a.begin(), b->columns.a.end(), columns);
  if (log_binom) std::copy(b->log_binom.begin(), b->log_binom.end(), log_binom);
  return 0;
}
int orc_objective(void* h, double xi, double* f) {
  return guarded([&] { *f = orc::objective(*static_cast<const orc::PowerBasis*>(h), xi); });
}
int orc_minimize_shift(void* h, double* xi, double* fmin, double* path, int64_t path_cap,
                       int64_t* path_len) {
  return guarded([&] {
    std::vector<double> pth;
    auto res = orc::minimize_shift(*static_cast<const orc::PowerBasis*>(h), path ? &pth : nullptr);
    *xi = res.first;
    *fmin = res.second;
    if (path) {
      *path_len = int64_t(pth.size());
      for (int64_t q = 0; q < int64_t(pth.size()) && q < path_cap; ++q) path[q] = pth[size_t(q)];
    }
  });
}
int orc_parameters_for_shift(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                             void* h, double xi, double tol, orc_scaling_shift* out) {
  return guarded([&] {
    *out = orc::parameters_for_shift(make_op(n, rp, ci, v), *static_cast<const orc::PowerBasis*>(h), xi,
                                     tol);
  });
}
int orc_log_shifted_power(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                          const double* x, double xi, int32_t m, double* out) {
  return guarded([&] { *out = orc::log_shifted_power(make_op(n, rp, ci, v), x, xi, m); });
}
int orc_select_parameters(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, int32_t m,
                          double tol, double delta, orc_scaling_shift* out) {
  return guarded([&] { *out = orc::select_parameters(make_op(n, rp, ci, v), m, tol, delta); });
}

// --- evaluators ---
int orc_phimv_block(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, int64_t r,
                    const double* t, const double* alpha, int32_t p, const double* V, int64_t ldv,
                    double tol, const orc_scaling_shift* params, double* W, int64_t ldw,
                    int64_t* rec4, int32_t* lens_F, int64_t lens_cap, double* trace,
                    int64_t trace_cap, int64_t* trace_len) {
  return guarded([&] {
    orc::Vec tv(t, t + r), av(alpha, alpha + r);
    orc::Mat Vm = wrap(V, n, p + 1, ldv);
    std::vector<double> tr;
    orc::Trace trc;
    trc.out = trace ? &tr : nullptr;
    orc::BlockResult res = orc::phimv_block(make_op(n, rp, ci, v), tv, av, Vm, tol, *params, trc);
    for (int64_t i = 0; i < r; ++i)
      for (int64_t q = 0; q < n; ++q) W[q + i * ldw] = res.W(q, i);
    fill_rec(res.rec, rec4, lens_F, lens_cap);
    if (trace) {
      *trace_len = int64_t(tr.size());
      for (int64_t q = 0; q < int64_t(tr.size()) && q < trace_cap; ++q) trace[q] = tr[size_t(q)];
    }
  });
}

// Timing sample for the CPU arms of bench.py: the same evaluation with its
// phases timed (phases7[9]: setup, S terms, S terms run, promotion, sweeps,
// sweeps run, assembly, first S term, first sweep), optionally stopped after max_s_terms S terms and
// max_sweeps recovery sweeps (0: all).  rec4 as in orc_phimv_block;
// term_times (optional, >= the S terms run): each S term's wall time.
int orc_phimv_block_timed(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                          int64_t r, const double* t, const double* alpha, int32_t p,
                          const double* V, int64_t ldv, double tol,
                          const orc_scaling_shift* params, int32_t max_s_terms,
                          int32_t max_sweeps, double* phases7, int64_t* rec4,
                          double* term_times) {
  return guarded([&] {
    orc::Vec tv(t, t + r), av(alpha, alpha + r);
    orc::Mat Vm = wrap(V, n, p + 1, ldv);
    orc::Trace trc;
    for (int q = 0; q < 9; ++q) phases7[q] = 0.0;
    orc::BlockResult res = orc::phimv_block(make_op(n, rp, ci, v), tv, av, Vm, tol, *params, trc,
                                            max_s_terms, max_sweeps, phases7, term_times);
    fill_rec(res.rec, rec4, nullptr, 0);
  });
}

// threads of the row-parallel loops (bench.py CPU arms); 1 = the reference's
// configuration
void orc_set_threads(int32_t threads) { orc::g_threads = threads < 1 ? 1 : threads; }
// test hook: the row-sum order of inf_norm (0 canonical; see rowsum_abs)
void orc_set_rowsum_order(int32_t order) { orc::g_rowsum_order = order; }

int orc_phimv(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, double t, double alpha,
              int32_t p, const double* V, int64_t ldv, double tol, const orc_scaling_shift* params,
              double* w, double* exp_v0, double* tail, int64_t* rec4, int32_t* lens_F,
              int64_t lens_cap) {
  return guarded([&] {
    orc::Mat Vm = wrap(V, n, p + 1, ldv);
    orc::SingleResult res = orc::phimv(make_op(n, rp, ci, v), t, alpha, Vm, tol, *params);
    std::copy(res.w.begin(), res.w.end(), w);
    if (exp_v0) std::copy(res.exp_v0.begin(), res.exp_v0.end(), exp_v0);
    if (tail) std::copy(res.tail.begin(), res.tail.end(), tail);
    fill_rec(res.rec, rec4, lens_F, lens_cap);
  });
}

int orc_reference_w(int64_t n, const double* A, int32_t p, const double* V, double t, double alpha,
                    double* out) {
  return guarded([&] {
    orc::Mat Am = wrap(A, n, n, n), Vm = wrap(V, n, p + 1, n);
    orc::Vec w = orc::reference_w(Am, Vm, t, alpha);
    std::copy(w.begin(), w.end(), out);
  });
}

int orc_dense_phi(int64_t d, const double* M, double t, int32_t jmax, double* out) {
  return guarded([&] {
    orc::Mat Mm = wrap(M, d, d, d);
    auto phis = orc::dense_phi(Mm, t, jmax);
    for (int k = 0; k <= jmax; ++k)
      std::copy(phis[size_t(k)].a.begin(), phis[size_t(k)].a.end(), out + size_t(k) * size_t(d * d));
  });
}

// --- block_series_direct ---
// coeffs: NULL (phi_series_coeffs) or (p+1) x ncoef column-major a_ij
int orc_block_series_direct(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                            int64_t r, const double* t, const double* alpha, int32_t p,
                            const double* V, int64_t ldv, double tol, const double* coeffs,
                            int64_t ncoef, double* G, int64_t ldg) {
  return guarded([&] {
    orc::Vec tv(t, t + r), av(alpha, alpha + r);
    orc::Mat Vm = wrap(V, n, p + 1, ldv);
    std::function<double(int, int)> cf = [&](int i, int j) -> double {
      if (j >= ncoef) throw std::invalid_argument("block_series_direct: coefficient table exhausted");
      return coeffs[size_t(i) + size_t(j) * size_t(p + 1)];
    };
    orc::Mat Gm = orc::block_series_direct(make_op(n, rp, ci, v), tv, av, Vm, tol,
                                           coeffs ? &cf : nullptr);
    for (int64_t k = 0; k < r; ++k)
      for (int64_t q = 0; q < n; ++q) G[q + k * ldg] = Gm(q, k);
  });
}

// --- Matrix Market: the reference's dense reader ---
// out: n*n column-major (NULL: only *n is set)
int orc_read_matrix_market(const char* path, int64_t* n, double* out, int64_t cap) {
  return guarded([&] {
    orc::Mat A = orc::read_matrix_market(path);
    *n = A.rows;
    if (out && cap >= int64_t(A.a.size())) std::copy(A.a.begin(), A.a.end(), out);
  });
}

// --- the integrator ---
void orc_adr_apply_stencil(int32_t nx, int32_t ny, double eps, double alpha_adv, const double* u,
                           double* y) {
  orc::adr_apply_stencil(nx, ny, eps, alpha_adv, u, y);
}
void orc_adr_u0(int32_t nx, int32_t ny, double* u0) { orc::adr_u0(nx, ny, u0); }

// rec4: 4 int64 per evaluator call (s_eff, L_S, sweeps, matvecs)
int orc_exprk4s6_step(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, double gamma,
                      const double* u, double h, double tol, const orc_scaling_shift* params,
                      double* u_next, int64_t* rec4) {
  return guarded([&] {
    orc::Vec uu(u, u + n);
    orc::RunRecord recs[4];
    orc::Vec out = orc::exprk4s6_step(make_op(n, rp, ci, v), gamma, uu, h, tol, *params, recs);
    std::copy(out.begin(), out.end(), u_next);
    if (rec4)
      for (int k = 0; k < 4; ++k) fill_rec(recs[k], rec4 + 4 * k, nullptr, 0);
  });
}

int orc_integrate(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, double gamma,
                  const double* u0, double h, double t_end, double tol,
                  const orc_scaling_shift* params, double* u_out, double* t_out, int64_t* rec4,
                  int64_t rec_cap) {
  return guarded([&] {
    orc::Vec uu(u0, u0 + n);
    orc::IntegrateResult res = orc::integrate(make_op(n, rp, ci, v), gamma, uu, h, t_end, tol,
                                              *params, rec4 != nullptr);
    std::copy(res.u.begin(), res.u.end(), u_out);
    if (t_out) *t_out = res.t;
    if (rec4)
      for (size_t k = 0; k < res.recs.size() && int64_t(k) < rec_cap; ++k)
        fill_rec(res.recs[k], rec4 + 4 * k, nullptr, 0);
  });
}

int orc_jexp_chain(double alpha, double s, int32_t p, double* out) {
  auto c = orc::jexp_chain(alpha, s, p);
  std::copy(c.begin(), c.end(), out);
  return 0;
}

}  // extern "C"
