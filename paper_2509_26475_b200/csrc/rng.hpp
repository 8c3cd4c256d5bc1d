// Deterministic random source of the reference (include/phiact/rng.hpp:15-62):
// mt19937_64 + Box-Muller with a spare, column-major fills.  Used by the
// product for the fixed-seed start vector of the power basis
// (params.cpp:99-115) and by the workload generators.  Host-only: the
// transcendental calls must be glibc's, not the device's, for the streams to
// match the reference bit for bit.
#pragma once
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

namespace phx {

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
  // column-major rows x cols normals (Rng::matrix)
  void matrix(int64_t rows, int64_t cols, double* out) {
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t i = 0; i < rows; ++i) out[i + j * rows] = normal();
  }

 private:
  std::mt19937_64 gen_;
  bool have_spare_ = false;
  double spare_ = 0.0;
};

// Canonical sum of squares: 4096-element chunks, 256 lanes per
// chunk (lane l sums elements l, l+256, ... from +0), lanes combined by a
// pairwise tree; chunks folded sequentially.  Eigen's norm() restated with a
// fixed order.
inline double canonical_chunk_sumsq(const double* x, int64_t len, double mul) {
  double lane[256];
  for (int l = 0; l < 256; ++l) {
    double s = 0.0;
    for (int64_t q = l; q < len; q += 256) {
      const double y = x[q] * mul;
      s = s + y * y;
    }
    lane[l] = s;
  }
  for (int h = 1; h < 256; h *= 2)
    for (int l = 0; l < 256; l += 2 * h) lane[l] = lane[l] + lane[l + h];
  return lane[0];
}

inline double canonical_norm2(const double* x, int64_t n) {
  double ssq = 0.0;
  for (int64_t b = 0; b < n; b += 4096)
    ssq = ssq + canonical_chunk_sumsq(x + b, n - b < 4096 ? n - b : 4096, 1.0);
  return std::sqrt(ssq);
}

// Rng::unit_vector (rng.hpp:53-56): v / v.norm()
inline std::vector<double> unit_vector(Rng& rng, int64_t n) {
  std::vector<double> v(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) v[size_t(i)] = rng.normal();
  const double nrm = canonical_norm2(v.data(), n);
  for (auto& x : v) x = x / nrm;
  return v;
}

}  // namespace phx
