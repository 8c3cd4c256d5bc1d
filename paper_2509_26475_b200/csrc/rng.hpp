// Deterministic random source of the reference (include/phiact/rng.hpp:15-62):
// mt19937_64 + Box-Muller with a spare, column-major fills.  Used by the
// product for the fixed-seed start vector of the power basis
// (params.cpp:99-115) and by the workload generators.  Host-only: the
// transcendental calls must be glibc's, not the device's, for the streams to
// match the reference bit for bit.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
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
    normals(out, rows * cols, std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
  }

  // n consecutive normal() draws, bit-identical to the sequential calls and
  // leaving the same generator / spare state: the mt19937_64 stream is
  // consumed sequentially (it is cheap), the Box-Muller transcendentals run on
  // host threads.
  void normals(double* out, int64_t n, unsigned threads) {
    int64_t i = 0;
    if (n > 0 && have_spare_) {
      out[i++] = spare_;
      have_spare_ = false;
    }
    const int64_t npairs = (n - i + 1) / 2;
    std::vector<double> u(static_cast<size_t>(2 * npairs));
    for (int64_t k = 0; k < npairs; ++k) {
      double u1 = 0.0;
      do {
        u1 = uniform();
      } while (u1 == 0.0);
      u[size_t(2 * k)] = u1;
      u[size_t(2 * k + 1)] = uniform();
    }
    const int64_t base = i;
    auto work = [&](int64_t k0, int64_t k1) {
      for (int64_t k = k0; k < k1; ++k) {
        const double radius = std::sqrt(-2.0 * std::log(u[size_t(2 * k)]));
        const double angle = 2.0 * M_PI * u[size_t(2 * k + 1)];
        const int64_t o = base + 2 * k;
        out[o] = radius * std::cos(angle);
        if (o + 1 < n) out[o + 1] = radius * std::sin(angle);
      }
    };
    if (threads <= 1 || npairs < 65536) {
      work(0, npairs);
    } else {
      std::vector<std::thread> ts;
      for (unsigned t = 0; t < threads; ++t)
        ts.emplace_back(work, npairs * t / threads, npairs * (t + 1) / threads);
      for (auto& t : ts) t.join();
    }
    if (npairs > 0 && base + 2 * npairs > n) {  // the last pair's sine is the spare
      const int64_t k = npairs - 1;
      spare_ = std::sqrt(-2.0 * std::log(u[size_t(2 * k)])) * std::sin(2.0 * M_PI * u[size_t(2 * k + 1)]);
      have_spare_ = true;
    }
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

// Rng::unit_vector (rng.hpp:53-56): v / v.norm(); the draws, the chunk sums
// of squares and the division run on host threads, bit-identical to the
// sequential definition (chunks are still folded in order)
inline std::vector<double> unit_vector(Rng& rng, int64_t n) {
  const unsigned threads = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<double> v(static_cast<size_t>(n));
  rng.normals(v.data(), n, threads);
  const int64_t nch = (n + 4095) / 4096;
  std::vector<double> part(static_cast<size_t>(nch));
  auto chunks = [&](int64_t c0, int64_t c1) {
    for (int64_t c = c0; c < c1; ++c) {
      const int64_t b = c * 4096;
      part[size_t(c)] = canonical_chunk_sumsq(v.data() + b, n - b < 4096 ? n - b : 4096, 1.0);
    }
  };
  auto divide = [&](double nrm, int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) v[size_t(i)] = v[size_t(i)] / nrm;
  };
  const bool par = threads > 1 && n >= (int64_t(1) << 18);
  if (par) {
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < threads; ++t)
      ts.emplace_back(chunks, nch * t / threads, nch * (t + 1) / threads);
    for (auto& t : ts) t.join();
  } else {
    chunks(0, nch);
  }
  double ssq = 0.0;
  for (int64_t c = 0; c < nch; ++c) ssq = ssq + part[size_t(c)];
  const double nrm = std::sqrt(ssq);
  if (par) {
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < threads; ++t)
      ts.emplace_back(divide, nrm, n * t / threads, n * (t + 1) / threads);
    for (auto& t : ts) t.join();
  } else {
    divide(nrm, 0, n);
  }
  return v;
}

}  // namespace phx
