// Seeded synthetic workloads for the five BASELINE.json configurations
// (SURVEY.md §8d and Appendix B).  BASELINE.json leaves several details open;
// the decisions recorded here are fixed for every run:
//
//  C1  1D Dirichlet Laplacian, n = N (default 1000): A = (N+1)^2 tridiag(1,-2,1).
//      p=3, r=6, c = {1/2,1/2,1/3,5/6,1/3,1}, t = 1e-3 c, alpha = c,
//      V = Rng(0).matrix(n, 4) (N(0,1)), tol 1e-12.
//  C2  2D advection-diffusion on an N x N interior grid (default 1024),
//      h = 1/(N+1), eps = 1e-2, velocity (1, 0.5), upwind first differences,
//      Dirichlet neighbours dropped, x-fastest numbering.  Row:
//      diag -4d - vx/h - vy/h, west d + vx/h, south d + vy/h, east/north d,
//      d = eps/h^2.  p=3, r=4, t = 1e-4 {1/4,1/2,3/4,1}, alpha = t/h =
//      {1/4,1/2,3/4,1}, V ~ U[-1,1] from Rng(2), tol 1e-10.
//  C3  3D convection-diffusion on N^3 (default 256), h = 1/(N+1), eps = 1e-2,
//      v = (1,1,1)/sqrt(3) (global Peclet |v| L / eps = 100), upwind,
//      Dirichlet.  Lower neighbours d + v/h, upper d, diag -6d - 3 v/h.
//      p=4, r=6, c as C1, t = 1e-3 c, alpha = c, V = Rng(3) N(0,1),
//      tol 2^-53 (reference default; BASELINE leaves it open).
//  C4  random stiff, n (default 2^22): per row 16 distinct uniform columns
//      != i (Rng(0xC4), rejection), sorted, values N(0,1) in sorted order,
//      diagonal -(sum|off| + U[1,1e4]); p=2, r=3, t = 1e-3 {0.1,0.5,1},
//      alpha = 1, V = Rng(4) N(0,1), tol 2^-53.
//  C5  upper bidiagonal, n (default 2^24): a_ii = -(1 + 999 i/(n-1)),
//      a_{i,i+1} = 50.  p=3, r=8, t_i = 10^(-3 + 4(i-1)/7), alpha_i = i/8,
//      V ~ U[-1,1] from Rng(5), tol 1e-8.
//
// The generators are input setup for tests and bench.py; they are not part
// of the product API (include/phx.h).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "rng.hpp"

extern "C" {

typedef struct {
  int64_t n;
  int64_t nnz;
  int32_t p;
  int32_t r;
  double tol;
  int64_t size;  // the size parameter actually used (N or n)
} phx_wl_info;

}  // extern "C"

namespace {

int64_t default_size(int cfg) {
  switch (cfg) {
    case 1: return 1000;
    case 2: return 1024;
    case 3: return 256;
    case 4: return int64_t(1) << 22;
    case 5: return int64_t(1) << 24;
    default: return 0;
  }
}

bool info(int cfg, int64_t size, phx_wl_info* o) {
  if (size <= 0) size = default_size(cfg);
  o->size = size;
  switch (cfg) {
    case 1:
      if (size < 2) return false;
      o->n = size;
      o->nnz = 3 * size - 2;
      o->p = 3;
      o->r = 6;
      o->tol = 1e-12;
      return true;
    case 2:
      if (size < 2) return false;
      o->n = size * size;
      o->nnz = 5 * size * size - 4 * size;
      o->p = 3;
      o->r = 4;
      o->tol = 1e-10;
      return true;
    case 3:
      if (size < 2) return false;
      o->n = size * size * size;
      o->nnz = 7 * size * size * size - 6 * size * size;
      o->p = 4;
      o->r = 6;
      o->tol = std::ldexp(1.0, -53);
      return true;
    case 4:
      if (size < 32) return false;
      o->n = size;
      o->nnz = 17 * size;
      o->p = 2;
      o->r = 3;
      o->tol = std::ldexp(1.0, -53);
      return true;
    case 5:
      if (size < 2) return false;
      o->n = size;
      o->nnz = 2 * size - 1;
      o->p = 3;
      o->r = 8;
      o->tol = 1e-8;
      return true;
    default:
      return false;
  }
}

const double kC[6] = {1.0 / 2.0, 1.0 / 2.0, 1.0 / 3.0, 5.0 / 6.0, 1.0 / 3.0, 1.0};

void fill_uniform_pm1(uint64_t seed, int64_t n, int cols, double* V) {
  phx::Rng rng(seed);
  for (int j = 0; j < cols; ++j)
    for (int64_t i = 0; i < n; ++i) V[i + int64_t(j) * n] = -1.0 + 2.0 * rng.uniform();
}

void fill_normal(uint64_t seed, int64_t n, int cols, double* V) {
  phx::Rng rng(seed);
  rng.matrix(n, cols, V);
}

}  // namespace

extern "C" {

// The reference Rng streams (for tests of the product's Rng against the
// oracle's): n normals from seed, and Rng(seed).unit_vector(n).
void phx_wl_normals(uint64_t seed, int64_t n, double* out) {
  phx::Rng rng(seed);
  rng.matrix(n, 1, out);
}
void phx_wl_unit_vector(uint64_t seed, int64_t n, double* out) {
  phx::Rng rng(seed);
  const std::vector<double> v = phx::unit_vector(rng, n);
  std::copy(v.begin(), v.end(), out);
}

int phx_wl_info_get(int32_t cfg, int64_t size, phx_wl_info* out) {
  return info(cfg, size, out) ? 0 : 1;
}

// Fills CSR (row_ptr n+1, col_idx/vals nnz), V (n x (p+1) column-major; may be
// NULL), t and alpha (r each; may be NULL).
int phx_wl_fill(int32_t cfg, int64_t size, int64_t* rp, int32_t* ci, double* av, double* V,
                double* t, double* alpha) {
  phx_wl_info o;
  if (!info(cfg, size, &o)) return 1;
  const int64_t n = o.n;
  int64_t e = 0;
  rp[0] = 0;
  if (cfg == 1) {
    const double s2 = double(o.size + 1) * double(o.size + 1);
    for (int64_t i = 0; i < n; ++i) {
      if (i > 0) { ci[e] = int32_t(i - 1); av[e++] = s2 * 1.0; }
      ci[e] = int32_t(i); av[e++] = s2 * -2.0;
      if (i < n - 1) { ci[e] = int32_t(i + 1); av[e++] = s2 * 1.0; }
      rp[i + 1] = e;
    }
    if (V) fill_normal(0, n, o.p + 1, V);
    for (int i = 0; i < o.r; ++i) {
      if (t) t[i] = 1e-3 * kC[i];
      if (alpha) alpha[i] = kC[i];
    }
  } else if (cfg == 2) {
    const int64_t N = o.size;
    const double h = 1.0 / double(N + 1);
    const double eps = 1e-2, vx = 1.0, vy = 0.5;
    const double d = eps / (h * h), ax = vx / h, ay = vy / h;
    const double diag = -4.0 * d - ax - ay, west = d + ax, south = d + ay, east = d, north = d;
    for (int64_t j = 0; j < N; ++j)
      for (int64_t i = 0; i < N; ++i) {
        const int64_t idx = j * N + i;
        if (j > 0) { ci[e] = int32_t(idx - N); av[e++] = south; }
        if (i > 0) { ci[e] = int32_t(idx - 1); av[e++] = west; }
        ci[e] = int32_t(idx); av[e++] = diag;
        if (i < N - 1) { ci[e] = int32_t(idx + 1); av[e++] = east; }
        if (j < N - 1) { ci[e] = int32_t(idx + N); av[e++] = north; }
        rp[idx + 1] = e;
      }
    if (V) fill_uniform_pm1(2, n, o.p + 1, V);
    const double cc[4] = {0.25, 0.5, 0.75, 1.0};
    for (int i = 0; i < 4; ++i) {
      if (t) t[i] = 1e-4 * cc[i];
      if (alpha) alpha[i] = cc[i];
    }
  } else if (cfg == 3) {
    const int64_t N = o.size;
    const double h = 1.0 / double(N + 1);
    const double eps = 1e-2;
    const double v = 1.0 / std::sqrt(3.0);
    const double d = eps / (h * h), a = v / h;
    const double diag = -6.0 * d - a - a - a, lower = d + a, upper = d;
    const int64_t P = N * N;
    for (int64_t k = 0; k < N; ++k)
      for (int64_t j = 0; j < N; ++j)
        for (int64_t i = 0; i < N; ++i) {
          const int64_t idx = k * P + j * N + i;
          if (k > 0) { ci[e] = int32_t(idx - P); av[e++] = lower; }
          if (j > 0) { ci[e] = int32_t(idx - N); av[e++] = lower; }
          if (i > 0) { ci[e] = int32_t(idx - 1); av[e++] = lower; }
          ci[e] = int32_t(idx); av[e++] = diag;
          if (i < N - 1) { ci[e] = int32_t(idx + 1); av[e++] = upper; }
          if (j < N - 1) { ci[e] = int32_t(idx + N); av[e++] = upper; }
          if (k < N - 1) { ci[e] = int32_t(idx + P); av[e++] = upper; }
          rp[idx + 1] = e;
        }
    if (V) fill_normal(3, n, o.p + 1, V);
    for (int i = 0; i < 6; ++i) {
      if (t) t[i] = 1e-3 * kC[i];
      if (alpha) alpha[i] = kC[i];
    }
  } else if (cfg == 4) {
    phx::Rng rng(0xC4);
    int64_t cols[16];
    double vals[16];
    for (int64_t i = 0; i < n; ++i) {
      int cnt = 0;
      while (cnt < 16) {
        const int64_t c = int64_t(rng.uniform() * double(n));
        if (c == i || c >= n) continue;
        bool dup = false;
        for (int q = 0; q < cnt; ++q) dup = dup || cols[q] == c;
        if (dup) continue;
        cols[cnt++] = c;
      }
      std::sort(cols, cols + 16);
      double sabs = 0.0;
      for (int q = 0; q < 16; ++q) {
        vals[q] = rng.normal();
        sabs = sabs + std::fabs(vals[q]);
      }
      const double diag = -(sabs + (1.0 + (1e4 - 1.0) * rng.uniform()));
      bool placed = false;
      for (int q = 0; q < 16; ++q) {
        if (!placed && cols[q] > i) {
          ci[e] = int32_t(i);
          av[e++] = diag;
          placed = true;
        }
        ci[e] = int32_t(cols[q]);
        av[e++] = vals[q];
      }
      if (!placed) { ci[e] = int32_t(i); av[e++] = diag; }
      rp[i + 1] = e;
    }
    if (V) fill_normal(4, n, o.p + 1, V);
    const double cc[3] = {0.1, 0.5, 1.0};
    for (int i = 0; i < 3; ++i) {
      if (t) t[i] = 1e-3 * cc[i];
      if (alpha) alpha[i] = 1.0;
    }
  } else if (cfg == 5) {
    for (int64_t i = 0; i < n; ++i) {
      ci[e] = int32_t(i);
      av[e++] = -(1.0 + 999.0 * double(i) / double(n - 1));
      if (i < n - 1) { ci[e] = int32_t(i + 1); av[e++] = 50.0; }
      rp[i + 1] = e;
    }
    if (V) fill_uniform_pm1(5, n, o.p + 1, V);
    for (int i = 0; i < 8; ++i) {
      if (t) t[i] = std::pow(10.0, -3.0 + 4.0 * double(i) / 7.0);
      if (alpha) alpha[i] = double(i + 1) / 8.0;
    }
  }
  return e == o.nnz ? 0 : 2;
}

}  // extern "C"
