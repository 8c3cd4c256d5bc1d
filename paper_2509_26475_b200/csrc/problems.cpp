// The expRK4s6 integrator's test problem: the 2D
// advection-diffusion-reaction semidiscretization of adr_build
// (proj/src/problems.cpp:184-250, problems.hpp:46-66) as a CSR operator.
//
// The reference applies the stencil matrix-free,
//   y = dxx (uw - 2uc + ue) + dyy (us - 2uc + un) - (ax (ue - uw) + ay (un - us)),
// with mirror ghosts at x = 0 / y = 0 (uw := u(idx+1), us := u(idx+nx)) and
// eliminated Dirichlet edges at x = 1 / y = 1 (ue, un := 0).  The product
// evaluates every operator as CSR, so the same linear map is stored as
// per-neighbour coefficients:
//   west dxx + ax, east dxx - ax, south dyy + ay, north dyy - ay,
//   centre (-2 dxx) + (-2 dyy),
// a mirrored neighbour's two coefficients summed (east + west at i = 0,
// north + south at j = 0), columns ascending.  The CSR row sum rounds
// differently from the stencil expression (agreement to ~1e-15 relative,
// tests/test_integrator.py); the evaluator and the oracle both consume this
// CSR, so GPU-vs-oracle parity stays bitwise.  u0 is the reference's
// initial condition, bit for bit (problems.cpp:239-246).
#include <cstdint>

#include "../../include/phx.h"

extern "C" {

phx_status phx_adr_csr(int32_t nx, int32_t ny, double eps, double alpha_adv, int64_t* row_ptr,
                       int32_t* col_idx, double* vals, double* u0) {
  if (nx < 8 || ny < 8) return PHX_EINVAL;  // "adr_build: grid must be at least 8x8"
  if (int64_t(nx) * int64_t(ny) >= (int64_t(1) << 31)) return PHX_EINVAL;
  const double hx = 1.0 / nx;
  const double hy = 1.0 / ny;
  const double dxx = eps / (hx * hx);
  const double dyy = eps / (hy * hy);
  const double ax = alpha_adv / (2.0 * hx);
  const double ay = alpha_adv / (2.0 * hy);
  const double cw = dxx + ax, ce = dxx - ax, cs = dyy + ay, cn = dyy - ay;
  const double cc = (-2.0 * dxx) + (-2.0 * dyy);
  int64_t e = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int64_t idx = int64_t(j) * nx + i;
      auto put = [&](int64_t col, double v) {
        if (col_idx) col_idx[e] = int32_t(col);
        if (vals) vals[e] = v;
        ++e;
      };
      if (j > 0) put(idx - nx, cs);
      if (i > 0) put(idx - 1, cw);
      put(idx, cc);
      if (i < nx - 1) put(idx + 1, i > 0 ? ce : ce + cw);            // mirror at x = 0
      if (j < ny - 1) put(idx + nx, j > 0 ? cn : cn + cs);           // mirror at y = 0
      if (row_ptr) row_ptr[idx + 1] = e;
    }
  if (u0)
    for (int j = 0; j < ny; ++j) {
      const double y = j * hy;
      for (int i = 0; i < nx; ++i) {
        const double x = i * hx;
        u0[int64_t(j) * nx + i] =
            256.0 * x * x * y * y * (1.0 - x) * (1.0 - x) * (1.0 - y) * (1.0 - y);
      }
    }
  return PHX_OK;
}

}  // extern "C"
