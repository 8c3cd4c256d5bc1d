// The reference's C++ call sequence (select_parameters + phimv_block, as in
// proj/src/integrator.cpp:13-25 and proj/tests/test_phi_block.cpp) compiled
// against include/phx/phiact.hpp and linked with libphx.so.  Prints one line
// per check; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "phx/phiact.hpp"

using namespace phiact;

int main() {
  int fails = 0;
  // 1D Dirichlet Laplacian (BASELINE config 1 at N = 120)
  const Index N = 120;
  const double s2 = double(N + 1) * double(N + 1);
  std::vector<std::int64_t> rp{0};
  std::vector<std::int32_t> ci;
  std::vector<double> av;
  for (Index i = 0; i < N; ++i) {
    if (i > 0) { ci.push_back(int32_t(i - 1)); av.push_back(s2); }
    ci.push_back(int32_t(i)); av.push_back(-2.0 * s2);
    if (i < N - 1) { ci.push_back(int32_t(i + 1)); av.push_back(s2); }
    rp.push_back(std::int64_t(ci.size()));
  }
  const LinearOperator op = csr_operator(N, rp, ci, av, "laplacian1d");
  const ScalingShift sel = select_parameters(op, kDefaultDegree, 1e-12);
  std::printf("select_parameters: s=%.17g xi=%.17g s0=%.17g r=%d\n", sel.s, sel.xi, sel.s0, sel.r);
  if (!(sel.s > 0.0) || sel.m != 61) ++fails;

  BlockPhiRequest req;
  req.t = Vector{1e-3 * 0.5, 1e-3 / 3.0, 1e-3};
  req.alpha = Vector{0.5, 1.0 / 3.0, 1.0};
  req.V = Matrix(N, 4);
  for (Index j = 0; j < 4; ++j)
    for (Index i = 0; i < N; ++i) req.V(i, j) = std::sin(0.1 * double(i + 1) * double(j + 1));
  req.tol = 1e-12;
  req.params = sel;
  const BlockPhiResult res = phimv_block(op, req);
  long want = long(res.stats.series_len_S - 1) * 12 + 3;
  for (int l : res.stats.series_lens_F) want += 6L * l;
  std::printf("phimv_block: s_eff=%ld L_S=%d sweeps=%zu matvecs=%ld W(0,0)=%.17g\n",
              res.stats.s_effective, res.stats.series_len_S, res.stats.series_lens_F.size(),
              res.stats.matvecs, res.W(0, 0));
  if (res.stats.matvecs != want) ++fails;
  if (long(res.stats.series_lens_F.size()) != res.stats.s_effective - 1) ++fails;

  // single variant: r = 1 agrees with the block column (test_phi_block.cpp:19-39)
  PhiRequest sreq;
  sreq.t = req.t(2);
  sreq.alpha = req.alpha(2);
  sreq.V = req.V;
  sreq.tol = 1e-12;
  sreq.params = sel;
  const PhiResult single = phimv(op, sreq);
  double num = 0.0, den = 0.0;
  for (Index i = 0; i < N; ++i) {
    num += (single.w(i) - res.W(i, 2)) * (single.w(i) - res.W(i, 2));
    den += res.W(i, 2) * res.W(i, 2);
  }
  std::printf("block-single rel err %.3e\n", std::sqrt(num / den));
  if (!(std::sqrt(num / den) <= 1e-11)) ++fails;

  // error behaviour: std::invalid_argument with the reference's message
  try {
    BlockPhiRequest bad = req;
    bad.t = Vector();
    bad.alpha = Vector();
    phimv_block(op, bad);
    ++fails;
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument: %s\n", e.what());
  }
  try {
    ScalingShift forced;
    forced.s = 1e-300;
    forced.xi = 1e5;
    BlockPhiRequest bad = req;
    bad.params = forced;
    bad.t = Vector{1.0};
    bad.alpha = Vector{1.0};
    phimv_block(op, bad);
    ++fails;
  } catch (const std::runtime_error& e) {
    std::printf("runtime_error: %s\n", e.what());
  }
  // the integrator (integrator.hpp): four block calls per step, state on the device
  {
    const ADRProblem prob = adr_build(16, 16);
    const ScalingShift isel = select_parameters(prob.op, kDefaultDegree, 1e-10);
    StepState st;
    st.u = prob.u0;
    st.h = 0.125 / 16.0;
    StepRecord rec;
    const Vector u1 = exprk4s6_step(prob, st, 1e-10, isel, &rec);
    const IntegrateResult ir = integrate(prob, st.h, 2 * st.h, 1e-10, isel);
    int ok = ir.steps.size() == 2 && ir.t == 2 * st.h;
    for (Index i = 0; i < u1.size(); ++i) ok = ok && std::isfinite(u1(i));
    for (const RunRecord& c : rec.calls) ok = ok && c.matvecs > 0;
    std::printf("integrator steps %zu t %.6f ok %d\n", ir.steps.size(), ir.t, ok);
    if (!ok) ++fails;
    try {
      integrate(prob, 0.3, 1.0, 1e-8, isel);
      ++fails;
    } catch (const std::invalid_argument& e) {
      std::printf("invalid_argument: %s\n", e.what());
    }
  }
  std::printf("%d failure(s)\n", fails);
  return fails;
}
