// A reference-style call site (Eigen types, dense_operator, concurrent
// evaluations on one operator) against include/phx/phiact.hpp.  Built with
// -I tests/cpp/fake_eigen: the header must pick Eigen::MatrixXd/VectorXd.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <thread>
#include <type_traits>

#include "phx/phiact.hpp"

static_assert(std::is_same<phiact::Matrix, Eigen::MatrixXd>::value, "phiact::Matrix is Eigen's");
static_assert(std::is_same<phiact::Vector, Eigen::VectorXd>::value, "phiact::Vector is Eigen's");

int main() {
  using namespace phiact;
  const Index n = 300;
  // A = (n+1)^2 tridiag(1, -2, 1) as a dense Eigen matrix (C1's operator)
  Eigen::MatrixXd A = Eigen::MatrixXd::Zero(n, n);
  const double h2 = double(n + 1) * double(n + 1);
  for (Index i = 0; i < n; ++i) {
    A(i, i) = -2.0 * h2;
    if (i > 0) A(i, i - 1) = h2;
    if (i + 1 < n) A(i, i + 1) = h2;
  }
  const LinearOperator op = dense_operator(A);
  try {
    dense_operator(Eigen::MatrixXd(3, 4));
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument: %s\n", e.what());
  }
  const ScalingShift ss = select_parameters(op, kDefaultDegree, 1e-12);
  BlockPhiRequest req;
  req.t = Eigen::VectorXd(3);
  req.alpha = Eigen::VectorXd(3);
  const double c[3] = {0.5, 1.0 / 3.0, 1.0};
  for (int i = 0; i < 3; ++i) {
    req.t(i) = 1e-3 * c[i];
    req.alpha(i) = c[i];
  }
  req.V = Eigen::MatrixXd(n, 4);
  for (Index j = 0; j < 4; ++j)
    for (Index i = 0; i < n; ++i) req.V(i, j) = std::sin(0.01 * double(i + 1) * double(j + 1));
  req.tol = 1e-12;
  req.params = ss;
  const BlockPhiResult ref = phimv_block(op, req);
  std::printf("s_eff %ld L_S %d sweeps %zu\n", ref.stats.s_effective, ref.stats.series_len_S,
              ref.stats.series_lens_F.size());
  // concurrent evaluations on one handle: each thread's W equals the serial one
  const int T = 4;
  BlockPhiResult outs[T];
  std::thread th[T];
  for (int k = 0; k < T; ++k) th[k] = std::thread([&, k] { outs[k] = phimv_block(op, req); });
  for (auto& x : th) x.join();
  bool same = true;
  for (int k = 0; k < T; ++k)
    same = same && std::memcmp(outs[k].W.data(), ref.W.data(), sizeof(double) * size_t(n * 3)) == 0 &&
           outs[k].stats.series_lens_F == ref.stats.series_lens_F;
  std::printf("concurrent equal %d\n", same ? 1 : 0);
  // phimv: V row check (phi_single.cpp:16)
  try {
    PhiRequest pr;
    pr.V = Eigen::MatrixXd(n + 1, 2);
    pr.params = ss;
    phimv(op, pr);
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument: %s\n", e.what());
  }
  return same ? 0 : 1;
}
