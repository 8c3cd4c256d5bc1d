"""Two implementations behind one test-facing interface, so the ported
reference tests run unchanged against the CPU oracle (`oracle`, CPU suite)
and the CUDA product through its C ABI (`gpu`, marked tests).

Both raise ValueError for std::invalid_argument and RuntimeError for
std::runtime_error, like the reference's exception types."""
from __future__ import annotations

import numpy as np

import oracle as O


class OracleImpl:
    name = "oracle"

    def op(self, A):
        return O.csr_from_dense(A)

    def op_csr(self, n, rp, ci, av):
        return O.csr_from_arrays(n, rp, ci, av)

    def apply(self, op, X):
        return O.apply(op, X)

    def shifted_apply(self, op, xi, X):
        return O.shifted_apply(op, xi, X)

    def select_parameters(self, op, m=61, tol=-1.0, delta=0.8):
        return O.select_parameters(op, m, tol, delta)

    def basis(self, op, m=61, delta=0.8):
        return O.build_power_basis(op, m, delta)

    def objective(self, basis, xi):
        return basis.objective(xi)

    def minimize_shift(self, basis):
        return basis.minimize_shift()

    def parameters_for_shift(self, op, basis, xi, tol):
        return basis.parameters_for_shift(xi, tol)

    def params(self, s=1.0, xi=0.0, s0=1.0, f_min=0.0, m=61, r=0):
        return O.ScalingShift(s, xi, s0, f_min, m, r)

    def phimv_block(self, op, t, alpha, V, tol, params):
        return O.phimv_block(op, np.atleast_1d(t), np.atleast_1d(alpha), V, tol,
                             O.ScalingShift(*params.astuple()))

    def phimv(self, op, t, alpha, V, tol, params):
        return O.phimv(op, t, alpha, V, tol, O.ScalingShift(*params.astuple()))

    def series_direct(self, op, t, alpha, V, tol, coeffs=None):
        return O.block_series_direct(op, t, alpha, V, tol, coeffs)

    # integrator.cpp: (u_next, records) / (u, t, records)
    def rk_step(self, op, gamma, u, h, tol, params):
        return O.exprk4s6_step(op, gamma, u, h, tol, O.ScalingShift(*params.astuple()))

    def integrate(self, op, gamma, u0, h, t_end, tol, params, keep_records=True):
        return O.integrate(op, gamma, u0, h, t_end, tol, O.ScalingShift(*params.astuple()),
                           keep_records)


class GpuImpl:
    name = "gpu"

    def __init__(self):
        import paper_2509_26475_b200 as P
        self.P = P

    def op(self, A):
        return self.P.CsrOperator.from_dense(A)

    def op_csr(self, n, rp, ci, av):
        return self.P.CsrOperator(n, rp, ci, av)

    def apply(self, op, X):
        return op.apply(np.asarray(X).reshape(op.n, -1))

    def shifted_apply(self, op, xi, X):
        return op.shifted_apply(xi, np.asarray(X).reshape(op.n, -1))

    def select_parameters(self, op, m=61, tol=-1.0, delta=0.8):
        return self.P.select_parameters(op, m, tol, delta)

    def basis(self, op, m=61, delta=0.8):
        b = self.P.build_power_basis(op, m, delta)
        b.columns_ = b.columns
        return b

    def objective(self, basis, xi):
        return self.P.objective(basis, xi)

    def minimize_shift(self, basis):
        return self.P.minimize_shift(basis)

    def parameters_for_shift(self, op, basis, xi, tol):
        return self.P.parameters_for_shift(op, basis, xi, tol)

    def params(self, s=1.0, xi=0.0, s0=1.0, f_min=0.0, m=61, r=0):
        return self.P.ScalingShift(s, xi, s0, f_min, m, r)

    def phimv_block(self, op, t, alpha, V, tol, params):
        P = self.P
        res = P.phimv_block(op, P.BlockPhiRequest(np.atleast_1d(t), np.atleast_1d(alpha), V, tol,
                                                  P.ScalingShift(*params.astuple())))
        return res.W, res.stats

    def phimv(self, op, t, alpha, V, tol, params):
        P = self.P
        res = P.phimv(op, P.PhiRequest(t, alpha, V, tol, P.ScalingShift(*params.astuple())))
        return res.w, res.exp_v0, res.tail, res.stats

    def series_direct(self, op, t, alpha, V, tol, coeffs=None):
        P = self.P
        req = P.BlockPhiRequest(np.atleast_1d(t), np.atleast_1d(alpha), V, tol,
                                P.ScalingShift(1.0, 0.0, 1.0, 0.0, 61, 0))
        return P.block_series_direct(op, req, coeffs)

    def _problem(self, op, gamma, u0):
        return self.P.ADRProblem(0, 0, 0.0, 0.0, float(gamma), op, np.asarray(u0, dtype=float))

    def rk_step(self, op, gamma, u, h, tol, params):
        P = self.P
        un, rec = P.exprk4s6_step(self._problem(op, gamma, u), P.StepState(0.0, u, h), tol,
                                  P.ScalingShift(*params.astuple()))
        return un, rec.calls

    def integrate(self, op, gamma, u0, h, t_end, tol, params, keep_records=True):
        P = self.P
        res = P.integrate(self._problem(op, gamma, u0), h, t_end, tol,
                          P.ScalingShift(*params.astuple()), keep_records)
        return res.u, res.t, [c for st in res.steps for c in st.calls]


def basis_columns(impl, b):
    return b.columns if impl.name == "oracle" else b.columns_


# ---------------------------------------------------------------------------
# reference test utilities, restated (proj/tests/test_util.hpp)
# ---------------------------------------------------------------------------
def rel_err(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    d = np.linalg.norm(want)
    return np.linalg.norm(got - want) / d if d > 0 else np.linalg.norm(got - want)


def spectral_scaled(A, target):
    """A * target / ||A||_2 (the tests' JacobiSVD scaling)."""
    nrm = np.linalg.svd(A, compute_uv=False)[0]
    return A * (target / nrm) if nrm > 0 else A


def log_shifted_power_norm(A, xi, v, m):  # test_util.hpp:47-60
    w = np.array(v, dtype=np.float64)
    acc = 0.0
    for _ in range(m):
        w = A @ w - xi * w
        nw = O.stable_norm(w)
        if nw == 0.0:
            return -np.inf
        acc += np.log(nw)
        w = w / nw
    return acc


def shifted_power_root(A, xi, v, m):  # test_util.hpp:62-67
    ln = log_shifted_power_norm(A, xi, v, m)
    return float(np.exp(ln / m)) if np.isfinite(ln) else 0.0


def grid_argmin(f, lo, hi, samples):  # test_util.hpp:69-81
    best_x, best_f = lo, f(lo)
    for i in range(1, samples + 1):
        x = lo + (hi - lo) * i / samples
        fx = f(x)
        if fx < best_f:
            best_f, best_x = fx, x
    return best_x


def taylor_expm(A, terms=60):  # test_util.hpp:35-45
    E = np.eye(A.shape[0])
    T = np.eye(A.shape[0])
    for k in range(1, terms + 1):
        T = (T @ A) / k
        E = E + T
    return E


def chebyshev_laplacian(N, L):
    """problems.cpp:11-34 restated (dense test operator)."""
    j = np.arange(N + 1)
    x = (np.cos(np.pi * j / N) + 1.0) * (L / 2.0)
    c = np.where((j == 0) | (j == N), 2.0, 1.0) * np.where(j % 2 == 0, 1.0, -1.0)
    D = np.empty((N + 1, N + 1))
    for i in range(N + 1):
        for k in range(N + 1):
            dx = x[i] - x[k] + (1.0 if i == k else 0.0)
            D[i, k] = (c[i] / c[k]) / dx
    D -= np.diag(D.sum(axis=1))
    A = ((2.0 / L) * (2.0 / L)) * (D @ D)
    return A[1:N, 1:N].copy()
