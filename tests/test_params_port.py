"""Port of proj/tests/test_params.cpp (parameter selection, Alg. 1), run
against the CPU oracle and — marked gpu — the CUDA product."""
import numpy as np
import pytest

import oracle as O
from impls import (GpuImpl, OracleImpl, basis_columns, chebyshev_laplacian, grid_argmin,
                   log_shifted_power_norm, rel_err, shifted_power_root)

IMPLS = [pytest.param("oracle"), pytest.param("gpu", marks=pytest.mark.gpu)]


@pytest.fixture(params=IMPLS)
def impl(request):
    return OracleImpl() if request.param == "oracle" else GpuImpl()


def test_forced_geometric_mean_2I(impl):  # test_params.cpp:10-15
    b = impl.basis(impl.op(2.0 * np.eye(12)))
    assert b.s0 == pytest.approx(2.0, rel=1e-12)
    assert b.r >= 3


def test_zero_operator(impl):  # :17-22
    b = impl.basis(impl.op(np.zeros((6, 6))))
    assert b.r == 0
    assert b.s0 == 1.0


def test_dominant_growth_rate(impl):  # :24-43
    A = np.diag([1.0, 1e6])
    b = impl.basis(impl.op(A))
    v = basis_columns(impl, b)[:, 0]
    logs = []
    w = v.copy()
    for _ in range(b.r):
        w = A @ w
        logs.append(np.log(O.stable_norm(w)))
    jr = max(2, b.r - 5)
    want = np.exp((logs[b.r - 1] - logs[jr - 1]) / (b.r - jr))
    assert b.s0 == pytest.approx(want, rel=1e-12)
    assert b.s0 / 1e6 == pytest.approx(1.0, rel=0.01)


def test_guard_replay(impl):  # :45-58
    b = impl.basis(impl.op(chebyshev_laplacian(24, 2.0)))
    g_max = 0.8 * np.log(np.finfo(float).max)
    g_min = 0.8 * np.log(np.finfo(float).tiny)
    ell_max = max(b.log_binom)
    assert len(b.logs) == b.r
    for k in range(1, b.r + 1):
        L = b.logs[k - 1]
        assert L + 0.5 * np.log(k + 1.0) + ell_max <= g_max
        assert L >= g_min


def test_normalized_powers(impl):  # :60-74
    A = O.Rng(61).matrix(9, 9)
    b = impl.basis(impl.op(A))
    cols = basis_columns(impl, b)
    v = cols[:, 0]
    assert np.linalg.norm(v) == pytest.approx(1.0, rel=1e-14)
    w = v.copy()
    scale = 1.0
    for k in range(1, min(b.m, 8) + 1):
        w = A @ w
        scale /= b.s0
        assert rel_err(cols[:, k], scale * w) < 1e-11


def test_objective_annihilating_shift_cI(impl):  # :77-91
    c = 1.7
    A = c * np.eye(8)
    b = impl.basis(impl.op(A))
    v = basis_columns(impl, b)[:, 0]
    assert shifted_power_root(A, c, v, b.m) == 0.0
    assert impl.objective(b, c) < 1.5
    assert impl.objective(b, 0.0) * b.s0 == pytest.approx(c, rel=1e-10)


def test_objective_zero_operator(impl):  # :92-97
    b = impl.basis(impl.op(np.zeros((5, 5))))
    assert impl.objective(b, 2.5) == pytest.approx(2.5, rel=1e-12)
    assert impl.objective(b, -0.3) == pytest.approx(0.3, rel=1e-12)


def test_objective_identity_dense(impl):  # :98-111
    rng = O.Rng(67)
    for trial in range(4):
        n = 10 + 5 * trial
        A = rng.matrix(n, n)
        b = impl.basis(impl.op(A))
        v = basis_columns(impl, b)[:, 0]
        for xi in (0.0, 0.4, -1.2):
            direct = shifted_power_root(A, xi, v, b.m) / b.s0
            assert impl.objective(b, xi) == pytest.approx(direct, rel=1e-8)


def test_minimize_shift_cI(impl):  # :115-126
    c = -2.4
    b = impl.basis(impl.op(c * np.eye(9)))
    xi, fmin = impl.minimize_shift(b)
    assert xi < 0.0
    assert xi > -np.sqrt(9.0) * b.s0
    assert fmin < impl.objective(b, 0.0)


def test_minimize_shift_skew(impl):  # :127-144
    A = np.array([[0.0, 10.0], [-10.0, 0.0]])
    b = impl.basis(impl.op(A))
    v = basis_columns(impl, b)[:, 0]
    f = lambda xi: shifted_power_root(A, xi, v, b.m)  # noqa: E731
    half = np.sqrt(2.0) * b.s0
    assert abs(grid_argmin(f, -half, half, 4000)) <= half * 2e-3
    assert abs(f(0.1) - f(-0.1)) <= 1e-10 * f(0.1)
    xi, fmin = impl.minimize_shift(b)
    assert abs(xi) <= 1e-6 * (1.0 + b.s0)
    assert fmin <= impl.objective(b, 0.0)


def test_minimize_shift_diag(impl):  # :145-169
    A = np.diag([-1.0, -3.0])
    b = impl.basis(impl.op(A))
    v = basis_columns(impl, b)[:, 0]
    half = np.sqrt(2.0) * b.s0
    f_true = lambda xi: shifted_power_root(A, xi, v, b.m)  # noqa: E731
    assert grid_argmin(f_true, -half, half, 40000) == pytest.approx(-2.0, rel=0.02)
    f_comp = lambda xi: impl.objective(b, xi)  # noqa: E731
    best = f_comp(grid_argmin(f_comp, -half, half, 2000))
    xi, fmin = impl.minimize_shift(b)
    assert fmin <= best * (1.0 + 1e-6)
    assert xi < 0.0


def test_minimizer_dominance(impl):  # :170-179
    A = O.Rng(71).matrix(14, 14)
    b = impl.basis(impl.op(A))
    xi, fmin = impl.minimize_shift(b)
    half = np.sqrt(14.0) * b.s0
    assert fmin <= impl.objective(b, 0.0)
    assert fmin <= impl.objective(b, -half)
    assert fmin <= impl.objective(b, half)


def test_select_zero_operator_floor(impl):  # :183-188
    sel = impl.select_parameters(impl.op(np.zeros((4, 4))))
    assert sel.xi == 0.0
    assert sel.s == 9.5367431640625e-7


def test_select_cI_shift_absorbs(impl):  # :189-195
    sel = impl.select_parameters(impl.op(50.0 * np.eye(6)))
    assert sel.xi > 0.0
    assert sel.s < 3.5


def test_select_defining_inequality_chebyshev(impl):  # :196-208
    A = chebyshev_laplacian(40, 2.0)
    op = impl.op(A)
    tol = 2.0 ** -53
    sel = impl.select_parameters(op, 61, tol)
    b = impl.basis(op)
    log_nu = log_shifted_power_norm(A, sel.xi, basis_columns(impl, b)[:, 0], sel.m)
    from math import lgamma, log
    lhs = -sel.m * log(sel.s) + log_nu - lgamma(sel.m + 1.0)
    assert lhs <= log(tol * (1.0 + 1e-8))


def test_select_s_recomputable(impl):  # :209-220
    A = O.Rng(73).matrix(10, 10)
    tol = 1e-10
    sel = impl.select_parameters(impl.op(A), 61, tol)
    if sel.f_min > 0.0:
        from math import exp, lgamma, log
        denom = exp((log(tol) + lgamma(62.0)) / 61.0)
        assert sel.s == pytest.approx(sel.s0 * sel.f_min / denom, rel=1e-12)


def test_invalid_arguments(impl):  # params.cpp:82-84, 216-217
    op = impl.op(np.eye(3))
    with pytest.raises(ValueError, match="m must be >= 1"):
        impl.basis(op, 0)
    with pytest.raises(ValueError, match="delta must be in"):
        impl.basis(op, 61, 0.0)
    b = impl.basis(op)
    with pytest.raises(ValueError, match="tol must be positive"):
        impl.parameters_for_shift(op, b, 0.0, 0.0)
    with pytest.raises(ValueError, match="shift must be finite"):
        impl.objective(b, float("inf"))
