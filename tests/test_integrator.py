"""The evaluator's consumer: the expRK4s6 integrator
(proj/src/integrator.cpp) on the ADR problem (proj/src/problems.cpp:184-250).

CPU suite: the oracle's restatement pinned by ports of
proj/tests/test_integrator.cpp and the ADR cases of test_problems.cpp, plus
the CSR form of the ADR operator checked against the reference's matrix-free
stencil.  gpu: the product (phx_exprk4s6_step / phx_integrate, state resident
on the device) bitwise against the oracle on the same CSR."""
import math

import numpy as np
import pytest
from scipy.linalg import expm  # dense_expm of the reference tests (test infrastructure)

import oracle as O
from impls import GpuImpl, OracleImpl, rel_err

IMPLS = [pytest.param("oracle"), pytest.param("gpu", marks=pytest.mark.gpu)]
U = 2.0 ** -53


@pytest.fixture(params=IMPLS)
def impl(request):
    return OracleImpl() if request.param == "oracle" else GpuImpl()


def adr_arrays(nx, ny, eps=1e-3, alpha_adv=-0.5):
    import paper_2509_26475_b200 as P  # phx_adr_csr is host code (no device work)
    return P.adr_csr(nx, ny, eps, alpha_adv)


def dense_of(n, rp, ci, av):
    A = np.zeros((n, n))
    for i in range(n):
        for e in range(rp[i], rp[i + 1]):
            A[i, ci[e]] += av[e]
    return A


# ------------------------------------------------------- the ADR operator
def test_adr_csr_is_the_reference_stencil():
    """The CSR rows reproduce adr_build's matrix-free apply (problems.cpp:206-231)."""
    for nx, ny, eps, al in [(8, 8, 1e-3, -0.5), (12, 9, 1e-3, -0.5), (16, 16, 2e-2, 0.7),
                            (10, 13, 1e-3, 0.0)]:
        rp, ci, av, u0 = adr_arrays(nx, ny, eps, al)
        n = nx * ny
        assert rp[n] <= 5 * n and np.all(np.diff(rp) >= 3)
        for i in range(n):  # sorted, distinct columns
            assert np.all(np.diff(ci[rp[i]:rp[i + 1]]) > 0)
        op = O.csr_from_arrays(n, rp, ci, av)
        rng = np.random.default_rng(nx * 100 + ny)
        for _ in range(3):
            u = rng.standard_normal(n)
            y_csr = O.apply(op, u.reshape(-1, 1)).ravel()
            y_st = O.adr_apply_stencil(nx, ny, eps, al, u)
            assert np.max(np.abs(y_csr - y_st)) <= 8 * U * np.max(np.abs(y_st))
        assert np.array_equal(u0, O.adr_u0(nx, ny))


def test_adr_problem_properties():  # test_problems.cpp:115-166
    import paper_2509_26475_b200 as P
    # reaction vanishes at u = 1/2
    prob_r = P.ADRProblem(8, 8, 1e-3, -0.5, 1000.0, None, np.zeros(64))
    assert np.abs(prob_r.reaction(np.full(64, 0.5))).max() == 0.0
    # initial condition vanishes on the Dirichlet side, peak inside
    _, _, _, u0 = adr_arrays(10, 10)
    assert u0.max() > 0.5 and u0.min() >= 0.0 and u0[0] == 0.0
    # operator matches a hand stencil at an interior node
    nx = ny = 12
    rp, ci, av, _ = adr_arrays(nx, ny, 1e-3, -0.5)
    u = O.Rng(211).matrix(nx * ny, 1).ravel()
    y = O.apply(O.csr_from_arrays(nx * ny, rp, ci, av), u.reshape(-1, 1)).ravel()
    h = 1.0 / nx
    i, j = 5, 7
    idx = j * nx + i
    lap = 1e-3 * (u[idx - 1] + u[idx + 1] + u[idx - nx] + u[idx + nx] - 4.0 * u[idx]) / (h * h)
    adv = -0.5 * ((u[idx + 1] - u[idx - 1]) + (u[idx + nx] - u[idx - nx])) / (2.0 * h)
    assert y[idx] == pytest.approx(lap - adv, rel=1e-12)
    # linear
    rp, ci, av, _ = adr_arrays(9, 9)
    op = O.csr_from_arrays(81, rp, ci, av)
    a, b = O.Rng(223).matrix(81, 1).ravel(), O.Rng(227).matrix(81, 1).ravel()
    lhs = O.apply(op, (2.0 * a - 3.0 * b).reshape(-1, 1)).ravel()
    rhs = 2.0 * O.apply(op, a.reshape(-1, 1)).ravel() - 3.0 * O.apply(op, b.reshape(-1, 1)).ravel()
    assert rel_err(lhs, rhs) < 1e-13
    # semidiscrete evolution matches the dense exponential
    rp, ci, av, u0 = adr_arrays(12, 12, 1e-3, -0.5)
    A = dense_of(144, rp, ci, av)
    want = expm(0.5 * A) @ u0
    got = O.reference_w(A, u0.reshape(-1, 1), 0.5, 1.0)
    assert rel_err(got, want) < 1e-13


# --------------------------------------------- test_integrator.cpp, ported
def test_scalar_linear_reproduces_exponential(impl):  # test_integrator.cpp:37-43
    op = impl.op(np.array([[-1.0]]))
    sel = impl.select_parameters(op)
    u1, recs = impl.rk_step(op, 0.0, np.array([2.0]), 0.1, 1e-14, sel)
    assert u1[0] == pytest.approx(2.0 * math.exp(-0.1), rel=1e-12)
    assert len(recs) == 4


def test_zero_rhs_leaves_state(impl):  # :45-52
    op = impl.op(np.array([[0.0]]))
    sel = impl.select_parameters(op)
    u, t, recs = impl.integrate(op, 0.0, np.array([1.5]), 0.25, 1.0, 1e-10, sel)
    assert u[0] == 1.5
    assert len(recs) == 4 * 4 and t == 1.0


def test_linear_adr_step_is_the_exponential(impl):  # :54-76
    rp, ci, av, u0 = adr_arrays(12, 12, 1e-3, -0.5)
    op = impl.op_csr(144, rp, ci, av)
    tol = 1e-12
    sel = impl.select_parameters(op, 61, tol)
    h = 0.05
    u1, recs = impl.rk_step(op, 0.0, u0, h, tol, sel)
    want = O.reference_w(dense_of(144, rp, ci, av), u0.reshape(-1, 1), h, 1.0)
    assert rel_err(u1, want) <= 10.0 * tol
    assert len(recs) == 4
    for c in recs:
        assert c.s_effective >= 1 and c.matvecs > 0


def test_linear_heat_many_steps_matches_expm(impl):  # :78-87
    rp, ci, av, u0 = adr_arrays(12, 12, 1e-3, 0.0)
    op = impl.op_csr(144, rp, ci, av)
    T = 0.1
    sel = impl.select_parameters(op, 61, 1e-12)
    u, t, _ = impl.integrate(op, 0.0, u0, T / 8.0, T, 1e-12, sel)
    want = expm(T * dense_of(144, rp, ci, av)) @ u0
    assert rel_err(u, want) <= 1e-9
    assert t == pytest.approx(T)


def test_nonlinear_convergence_order():  # :89-112 (oracle; the GPU matches it bitwise below)
    impl = OracleImpl()
    rp, ci, av, u0 = adr_arrays(16, 16)
    op = impl.op_csr(256, rp, ci, av)
    tol = 1e-10
    sel = impl.select_parameters(op, 61, tol)
    t_end = 0.125
    h0 = t_end / 16.0
    ref, _, _ = impl.integrate(op, 1000.0, u0, h0 / 32.0, t_end, U, sel, keep_records=False)
    errs = []
    for h in (h0, h0 / 2.0, h0 / 4.0):
        u, _, _ = impl.integrate(op, 1000.0, u0, h, t_end, tol, sel, keep_records=False)
        errs.append(np.abs(u - ref).max() / np.abs(ref).max())
    assert errs[1] < errs[0] and errs[2] < errs[1]
    assert math.log2(errs[0] / errs[2]) / 2.0 >= 3.2


def test_integrate_input_validation(impl):  # :114-119
    op = impl.op(np.array([[-1.0]]))
    sel = impl.select_parameters(op)
    with pytest.raises(ValueError, match="h must be positive"):
        impl.integrate(op, 0.0, np.array([1.0]), -0.1, 1.0, 1e-8, sel)
    with pytest.raises(ValueError, match="not a multiple"):
        impl.integrate(op, 0.0, np.array([1.0]), 0.3, 1.0, 1e-8, sel)


# ------------------------------------------------- GPU vs oracle, bitwise
def _recs_equal(a, b):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert (x.s_effective, x.series_len_S, x.matvecs) == (y.s_effective, y.series_len_S,
                                                              y.matvecs)


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,steps,gamma", [(16, 16, 4, 1000.0), (33, 20, 3, 1000.0),
                                               (128, 128, 2, 1000.0), (24, 24, 3, 0.0)])
def test_gpu_integrate_bitwise(nx, ny, steps, gamma):
    rp, ci, av, u0 = adr_arrays(nx, ny)
    n = nx * ny
    o, g = OracleImpl(), GpuImpl()
    oop, gop = o.op_csr(n, rp, ci, av), g.op_csr(n, rp, ci, av)
    tol = 1e-10
    sel = g.select_parameters(gop, 61, tol)
    h = 0.125 / 16.0
    uo, to, ro = o.integrate(oop, gamma, u0, h, steps * h, tol, sel)
    ug, tg, rg = g.integrate(gop, gamma, u0, h, steps * h, tol, sel)
    assert np.array_equal(ug, uo) and tg == to
    _recs_equal(rg, ro)
    # the single-step entry point
    uo1, ro1 = o.rk_step(oop, gamma, u0, h, tol, sel)
    ug1, rg1 = g.rk_step(gop, gamma, u0, h, tol, sel)
    assert np.array_equal(ug1, uo1)
    _recs_equal(rg1, ro1)


@pytest.mark.gpu
def test_gpu_integrate_rejects_partitioned():
    import paper_2509_26475_b200 as P
    rp, ci, av, u0 = adr_arrays(16, 16)
    op = P.CsrOperator(256, rp, ci, av, parts=2)
    sel = P.ScalingShift(1.0, 0.0, 1.0, 0.0, 61, 0)
    with pytest.raises(ValueError, match="partitioned"):
        P.integrate(P.ADRProblem(16, 16, 1e-3, -0.5, 1000.0, op, u0), 0.01, 0.02, 1e-8, sel)


@pytest.mark.gpu
def test_gpu_integrate_traced_matches_untraced():
    """A step's four evaluations are decoded after one synchronize; with the
    stopping trace on they run synchronously instead. Same state, same records."""
    import paper_2509_26475_b200 as P
    rp, ci, av, u0 = adr_arrays(20, 20)
    g = GpuImpl()
    gop = g.op_csr(400, rp, ci, av)
    tol = 1e-10
    sel = g.select_parameters(gop, 61, tol)
    h = 0.125 / 16.0
    ua, ta, ra = g.integrate(gop, 1000.0, u0, h, 3 * h, tol, sel)
    P.set_trace(3 * 100000)
    try:
        ub, tb, rb = g.integrate(gop, 1000.0, u0, h, 3 * h, tol, sel)
    finally:
        P.set_trace(0)
    assert np.array_equal(ua, ub) and ta == tb
    _recs_equal(ra, rb)
    assert all(r.matvecs > 0 for r in rb)
