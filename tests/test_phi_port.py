"""Port of proj/tests/test_phi_block.cpp, test_phi_single.cpp and the
hot-path acceptance criteria (acceptance.cpp criteria 5, 7, 8), run against
the CPU oracle and — marked gpu — the CUDA product."""
import math

import numpy as np
import pytest

import oracle as O
from impls import GpuImpl, OracleImpl, rel_err, spectral_scaled, taylor_expm

IMPLS = [pytest.param("oracle"), pytest.param("gpu", marks=pytest.mark.gpu)]
U = 2.0 ** -53


@pytest.fixture(params=IMPLS)
def impl(request):
    return OracleImpl() if request.param == "oracle" else GpuImpl()


def params_for(impl, A, tol=-1.0):
    return impl.select_parameters(impl.op(A), 61, tol if tol > 0 else U)


# ------------------------------------------------------------ test_phi_block
def test_r1_collapses_to_single(impl):  # test_phi_block.cpp:19-39
    rng = O.Rng(151)
    A = spectral_scaled(rng.matrix(7, 7), 3.0)
    V = rng.matrix(7, 4)
    tol = 1e-12
    sel = params_for(impl, A, tol)
    op = impl.op(A)
    W, _ = impl.phimv_block(op, [0.8], [1.3], V, tol, sel)
    w, *_ = impl.phimv(op, 0.8, 1.3, V, tol, sel)
    assert rel_err(W[:, 0], w) <= 10.0 * tol


def test_degenerate_nodes_identical(impl):  # :41-53
    rng = O.Rng(157)
    A = rng.matrix(6, 6)
    V = rng.matrix(6, 3)
    W, _ = impl.phimv_block(impl.op(A), [1.0] * 3, [0.4] * 3, V, -1.0, params_for(impl, A))
    assert np.abs(W[:, 0] - W[:, 1]).max() == 0.0
    assert np.abs(W[:, 1] - W[:, 2]).max() == 0.0


def test_alpha_eq_t_vs_augmented_oracle(impl):  # :55-71
    rng = O.Rng(163)
    A = spectral_scaled(rng.matrix(6, 6), 2.0)
    V = rng.matrix(6, 5)
    t = np.array([0.1, 0.5, 1.0])
    W, _ = impl.phimv_block(impl.op(A), t, t, V, -1.0, params_for(impl, A))
    for i in range(3):
        assert rel_err(W[:, i], O.reference_w(A, V, t[i], t[i])) < 1e-12


def test_block_single_consistency(impl):  # :73-98
    rng = O.Rng(167)
    for trial in range(8):
        n = 5 + trial % 4
        A = spectral_scaled(rng.matrix(n, n), 0.5 + trial)
        p = 1 + trial % 5
        r = 1 + trial % 4
        V = rng.matrix(n, p + 1)
        t = np.empty(r)
        alpha = np.empty(r)
        for i in range(r):
            t[i] = 0.1 + rng.uniform()
            alpha[i] = -1.0 + 2.0 * rng.uniform()
        tol = 1e-12
        sel = params_for(impl, A, tol)
        op = impl.op(A)
        W, _ = impl.phimv_block(op, t, alpha, V, tol, sel)
        for i in range(r):
            w, *_ = impl.phimv(op, t[i], alpha[i], V, tol, sel)
            assert rel_err(W[:, i], w) <= 1e-11


def test_joint_permutation(impl):  # :100-124
    rng = O.Rng(173)
    A = rng.matrix(6, 6)
    V = rng.matrix(6, 3)
    sel = params_for(impl, A)
    op = impl.op(A)
    W, _ = impl.phimv_block(op, [0.2, 0.7, 1.0], [1.0, -0.5, 2.0], V, -1.0, sel)
    Wp, _ = impl.phimv_block(op, [1.0, 0.2, 0.7], [2.0, 1.0, -0.5], V, -1.0, sel)
    assert np.abs(W[:, 0] - Wp[:, 1]).max() == 0.0
    assert np.abs(W[:, 1] - Wp[:, 2]).max() == 0.0
    assert np.abs(W[:, 2] - Wp[:, 0]).max() == 0.0


def test_fixed_k_mode(impl):  # :126-145
    rng = O.Rng(179)
    A = spectral_scaled(rng.matrix(8, 8), 1.5)
    p, k = 3, 2
    V = np.zeros((8, p + 1))
    V[:, k] = rng.vector(8)
    t = np.array([0.3, 0.8, 1.2])
    W, _ = impl.phimv_block(impl.op(A), t, np.ones(3), V, -1.0, params_for(impl, A))
    for i in range(3):
        want = O.dense_phi(A, t[i], k)[k] @ V[:, k]
        assert rel_err(W[:, i], want) <= 1e-11


def test_zero_weight_in_block(impl):  # :147-164
    rng = O.Rng(227)
    A = spectral_scaled(rng.matrix(6, 6), 2.0)
    V = rng.matrix(6, 3)
    W, _ = impl.phimv_block(impl.op(A), [0.8, 1.1], [0.0, 0.7], V, -1.0, params_for(impl, A))
    assert rel_err(W[:, 0], O.reference_w(A, V[:, :1], 0.8, 1.0)) < 1e-12
    assert rel_err(W[:, 1], O.reference_w(A, V, 1.1, 0.7)) < 1e-12


def test_r0_rejected(impl):  # :166-174
    A = np.eye(3)
    with pytest.raises(ValueError, match="at least one abscissa"):
        impl.phimv_block(impl.op(A), np.zeros(0), np.zeros(0), np.ones((3, 1)), -1.0,
                         params_for(impl, A))


def test_nonfinite_inputs_rejected(impl):  # phi_block.cpp:25-26
    A = np.eye(3)
    V = np.ones((3, 2))
    V[1, 1] = np.nan
    with pytest.raises(ValueError, match="inputs must be finite"):
        impl.phimv_block(impl.op(A), [1.0], [1.0], V, -1.0, params_for(impl, A))
    with pytest.raises(ValueError, match="inputs must be finite"):
        impl.phimv_block(impl.op(A), [np.inf], [1.0], np.ones((3, 2)), -1.0, params_for(impl, A))


def test_mu_overflow(impl):  # phi_block.cpp:62-68
    A = np.eye(3)
    sel = impl.params(s=1e-300, xi=1e5)
    with pytest.raises(RuntimeError, match="shift undo factor"):
        impl.phimv_block(impl.op(A), [1.0], [1.0], np.ones((3, 2)), -1.0, sel)


# ------------------------------------------------------------ test_phi_single
def test_t0_exact(impl):  # test_phi_single.cpp:58-69
    rng = O.Rng(79)
    A = rng.matrix(7, 7)
    V = rng.matrix(7, 4)
    a = 0.8
    w, _, _, rec = impl.phimv(impl.op(A), 0.0, a, V, -1.0, params_for(impl, A))
    want = V[:, 0] + a * V[:, 1] + a * a * V[:, 2] / 2.0 + a * a * a * V[:, 3] / 6.0
    assert rel_err(w, want) < 1e-15
    assert rec.s_effective == 1


def test_zero_operator_exact(impl):  # :71-79
    A = np.zeros((5, 5))
    V = O.Rng(83).matrix(5, 2)
    w, *_ = impl.phimv(impl.op(A), 1.0, 0.6, V, -1.0, params_for(impl, A))
    assert rel_err(w, V[:, 0] + 0.6 * V[:, 1]) < 1e-15


def test_nilpotent_closed_form(impl):  # :81-90
    A = np.array([[0.0, 1.0], [0.0, 0.0]])
    v0 = np.array([0.0, 1.0])
    _, e0, _, _ = impl.phimv(impl.op(A), 1.0, 1.0, v0.reshape(2, 1), -1.0, params_for(impl, A))
    assert e0[0] == pytest.approx(1.0, rel=1e-15)
    assert e0[1] == pytest.approx(1.0, rel=1e-15)


def test_p0_vs_dense_oracle(impl):  # :92-101
    rng = O.Rng(89)
    A = rng.matrix(6, 6)
    v0 = rng.vector(6)
    w, _, tail, _ = impl.phimv(impl.op(A), 1.0, 1.0, v0.reshape(6, 1), -1.0, params_for(impl, A))
    assert rel_err(w, O.reference_w(A, v0.reshape(6, 1), 1.0, 1.0)) < 1e-13
    assert np.linalg.norm(tail) == 0.0


def test_moderate_norm_recovery(impl):  # :103-114
    rng = O.Rng(97)
    A = spectral_scaled(rng.matrix(8, 8), 30.0)
    V = rng.matrix(8, 4)
    w, _, _, rec = impl.phimv(impl.op(A), 1.0, 0.9, V, -1.0, params_for(impl, A))
    assert rel_err(w, O.reference_w(A, V, 1.0, 0.9)) < 1e-12
    assert rec.s_effective > 1


def replay_series_len(A, V, t, alpha, tol, params):  # :19-54
    p = V.shape[1] - 1
    s = max(1, math.ceil(abs(t) * params.s))
    mu = math.exp(t * params.xi / s)
    J = np.zeros((p + 1, p + 1))
    for i in range(1, p):
        J[i, i + 1] = 1.0
    Jiter = (alpha * J - t * params.xi * np.eye(p + 1)) / s
    A1 = A - params.xi * np.eye(A.shape[0])
    Vw = np.column_stack([V[:, 0]] + [V[:, p + 1 - j] for j in range(1, p + 1)]) * (mu / s)
    S = Vw.copy()
    D = Vw.copy()
    k, sigma, c1 = 1, 1.0, np.inf
    c2 = np.abs(D).sum(axis=1).max()
    while c1 + c2 > tol * np.abs(S).sum(axis=1).max():
        k += 1
        c1 = c2
        sigma *= k
        Vw = Vw @ Jiter
        D = (t / s) * (A1 @ D) + Vw
        c2 = np.abs(D).sum(axis=1).max() / sigma
        S = S + D / sigma
        assert k < 500
    return k


def test_series_length_replay(impl):  # :116-127
    A = np.diag([-0.5, -1.0, -1.5, -2.0, -2.5, -3.0])
    V = O.Rng(101).matrix(6, 3)
    tol = 1e-10
    sel = params_for(impl, A, tol)
    _, _, _, rec = impl.phimv(impl.op(A), 1.0, 1.0, V, tol, sel)
    assert rec.series_len_S == replay_series_len(A, V, 1.0, 1.0, tol, sel)


def test_assembly_identity_exact(impl):  # :129-137
    rng = O.Rng(103)
    A = rng.matrix(9, 9)
    V = rng.matrix(9, 5)
    w, e0, tail, _ = impl.phimv(impl.op(A), 0.7, -1.3, V, -1.0, params_for(impl, A))
    assert np.abs(w - (e0 + (-1.3) * tail)).max() == 0.0


def test_shift_override_and_scaling(impl):  # :205-230
    rng = O.Rng(109)
    A = spectral_scaled(rng.matrix(8, 8), 2.0)
    V = rng.matrix(8, 4)
    tol = 1e-12
    op = impl.op(A)
    b = impl.basis(op)
    xi, _ = impl.minimize_shift(b)
    sel = impl.parameters_for_shift(op, b, xi, tol)
    w, *_ = impl.phimv(op, 1.0, 1.0, V, tol, sel)
    shifted = impl.parameters_for_shift(op, b, xi + 1.0, tol)
    ws, *_ = impl.phimv(op, 1.0, 1.0, V, tol, shifted)
    assert np.linalg.norm(ws - w) <= 100.0 * tol * np.linalg.norm(w)
    doubled = impl.params(*sel.astuple())
    doubled.s *= 2.0
    wd, *_ = impl.phimv(op, 1.0, 1.0, V, tol, doubled)
    assert np.linalg.norm(wd - w) <= 100.0 * tol * np.linalg.norm(w)


def test_linearity(impl):  # :232-245
    rng = O.Rng(113)
    A = rng.matrix(7, 7)
    V1 = rng.matrix(7, 3)
    V2 = rng.matrix(7, 3)
    tol = 1e-12
    sel = params_for(impl, A, tol)
    op = impl.op(A)
    lhs, *_ = impl.phimv(op, 0.9, 1.4, V1 + V2, tol, sel)
    r1, *_ = impl.phimv(op, 0.9, 1.4, V1, tol, sel)
    r2, *_ = impl.phimv(op, 0.9, 1.4, V2, tol, sel)
    assert np.linalg.norm(lhs - (r1 + r2)) <= 50.0 * tol * np.linalg.norm(lhs) + 1e-300


def test_alpha_eq_t(impl):  # :247-257
    rng = O.Rng(127)
    A = spectral_scaled(rng.matrix(9, 9), 4.0)
    V = rng.matrix(9, 4)
    w, *_ = impl.phimv(impl.op(A), 0.6, 0.6, V, -1.0, params_for(impl, A))
    assert rel_err(w, O.reference_w(A, V, 0.6, 0.6)) < 1e-12


def test_alpha_zero(impl):  # :259-268
    rng = O.Rng(131)
    A = rng.matrix(6, 6)
    V = rng.matrix(6, 3)
    w, e0, _, _ = impl.phimv(impl.op(A), 1.0, 0.0, V, -1.0, params_for(impl, A))
    assert rel_err(w, O.reference_w(A, V[:, :1], 1.0, 1.0)) < 1e-13
    assert np.linalg.norm(w - e0) == 0.0


def test_phi_tail(impl):  # :270-280 (phi_tail = phimv with v0 = 0, alpha = 1)
    rng = O.Rng(137)
    A = rng.matrix(6, 6)
    V1p = rng.matrix(6, 3)
    V = np.zeros((6, 4))
    V[:, 1:] = V1p
    w, *_ = impl.phimv(impl.op(A), 1.0, 1.0, V, -1.0, params_for(impl, A))
    assert rel_err(w, O.reference_w(A, V, 1.0, 1.0)) < 1e-13


def test_matvec_accounting(impl):  # :282-294
    rng = O.Rng(139)
    A = spectral_scaled(rng.matrix(8, 8), 6.0)
    V = rng.matrix(8, 3)
    *_, rec = impl.phimv(impl.op(A), 1.0, 1.0, V, -1.0, params_for(impl, A))
    want = (rec.series_len_S - 1) * V.shape[1] + 1 + sum(2 * x for x in rec.series_lens_F)
    assert rec.matvecs == want
    assert len(rec.series_lens_F) == rec.s_effective - 1


def test_block_matvec_accounting(impl):  # SURVEY §8a accounting identity
    rng = O.Rng(141)
    A = spectral_scaled(rng.matrix(9, 9), 60.0)
    V = rng.matrix(9, 4)
    t = np.array([0.5, 1.0, 0.25])
    W, rec = impl.phimv_block(impl.op(A), t, [1.0, 0.3, -2.0], V, -1.0, params_for(impl, A))
    w = 4 * 3
    want = (rec.series_len_S - 1) * w + 3 + sum(6 * x for x in rec.series_lens_F)
    assert rec.matvecs == want
    assert rec.s_effective > 1 and len(rec.series_lens_F) == rec.s_effective - 1


def test_non_convergence(impl):  # :296-304
    rng = O.Rng(149)
    A = spectral_scaled(rng.matrix(6, 6), 800.0)
    forced = impl.params(s=9.5367431640625e-7, xi=0.0)
    with pytest.raises(RuntimeError):
        impl.phimv(impl.op(A), 1.0, 1.0, rng.matrix(6, 2), 1e-14, forced)
    with pytest.raises(RuntimeError, match="phimv_block: series"):
        impl.phimv_block(impl.op(A), [1.0], [1.0], rng.matrix(6, 2), 1e-14, forced)


# ------------------------------------------------------------ acceptance
def test_acceptance5_block_single(impl):  # acceptance.cpp:116-147 (negative t)
    rng = O.Rng(20250809)
    worst = 0.0
    for trial in range(50):
        n = 5 + trial % 7
        A = rng.matrix(n, n)
        target = 0.5 + 5.0 * rng.uniform()
        A = spectral_scaled(A, target)
        p = trial % 6
        r = 1 + trial % 4
        V = rng.matrix(n, p + 1)
        t = np.empty(r)
        alpha = np.empty(r)
        for i in range(r):
            t[i] = -1.0 + 2.5 * rng.uniform()
            alpha[i] = -1.0 + 2.0 * rng.uniform()
        op = impl.op(A)
        sel = impl.select_parameters(op)
        W, _ = impl.phimv_block(op, t, alpha, V, -1.0, sel)
        for i in range(r):
            w, *_ = impl.phimv(op, t[i], alpha[i], V, -1.0, sel)
            worst = max(worst, rel_err(W[:, i], w))
    assert worst <= 1e-11


def test_acceptance7_exactness(impl):  # acceptance.cpp:181-276
    rng = O.Rng(424242)
    A = rng.matrix(9, 9)
    V = rng.matrix(9, 5)
    a = -0.8
    w, *_ = impl.phimv(impl.op(A), 0.0, a, V, -1.0, impl.select_parameters(impl.op(A)))
    want = np.zeros(9)
    apow, fact = 1.0, 1.0
    for j in range(5):
        if j > 0:
            apow *= a
            fact *= j
        want = want + apow / fact * V[:, j]
    assert rel_err(w, want) <= 1e-14
    N = np.diag(np.ones(5), 1)
    V = rng.matrix(6, 3)
    op = impl.op(N)
    w, *_ = impl.phimv(op, 1.0, 1.0, V, -1.0, impl.select_parameters(op))
    assert rel_err(w, O.reference_w(N, V, 1.0, 1.0)) <= 1e-13
    for trial in range(4):  # theorem identity e^{tA} v0 = tA phi_1(tA) v0 + v0
        n = 7 + 3 * trial
        A = spectral_scaled(rng.matrix(n, n), 1.0 + trial)
        v0 = rng.vector(n)
        op = impl.op(A)
        _, e0, _, _ = impl.phimv(op, 0.9, 1.0, v0.reshape(n, 1), U, impl.select_parameters(op))
        phi1 = O.dense_phi(A, 0.9, 1)[1] @ v0
        assert rel_err(e0, 0.9 * (A @ phi1) + v0) <= 10.0 * U + 1e-14


def test_jexp_chain_vs_taylor():  # test_nilpotent.cpp:106-120, acceptance crit. 7
    for p in (0, 1, 2, 3, 5, 8):
        for c in (0.1, -2.0, 7.5):
            J = np.diag(np.ones(max(p - 1, 0)), 1) if p >= 1 else np.zeros((1, 1))
            Jf = np.zeros((p + 1, p + 1))
            if p >= 2:
                Jf[1:, 1:] = J
            want = taylor_expm(c * Jf, 60)
            chain = O.jexp_chain(c, 1.0, p)
            for l in range(1, p + 1):
                for j in range(l, p + 1):
                    wv = want[l, j]
                    ulp = 2.0 * 2.0 ** -52 * max(1.0, abs(wv))
                    assert abs(chain[j - l] - wv) <= ulp
