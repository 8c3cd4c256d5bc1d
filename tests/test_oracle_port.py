"""Port of proj/tests/test_oracle.cpp (the long-double high-precision oracle:
dense_expm, reference_w, dense_phi), run against the restatement in
oracle/phx_oracle.cpp -- it is the independent reference the evaluator's
"within tolerance of a high-precision check" is measured against.  The
low-rank cases are out of scope.  dense_expm(M) is
dense_phi(M, 1, 0)[0]."""
import math

import numpy as np
import pytest

import oracle as O
from impls import rel_err


def expm(M):
    return O.dense_phi(M, 1.0, 0)[0]


def eig_expm(S, t=1.0):
    w, Q = np.linalg.eigh(S)
    return (Q * np.exp(t * w)) @ Q.T


def test_dense_expm_basics():  # :10-39
    assert np.linalg.norm(expm(np.zeros((4, 4))) - np.eye(4)) == 0.0
    S = O.Rng(23).matrix(8, 8)
    S = 0.5 * (S + S.T)
    assert rel_err(expm(S), eig_expm(S)) < 1e-13
    S = O.Rng(29).matrix(6, 6)
    S = 12.0 * 0.5 * (S + S.T)
    assert rel_err(expm(S), eig_expm(S)) < 1e-12
    with pytest.raises(RuntimeError, match="overflowed"):
        expm(np.eye(2) * 1e4)


def test_reference_w_trivial_cases():  # :41-75
    V = O.Rng(31).matrix(5, 3)
    got = O.reference_w(np.zeros((5, 5)), V, 1.0, 1.0)
    assert rel_err(got, V[:, 0] + V[:, 1] + 0.5 * V[:, 2]) < 1e-15
    rng = O.Rng(37)
    S = rng.matrix(6, 6)
    S = 0.5 * (S + S.T)
    v = rng.matrix(6, 1)
    assert rel_err(O.reference_w(S, v, 0.3, 1.0), eig_expm(S, 0.3) @ v.ravel()) < 1e-13
    with pytest.raises(ValueError, match="2000"):
        O.reference_w(np.zeros((2001, 2001)), np.ones((2001, 1)), 1.0, 1.0)
    A = np.array([[0.0, 1.0], [0.0, 0.0]])
    Vn = np.zeros((2, 2))
    Vn[0, 1] = 1.0  # v0 = 0, v1 = e1; phi_1(A) = I + A/2
    got = O.reference_w(A, Vn, 1.0, 1.0)
    assert got[0] == pytest.approx(1.0, rel=1e-15) and abs(got[1]) < 1e-16


def test_reference_w_alpha_absorption():  # :77-98
    rng = O.Rng(41)
    A = 0.7 * rng.matrix(7, 7)
    V = rng.matrix(7, 4)
    t, alpha, n, p = 0.9, -1.7, 7, 3
    base = O.reference_w(A, V, t, alpha)
    B = np.zeros((n + p, n + p))
    B[:n, :n] = t * A
    for j in range(1, p + 1):
        B[:n, n + p - j] = V[:, j]
    for i in range(p - 1):
        B[n + i, n + i + 1] = alpha
    tail = np.zeros(n + p)
    tail[:n] = V[:, 0]
    tail[n + p - 1] = alpha
    alt = (expm(B) @ tail)[:n]
    assert rel_err(alt, base) < 1e-14


def test_dense_phi():  # :100-142
    phis = O.dense_phi(np.zeros((3, 3)), 1.0, 4)
    fact = 1.0
    for j in range(5):
        if j > 0:
            fact *= j
        assert np.linalg.norm(phis[j] - np.eye(3) / fact) < 1e-16
    assert O.dense_phi(np.array([[1.0]]), 1.0, 1)[1][0, 0] == pytest.approx(math.e - 1.0,
                                                                            rel=1e-15)
    rng = O.Rng(43)
    a, b, c, d, e = 2e10, 4e8 / 6.0, 200.0 / 3.0, 3.0, 1e-8
    core_m3 = np.array([[0.0, e, 0.0], [-(a + b), -d, a], [c, 0.0, -c]])
    for M, t in [(0.5 * rng.matrix(6, 6), 0.8), (rng.matrix(4, 4), 0.8), (core_m3, 1e-5)]:
        phis = O.dense_phi(M, t, 4)
        fact = 1.0
        for j in range(4):
            if j > 0:
                fact *= j
            lhs = t * M @ phis[j + 1]
            rhs = phis[j] - np.eye(M.shape[0]) / fact
            assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(phis[j])
