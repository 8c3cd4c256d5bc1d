"""Port of proj/tests/test_linop.cpp:13-95 (operators and shifted_apply),
run against the CPU oracle and -- marked gpu -- the product's CSR operator.
Dense test matrices enter as CSR with every entry stored."""
import numpy as np
import pytest

import oracle as O
from impls import GpuImpl, OracleImpl, rel_err

IMPLS = [pytest.param("oracle"), pytest.param("gpu", marks=pytest.mark.gpu)]


@pytest.fixture(params=IMPLS)
def impl(request):
    return OracleImpl() if request.param == "oracle" else GpuImpl()


def test_identity_and_nilpotent_shift(impl):  # :13-27
    X = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert np.abs(impl.apply(impl.op(np.eye(2)), X) - X).max() == 0.0
    y = impl.apply(impl.op(np.array([[0.0, 1.0], [0.0, 0.0]])), np.array([0.0, 1.0]))
    assert y.ravel()[0] == 1.0 and y.ravel()[1] == 0.0


def test_matches_naive_triple_loop(impl):  # :29-36
    rng = O.Rng(7)
    A = rng.matrix(5, 5)
    X = rng.matrix(5, 3)
    want = np.array([[sum(A[i, k] * X[k, j] for k in range(5)) for j in range(3)]
                     for i in range(5)])
    assert rel_err(impl.apply(impl.op(A), X), want) < 1e-14


@pytest.mark.gpu
def test_rejects_bad_input():  # :38-45 (the product's dense_operator / apply checks)
    import paper_2509_26475_b200 as P
    with pytest.raises(ValueError):
        P.CsrOperator.from_dense(np.zeros((2, 3)))
    bad = np.zeros((2, 2))
    bad[0, 0] = np.nan
    with pytest.raises(ValueError):
        P.CsrOperator.from_dense(bad)
    op = P.CsrOperator.from_dense(np.eye(3))
    with pytest.raises((ValueError, Exception)):
        op.apply(np.zeros((2, 2)))


def test_linear_shape_preserving_deterministic(impl):  # :47-62
    rng = O.Rng(11)
    A = rng.matrix(8, 8)
    op = impl.op(A)
    X, Y = rng.matrix(8, 4), rng.matrix(8, 4)
    a, b = 0.37, -2.25
    lhs = impl.apply(op, a * X + b * Y)
    rhs = a * impl.apply(op, X) + b * impl.apply(op, Y)
    scale = 10.0 * 2.0 ** -53 * np.linalg.norm(a * X + b * Y)
    assert np.linalg.norm(lhs - rhs) <= 10 * scale * np.linalg.norm(A)
    assert lhs.shape == (8, 4)
    assert np.abs(impl.apply(op, X) - impl.apply(op, X)).max() == 0.0


def test_shifted_apply(impl):  # :64-95
    x = np.array([3.0, -4.0])
    assert np.linalg.norm(impl.shifted_apply(impl.op(np.eye(2)), 1.0, x)) == 0.0
    y = impl.shifted_apply(impl.op(np.zeros((2, 2))), -2.0, np.array([1.0, 1.0])).ravel()
    assert y[0] == 2.0 and y[1] == 2.0
    rng = O.Rng(3)
    A = rng.matrix(4, 4)
    xv = rng.matrix(4, 1).ravel()
    got = impl.shifted_apply(impl.op(A), 0.7, xv).ravel()
    assert rel_err(got, A @ xv - 0.7 * xv) < 1e-14
    rng = O.Rng(5)
    A = rng.matrix(6, 6)
    X = rng.matrix(6, 2)
    op = impl.op(A)
    assert np.abs(impl.shifted_apply(op, 0.0, X) - impl.apply(op, X)).max() == 0.0
