"""block_series_direct (proj/src/phi_block.cpp:158-212),
the reference's direct power-series cross-check of the scaled evaluator.
Ported test_phi_block.cpp:176-262 cases on the oracle and (gpu) the product;
the product bitwise against the oracle on sparse operators."""
import numpy as np
import pytest

import oracle as O
from impls import GpuImpl, OracleImpl, rel_err, spectral_scaled

IMPLS = [pytest.param("oracle"), pytest.param("gpu", marks=pytest.mark.gpu)]
U = 2.0 ** -53


@pytest.fixture(params=IMPLS)
def impl(request):
    return OracleImpl() if request.param == "oracle" else GpuImpl()


def test_zero_operator_columns(impl):  # test_phi_block.cpp:177-194
    V = O.Rng(181).matrix(5, 3)
    G = impl.series_direct(impl.op(np.zeros((5, 5))), [0.5, 2.0], [1.0, -2.0], V, -1.0)
    for k, a in enumerate([1.0, -2.0]):
        want = V[:, 0] + a * V[:, 1] + a * a * V[:, 2] / 2.0
        assert rel_err(G[:, k], want) < 1e-14


def test_p0_exponential_columns(impl):  # :195-212
    rng = O.Rng(191)
    A = rng.matrix(5, 5)
    A = A * (1.0 / np.linalg.svd(A, compute_uv=False)[0])
    v0 = rng.matrix(5, 1)
    G = impl.series_direct(impl.op(A), [0.4, 1.0], [1.0, 1.0], v0, -1.0)
    for i, t in enumerate([0.4, 1.0]):
        assert rel_err(G[:, i], O.reference_w(A, v0, t, 1.0)) < 1e-13


def test_equal_alphas_collapse(impl):  # :213-229
    rng = O.Rng(193)
    A = spectral_scaled(rng.matrix(6, 6), 0.8)
    V = rng.matrix(6, 3)
    G = impl.series_direct(impl.op(A), [0.7] * 3, [1.4] * 3, V, -1.0)
    assert np.abs(G[:, 0] - G[:, 1]).max() == 0.0
    assert rel_err(G[:, 0], O.reference_w(A, V, 0.7, 1.4)) < 1e-13


def test_slow_series_is_reported(impl):  # :230-243
    rng = O.Rng(199)
    A = spectral_scaled(rng.matrix(6, 6), 400.0)
    with pytest.raises(RuntimeError):
        impl.series_direct(impl.op(A), [1.0], [1.0], rng.matrix(6, 2), -1.0)


def test_cross_checks_scaled_evaluator(impl):  # :245-262
    rng = O.Rng(197)
    A = spectral_scaled(rng.matrix(7, 7), 2.0)
    V = rng.matrix(7, 4)
    t, alpha, tol = [0.5, 1.0], [1.0, 0.5], 1e-13
    op = impl.op(A)
    G = impl.series_direct(op, t, alpha, V, tol)
    W, _ = impl.phimv_block(op, t, alpha, V, tol, impl.select_parameters(op, 61, tol))
    assert rel_err(G, W) < 1e-11


def test_coefficient_table_matches_phi_coeffs():
    """An explicit a_ij table equal to phi_series_coeffs gives the same bits."""
    import paper_2509_26475_b200 as P
    rng = O.Rng(211)
    A = spectral_scaled(rng.matrix(6, 6), 0.5)
    V = rng.matrix(6, 3)
    op = O.csr_from_dense(A)
    G0 = O.block_series_direct(op, [0.3, 0.9], [1.0, 2.0], V, -1.0)
    G1 = O.block_series_direct(op, [0.3, 0.9], [1.0, 2.0], V, -1.0, P.phi_series_coeffs(2, 200))
    assert np.array_equal(G0, G1)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,size,tscale", [(2, 24, 1e-3), (1, 200, 1e-2), (4, 4096, 1e-3),
                                            (5, 3000, 1e-2)])
def test_gpu_bitwise_vs_oracle(cfg, size, tscale):
    import paper_2509_26475_b200 as P
    wl = P.workload(cfg, size)
    o, g = OracleImpl(), GpuImpl()
    # a short horizon so the direct series converges: t scaled down
    h = 1.0 / max(1.0, float(np.abs(wl.av).max()))
    t = wl.t / np.abs(wl.t).max() * tscale * h * 50.0
    Go = o.series_direct(o.op_csr(wl.n, wl.rp, wl.ci, wl.av), t, wl.alpha, wl.V, wl.tol)
    Gg = g.series_direct(g.op_csr(wl.n, wl.rp, wl.ci, wl.av), t, wl.alpha, wl.V, wl.tol)
    assert np.array_equal(Gg, Go)
