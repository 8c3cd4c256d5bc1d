"""Seeded randomized parity sweep of the CUDA path against the oracle.

Each case draws a CSR operator: size, row lengths, empty rows, unsorted and
duplicate columns, diagonal dominance or not, and a spectral scale. It also
draws a block request: p, r, t of either sign, alpha, and tol. The CUDA path
must reproduce the oracle bitwise: ScalingShift, RunRecord (s_eff, L_S, every
L_F, matvecs) and W. A second draw checks `phimv` the same way. Sizes stay
where the oracle finishes in well under a second per case.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def P():
    import paper_2509_26475_b200 as P_
    return P_


def _draw_operator(rng):
    n = int(rng.choice([1, 7, 64, 300, 1000, 2047]))
    kmax = int(rng.integers(0, 9))
    dominant = bool(rng.integers(0, 2))
    scale = float(10.0 ** rng.uniform(-1, 3))
    rp = [0]
    ci, av = [], []
    for i in range(n):
        if n > 8 and rng.random() < 0.03:
            rp.append(len(ci))  # empty row
            continue
        k = int(rng.integers(0, kmax + 1))
        cols = list(rng.integers(0, n, size=k))
        if k and rng.random() < 0.1:
            cols.append(cols[0])  # duplicate entry
        if rng.random() < 0.9:
            cols.append(i)
        rng.shuffle(cols)
        vals = rng.standard_normal(len(cols)) * scale
        if dominant:
            for j, c in enumerate(cols):
                if c == i:
                    vals[j] = -(np.abs(vals).sum() + scale)
        ci += [int(c) for c in cols]
        av += vals.tolist()
        rp.append(len(ci))
    return (n, np.array(rp, dtype=np.int64), np.array(ci, dtype=np.int32),
            np.array(av, dtype=np.float64))


def _draw_request(rng, n):
    p = int(rng.integers(0, 6))
    r = int(rng.integers(1, 9))
    sign = -1.0 if rng.random() < 0.25 else 1.0
    t = sign * 10.0 ** rng.uniform(-3, 0.3, size=r)
    alpha = rng.uniform(-2, 2, size=r)
    tol = float(rng.choice([1e-6, 1e-10, 2.0 ** -53]))
    V = O.Rng(int(rng.integers(1, 1 << 30))).matrix(n, p + 1)
    return p, r, t, alpha, tol, V


@pytest.mark.parametrize("seed", range(64))
def test_random_block_bitwise(seed):
    P_ = P()
    rng = np.random.default_rng(1000 + seed)
    n, rp, ci, av = _draw_operator(rng)
    op = P_.CsrOperator(n, rp, ci, av)
    oop = O.csr_from_arrays(n, rp, ci, av)
    p, r, t, alpha, tol, V = _draw_request(rng, n)
    sso = O.select_parameters(oop, 61, tol)
    ss = P_.select_parameters(op, 61, tol)
    assert ss.astuple() == sso.astuple()
    if sso.s * float(np.max(np.abs(t))) > 400.0:  # keep the oracle's sweeps bounded
        t = t * (400.0 / (sso.s * float(np.max(np.abs(t)))))
    try:
        Wo, ro = O.phimv_block(oop, t, alpha, V, tol, sso)
    except Exception as e:  # the same error, with the reference's message
        with pytest.raises(Exception) as got:
            P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, ss))
        assert str(got.value) == str(e)
        return
    res = P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, ss))
    st = res.stats
    assert (st.s_effective, st.series_len_S, st.matvecs) == (ro.s_effective, ro.series_len_S,
                                                             ro.matvecs)
    assert st.series_lens_F == ro.series_lens_F
    assert np.array_equal(res.W, Wo)


@pytest.mark.parametrize("seed", range(16))
def test_random_single_bitwise(seed):
    P_ = P()
    rng = np.random.default_rng(5000 + seed)
    n, rp, ci, av = _draw_operator(rng)
    op = P_.CsrOperator(n, rp, ci, av)
    oop = O.csr_from_arrays(n, rp, ci, av)
    p, _, t, alpha, tol, V = _draw_request(rng, n)
    sso = O.select_parameters(oop, 61, tol)
    t0 = float(t[0])
    if sso.s * abs(t0) > 400.0:
        t0 = t0 * 400.0 / (sso.s * abs(t0))
    try:
        w, e0, tail, rec = O.phimv(oop, t0, float(alpha[0]), V, tol, sso)
    except Exception as e:
        with pytest.raises(Exception) as got:
            P_.phimv(op, P_.PhiRequest(t0, float(alpha[0]), V, tol, P_.ScalingShift(*sso.astuple())))
        assert str(got.value) == str(e)
        return
    res = P_.phimv(op, P_.PhiRequest(t0, float(alpha[0]), V, tol, P_.ScalingShift(*sso.astuple())))
    assert (res.stats.s_effective, res.stats.series_len_S) == (rec.s_effective, rec.series_len_S)
    assert res.stats.series_lens_F == rec.series_lens_F
    assert np.array_equal(res.w, w)
    assert np.array_equal(res.exp_v0, e0) and np.array_equal(res.tail, tail)


@pytest.mark.parametrize("seed", range(16))
def test_random_partitioned_bitwise(seed):
    """The row-partitioned operator (2-5 parts on one device) on the same draws:
    selection and evaluation stay the oracle's."""
    P_ = P()
    parts = 2 + seed % 4
    for attempt in range(20):  # a draw with at least 4 rows per part
        rng = np.random.default_rng(9000 + seed + 1000 * attempt)
        n, rp, ci, av = _draw_operator(rng)
        if n >= 4 * parts:
            break
    op = P_.CsrOperator(n, rp, ci, av, parts=parts)
    oop = O.csr_from_arrays(n, rp, ci, av)
    p, r, t, alpha, tol, V = _draw_request(rng, n)
    sso = O.select_parameters(oop, 61, tol)
    ss = P_.select_parameters(op, 61, tol)
    assert ss.astuple() == sso.astuple()
    if sso.s * float(np.max(np.abs(t))) > 400.0:
        t = t * (400.0 / (sso.s * float(np.max(np.abs(t)))))
    try:
        Wo, ro = O.phimv_block(oop, t, alpha, V, tol, sso)
    except Exception as e:
        with pytest.raises(Exception) as got:
            P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, ss))
        assert str(got.value) == str(e)
        return
    res = P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, ss))
    assert (res.stats.s_effective, res.stats.series_len_S) == (ro.s_effective, ro.series_len_S)
    assert res.stats.series_lens_F == ro.series_lens_F
    assert np.array_equal(res.W, Wo)
