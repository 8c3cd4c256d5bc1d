"""Seeded randomized parity sweep of the bulk-copy evaluator (PHX_BULK=1)
and of its row-partitioned instantiation against the oracle.

Each case draws a banded operator the tile plan accepts: a few offset
diagonals (they become offset groups or stay in the window), rare far
entries (single rows), empty rows, duplicate and unsorted columns, a random
spectral scale; and a request with both block widths even (the bulk
kernel's double2 lanes): p, r, t of either sign, alpha, tol.  ScalingShift,
RunRecord and W must be the oracle's bit for bit."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def force_bulk(monkeypatch):
    monkeypatch.setenv("PHX_BULK", "1")


def P():
    import paper_2509_26475_b200 as mod
    return mod


def _draw_operator(rng):
    n = int(rng.choice([40, 333, 1000, 2500, 4097]))
    offs = sorted(set(int(o) for o in rng.choice([-257, -64, -33, -1, 1, 33, 64, 257],
                                                   size=int(rng.integers(1, 5)))))
    scale = float(10.0 ** rng.uniform(-1, 2.5))
    rp, ci, av = [0], [], []
    for i in range(n):
        if rng.random() < 0.02:
            rp.append(len(ci))  # empty row
            continue
        cols = [i + o for o in offs if 0 <= i + o < n]
        if rng.random() < 0.05:
            cols.append(int(rng.integers(0, n)))  # a far entry (single row)
        if cols and rng.random() < 0.05:
            cols.append(cols[0])  # duplicate
        cols.append(i)
        if rng.random() < 0.3:
            rng.shuffle(cols)
        vals = rng.standard_normal(len(cols)) * scale
        for j, c in enumerate(cols):
            if c == i:
                vals[j] = -(np.abs(vals).sum() + scale)
        ci += [int(c) for c in cols]
        av += vals.tolist()
        rp.append(len(ci))
    return (n, np.array(rp, dtype=np.int64), np.array(ci, dtype=np.int32),
            np.array(av, dtype=np.float64))


def _draw_request(rng, n):
    while True:
        p = int(rng.integers(0, 5))
        r = int(rng.integers(1, 9))
        w, fc = (p + 1) * r, (r if p == 0 else 2 * r)
        if w % 2 == 0 and fc % 2 == 0 and w <= 64:
            break
    sign = -1.0 if rng.random() < 0.25 else 1.0
    t = sign * 10.0 ** rng.uniform(-3, 0.3, size=r)
    alpha = rng.uniform(-2, 2, size=r)
    tol = float(rng.choice([1e-6, 1e-10, 2.0 ** -53]))
    V = O.Rng(int(rng.integers(1, 1 << 30))).matrix(n, p + 1)
    return p, r, t, alpha, tol, V


def _case(seed, parts):
    P_ = P()
    rng = np.random.default_rng(seed)
    n, rp, ci, av = _draw_operator(rng)
    op = P_.CsrOperator(n, rp, ci, av, parts=parts) if parts > 1 else P_.CsrOperator(n, rp, ci, av)
    oop = O.csr_from_arrays(n, rp, ci, av)
    p, r, t, alpha, tol, V = _draw_request(rng, n)
    sso = O.select_parameters(oop, 61, tol)
    ss = P_.select_parameters(op, 61, tol)
    assert ss.astuple() == sso.astuple()
    if sso.s * float(np.max(np.abs(t))) > 300.0:  # keep the oracle's sweeps bounded
        t = t * (300.0 / (sso.s * float(np.max(np.abs(t)))))
    try:
        Wo, ro = O.phimv_block(oop, t, alpha, V, tol, sso)
    except Exception as e:  # the same error, with the reference's message
        with pytest.raises(Exception) as got:
            P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, ss))
        assert str(got.value) == str(e)
        return None
    res = P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, ss))
    var = P_.last_eval_variant()
    st = res.stats
    assert (st.s_effective, st.series_len_S, st.matvecs) == (ro.s_effective, ro.series_len_S,
                                                             ro.matvecs)
    assert st.series_lens_F == ro.series_lens_F
    assert np.array_equal(res.W, Wo)
    return var


@pytest.mark.parametrize("seed", range(96))
def test_random_bulk_bitwise(seed):
    var = _case(20000 + seed, 1)
    if var is not None:
        assert var["dynamic_tail"] == 2  # the bulk kernel ran


@pytest.mark.parametrize("seed", range(32))
def test_random_bulk_partitioned_bitwise(seed):
    _case(30000 + seed, 2 + seed % 3)


@pytest.mark.parametrize("seed,parts", [(50098, 1), (50153, 1), (50192, 2)])
def test_ring_sizes_next_to_the_shared_memory_limit(seed, parts):
    """Draws whose deepest candidate ring fits the opt-in shared-memory limit
    by itself but not together with the kernel's static shared memory: the
    ring search must take the next candidate (it once failed the evaluation
    with `invalid argument`; found by tools/tools_fuzz_extended.py)."""
    _case(seed, parts)
