"""GPU parity of the bulk-copy evaluator (csrc/phx_bulk.cu: tile plan +
warp-specialised cp.async.bulk pipeline), forced with PHX_BULK=1 on small
operators so every path runs: offset groups (3D / 2D stencils), singles
(random far columns), window-only rows with hundreds of recovery sweeps
(C5), the single-combination variant, trace mode, and the fallback when an
operator has no plan.  The bar is the same as for k_phimv_block: bitwise
the oracle."""
import json
import os

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


def bulk_used():
    return P().last_eval_variant()["dynamic_tail"] == 2


@pytest.mark.parametrize("name", ["cfg1_s200", "cfg2_s64", "cfg3_s12", "cfg5_s2000", "cfg1_s1000"])
def test_fixture_bitwise_bulk(golden_dir, name):
    with open(os.path.join(golden_dir, name + ".json")) as f:
        meta = json.load(f)
    arr = np.load(os.path.join(golden_dir, name + ".npz"))
    p = P()
    wl = p.workload(meta["cfg"], meta["size"])
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(op, 61, wl.tol)
    p.set_trace(3 * 400000)
    res = p.phimv_block(op, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    tr = p.get_trace(3 * 400000)
    p.set_trace(0)
    assert bulk_used()
    st = res.stats
    assert (st.s_effective, st.series_len_S, st.series_lens_F, st.matvecs) == (
        meta["s_effective"], meta["series_len_S"], meta["series_lens_F"], meta["matvecs"])
    assert np.array_equal(tr, arr["trace"])
    assert np.array_equal(res.W, arr["W"])


@pytest.mark.parametrize("cfg,size", [(3, 24), (3, 41), (2, 200), (5, 1 << 14)])
def test_configs_bitwise_bulk(cfg, size):
    """C3 (four offset groups), C2 (two), C5 (window only, recovery sweeps) at
    sizes with thousands of tiles and a ragged last tile."""
    p = P()
    wl = p.workload(cfg, size)
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    ss = O.select_parameters(oop, 61, wl.tol)
    Wo, ro = O.phimv_block(oop, wl.t, wl.alpha, wl.V, wl.tol, ss)
    res = p.phimv_block(op, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol,
                                              p.ScalingShift(*ss.astuple())))
    assert bulk_used()
    assert (res.stats.series_len_S, res.stats.series_lens_F) == (ro.series_len_S, ro.series_lens_F)
    assert np.array_equal(res.W, Wo)


def _banded_with_far(n, seed, far_prob, scale):
    rng = np.random.default_rng(seed)
    rp, ci, av = [0], [], []
    for i in range(n):
        cols = {i} | {c for c in (i - 1, i + 1, i - 40, i + 97) if 0 <= c < n}
        if rng.random() < far_prob:
            cols.add(int(rng.integers(0, n)))
        cols = sorted(cols)
        vals = rng.standard_normal(len(cols))
        vals[cols.index(i)] = -(np.abs(vals).sum() + 1.0)
        ci += cols
        av += (vals * scale).tolist()
        rp.append(len(ci))
    return n, np.array(rp), np.array(ci, dtype=np.int32), np.array(av)


@pytest.mark.parametrize("p_,r", [(3, 4), (4, 6), (1, 8), (0, 6), (7, 8), (1, 2)])
def test_groups_and_singles_bitwise_bulk(p_, r):
    """Offset groups (-40, +97) plus random far columns staged as single rows;
    even widths (p+1) r <= 64, with recovery sweeps."""
    P_ = P()
    n, rp, ci, av = _banded_with_far(20011, 50 + p_ + r, 0.25, 20.0)
    info, *_ = P_.tile_plan(n, rp, ci)
    assert info["ok"] and info["singles"] > 0
    op = P_.CsrOperator(n, rp, ci, av)
    oop = O.csr_from_arrays(n, rp, ci, av)
    tol = 1e-10
    ss = O.select_parameters(oop, 61, tol)
    rng = O.Rng(7 + p_ + r)
    V = rng.matrix(n, p_ + 1)
    t = (0.5 + rng.uniforms(r)) * (2.5 / ss.s)
    alpha = -1.0 + 2.0 * rng.uniforms(r)
    Wo, ro = O.phimv_block(oop, t, alpha, V, tol, ss)
    res = P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, P_.ScalingShift(*ss.astuple())))
    assert bulk_used()
    assert ro.s_effective > 1
    assert (res.stats.series_len_S, res.stats.series_lens_F) == (ro.series_len_S, ro.series_lens_F)
    assert np.array_equal(res.W, Wo)


@pytest.mark.parametrize("p_,r", [(4, 6), (3, 8), (2, 6), (1, 8), (1, 6), (2, 10)])
def test_specialised_consumers_bitwise(p_, r, monkeypatch):
    """The specialised S-term consumer (16 < w <= 32, r even, xi != 0) and the
    specialised recovery-term consumer (8 < 2r <= 16) against the oracle and
    against the general consumers (PHX_BULK_FLAGS bit 2 switches them off):
    groups, single rows, a ragged last tile, recovery sweeps."""
    P_ = P()
    n, rp, ci, av = _banded_with_far(20011 + 7 * r, 90 + p_ + r, 0.2, 20.0)
    op = P_.CsrOperator(n, rp, ci, av)
    oop = O.csr_from_arrays(n, rp, ci, av)
    tol = 1e-10
    ss = O.select_parameters(oop, 61, tol)
    assert ss.xi != 0.0
    rng = O.Rng(17 + p_ + r)
    V = rng.matrix(n, p_ + 1)
    t = (0.5 + rng.uniforms(r)) * (2.5 / ss.s)
    alpha = -1.0 + 2.0 * rng.uniforms(r)
    Wo, ro = O.phimv_block(oop, t, alpha, V, tol, ss)
    req = P_.BlockPhiRequest(t, alpha, V, tol, P_.ScalingShift(*ss.astuple()))
    res = P_.phimv_block(op, req)
    assert bulk_used()
    assert ro.s_effective > 1
    assert (res.stats.series_len_S, res.stats.series_lens_F) == (ro.series_len_S, ro.series_lens_F)
    assert np.array_equal(res.W, Wo)
    monkeypatch.setenv("PHX_BULK_FLAGS", "6")  # the general consumers
    gen = P_.phimv_block(op, req)
    assert bulk_used()
    assert np.array_equal(gen.W, Wo)


def test_specialised_consumers_window_only_plan(monkeypatch):
    """A banded operator whose plan merges tiles per stage (window-only, C5's
    shape) with w = 32 and fc = 16: both specialised consumers on merged stages."""
    P_ = P()
    wl = P_.workload(5, (1 << 13) + 77)
    op = P_.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    ss = O.select_parameters(oop, 61, wl.tol)
    Wo, ro = O.phimv_block(oop, wl.t, wl.alpha, wl.V, wl.tol, ss)
    req = P_.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, P_.ScalingShift(*ss.astuple()))
    res = P_.phimv_block(op, req)
    assert bulk_used()
    assert (res.stats.series_len_S, res.stats.series_lens_F) == (ro.series_len_S, ro.series_lens_F)
    assert np.array_equal(res.W, Wo)
    monkeypatch.setenv("PHX_BULK_FLAGS", "6")
    assert np.array_equal(P_.phimv_block(op, req).W, Wo)


def test_single_variant_bulk():
    """phimv (Alg. 2, r = 1): w, exp_v0 and the tail through the bulk kernel."""
    P_ = P()
    n, rp, ci, av = _banded_with_far(9001, 5, 0.1, 20.0)
    op = P_.CsrOperator(n, rp, ci, av)
    oop = O.csr_from_arrays(n, rp, ci, av)
    tol = 1e-12
    ss = O.select_parameters(oop, 61, tol)
    V = O.Rng(12).matrix(n, 4)
    t = 3.5 / ss.s
    w, e0, tail, rec = O.phimv(oop, t, 0.75, V, tol, ss)
    res = P_.phimv(op, P_.PhiRequest(t, 0.75, V, tol, P_.ScalingShift(*ss.astuple())))
    assert bulk_used()
    assert rec.s_effective > 1
    assert res.stats.series_lens_F == rec.series_lens_F
    assert np.array_equal(res.w, w)
    assert np.array_equal(res.exp_v0, e0) and np.array_equal(res.tail, tail)


def test_no_plan_falls_back():
    """An operator whose tiles exceed the stage (here > 1024 entries in one
    tile) has no plan: the evaluation runs k_phimv_block, still bitwise."""
    P_ = P()
    n, rp, ci, av = _banded_with_far(3000, 9, 0.0, 5.0)
    rows = [list(ci[rp[i]:rp[i + 1]]) for i in range(n)]
    vals = [list(av[rp[i]:rp[i + 1]]) for i in range(n)]
    rows[100] = sorted(set(range(0, 3000, 2)) | {100})
    vals[100] = [(-4000.0 if c == 100 else 1.0) for c in rows[100]]
    rp = np.concatenate([[0], np.cumsum([len(x) for x in rows])])
    ci = np.array([c for x in rows for c in x], dtype=np.int32)
    av = np.array([v for x in vals for v in x])
    assert P_.tile_plan(n, rp, ci)[0]["ok"] == 0
    op = P_.CsrOperator(n, rp, ci, av)
    oop = O.csr_from_arrays(n, rp, ci, av)
    tol = 1e-10
    ss = O.select_parameters(oop, 61, tol)
    V = O.Rng(3).matrix(n, 2)
    t = np.array([0.5, 1.0]) / ss.s
    alpha = np.array([1.0, -1.0])
    Wo, ro = O.phimv_block(oop, t, alpha, V, tol, ss)
    res = P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, P_.ScalingShift(*ss.astuple())))
    assert not bulk_used()
    assert np.array_equal(res.W, Wo)


def test_odd_width_falls_back():
    """C4's width (p+1) r = 9 is odd (scalar lanes): k_phimv_block runs."""
    p = P()
    wl = p.workload(4, 4096)
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(op, 61, wl.tol)
    p.phimv_block(op, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    assert not bulk_used()


def test_bulk_repeatable_and_equal_to_grid_kernel(monkeypatch):
    """The bulk kernel three times and the register-gather kernel once on a
    C3-shaped operator: four bit-identical W (no race in the ring protocol)."""
    p = P()
    wl = p.workload(3, 48)
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(op, 61, wl.tol)
    req = p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)
    Ws = [p.phimv_block(op, req).W for _ in range(3)]
    monkeypatch.setenv("PHX_BULK", "0")
    W0 = p.phimv_block(op, req).W
    assert not bulk_used()
    for W in Ws:
        assert np.array_equal(W, W0)
