"""GPU parity: the CUDA path (libphx.so through its C ABI) against the CPU
oracle and the committed golden fixtures.  The bar is bit-for-bit equality
of ScalingShift, RunRecord, the per-step stopping-test trace and W (the
device path is designed to reproduce the oracle's operation order exactly,
DESIGN.md §3); where only a property can be checked at full size, the test
says so."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

SMALL = ["cfg1_s200", "cfg2_s64", "cfg3_s12", "cfg4_s1024", "cfg5_s2000", "cfg1_s1000"]


def P():
    import paper_2509_26475_b200 as mod
    return mod


def sha(a):
    return hashlib.sha256(np.asfortranarray(a, dtype=np.float64).tobytes(order="F")).hexdigest()


def load(golden_dir, name):
    with open(os.path.join(golden_dir, name + ".json")) as f:
        meta = json.load(f)
    return meta, np.load(os.path.join(golden_dir, name + ".npz"))


def gpu_eval(wl, trace=False):
    p = P()
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(op, 61, wl.tol)
    p.set_trace(3 * 400000 if trace else 0)
    res = p.phimv_block(op, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    tr = p.get_trace(3 * 400000) if trace else None
    p.set_trace(0)
    return op, ss, res, tr


@pytest.mark.parametrize("name", SMALL)
def test_fixture_bitwise(golden_dir, name):
    meta, arr = load(golden_dir, name)
    wl = P().workload(meta["cfg"], meta["size"])
    op, ss, res, tr = gpu_eval(wl, trace=True)
    assert list(ss.astuple()) == meta["params"]
    st = res.stats
    assert (st.s_effective, st.series_len_S, st.series_lens_F, st.matvecs) == (
        meta["s_effective"], meta["series_len_S"], meta["series_lens_F"], meta["matvecs"])
    assert np.array_equal(tr, arr["trace"])
    assert np.array_equal(res.W, arr["W"])
    assert sha(res.W) == meta["W_sha256"]


@pytest.mark.parametrize("cfg", [2, 4, 3])
def test_full_size_bitwise(golden_dir, cfg):
    """BASELINE full sizes (C2 n=2^20, C4 n=2^22, C3 n=2^24) against the
    oracle's SHA-256 of W and its sampled rows."""
    name = f"full_cfg{cfg}"
    if not os.path.exists(os.path.join(golden_dir, name + ".json")):
        pytest.skip("full-size fixture not generated")
    meta, arr = load(golden_dir, name)
    wl = P().workload(cfg, 0)
    op, ss, res, _ = gpu_eval(wl)
    assert list(ss.astuple()) == meta["params"]
    assert res.stats.series_len_S == meta["series_len_S"]
    assert res.stats.matvecs == meta["matvecs"]
    assert np.array_equal(res.W[arr["sample_rows"]], arr["sample_W"])
    assert sha(res.W) == meta["W_sha256"]


def test_repeatable_full_c2():
    """Three evaluations of the full C2 block are bit-identical (no races in
    the persistent kernel's staging / slot protocol)."""
    p = P()
    wl = p.workload(2, 0)
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(op, 61, wl.tol)
    Ws = [p.phimv_block(op, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)).W
          for _ in range(3)]
    assert np.array_equal(Ws[0], Ws[1]) and np.array_equal(Ws[1], Ws[2])


def test_device_api_matches_host_api():
    import torch
    p = P()
    wl = p.workload(2, 128)
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(op, 61, wl.tol)
    W = p.phimv_block(op, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)).W
    dV = torch.from_numpy(np.ascontiguousarray(wl.V.T)).cuda()
    dW = torch.empty((wl.r, wl.n), dtype=torch.float64, device="cuda")
    rec = p.phimv_block_device(op, wl.t, wl.alpha, wl.p, dV.data_ptr(), wl.tol, ss, dW.data_ptr())
    assert np.array_equal(dW.cpu().numpy().T, W)
    assert rec.series_len_S > 1


def test_leading_dimensions():
    """Host V / W with leading dimensions larger than n (Eigen blocks of a
    bigger matrix)."""
    import ctypes as C
    p = P()
    wl = p.workload(1, 300)
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(op, 61, wl.tol)
    W = p.phimv_block(op, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)).W
    ld = wl.n + 7
    Vp = np.zeros((ld, wl.p + 1), order="F")
    Vp[: wl.n] = wl.V
    Wp = np.full((ld, wl.r), np.nan, order="F")
    t = np.ascontiguousarray(wl.t)
    a = np.ascontiguousarray(wl.alpha)
    c = ss._c()
    code = p.lib().phx_phimv_block(op._h, wl.r, t.ctypes.data_as(p.dp), a.ctypes.data_as(p.dp),
                                   wl.p, Vp.ctypes.data_as(p.dp), ld, wl.tol, C.byref(c),
                                   Wp.ctypes.data_as(p.dp), ld, None)
    p._check(code)
    assert np.array_equal(Wp[: wl.n], W)
    assert np.all(np.isnan(Wp[wl.n:]))


def test_apply_bitwise():
    """CSR apply / shifted_apply (linop.cpp:10-49) equal the oracle's ApplyFn."""
    p = P()
    wl = p.workload(4, 2048)
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    X = O.Rng(5).matrix(wl.n, 3)
    assert np.array_equal(op.apply(X), O.apply(oop, X))
    Y = op.shifted_apply(0.75, X)
    want = O.apply(oop, X) - 0.75 * X
    assert np.array_equal(Y, want)
    assert np.array_equal(op.shifted_apply(0.0, X), O.apply(oop, X))


def test_selection_parts_bitwise():
    """build_power_basis / objective / Brent path / parameters_for_shift
    against the oracle, with the Brent trial points compared one by one."""
    p = P()
    wl = p.workload(3, 16)
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    b = p.build_power_basis(op)
    ob = O.build_power_basis(oop)
    assert (b.r, b.m, b.s0) == (ob.r, ob.m, ob.s0)
    assert np.array_equal(b.logs, ob.logs)
    assert np.array_equal(b.columns, ob.columns)
    for xi in (0.0, -3.5, 17.25, -ob.s0):
        assert p.objective(b, xi) == ob.objective(xi)
    xi, fm, path = p.minimize_shift(b, with_path=True)
    oxi, ofm, opath = ob.minimize_shift(with_path=True)
    assert np.array_equal(path, opath)
    assert (xi, fm) == (oxi, ofm)
    assert p.parameters_for_shift(op, b, xi, 1e-9).astuple() == ob.parameters_for_shift(xi, 1e-9).astuple()


def test_c5_large_linearity_and_duplicates():
    """C5 (nonnormal bidiagonal) at n = 2^18: properties that hold at any size
    — linearity in V and identical columns for duplicated (t, alpha) — on a
    run with hundreds of recovery sweeps."""
    p = P()
    wl = p.workload(5, 1 << 18)
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(op, 61, wl.tol)
    t = np.array([wl.t[3], wl.t[3], 0.05])
    a = np.array([wl.alpha[3], wl.alpha[3], 0.5])
    V1 = wl.V
    V2 = np.asfortranarray(np.roll(wl.V, 7, axis=0))
    W1 = p.phimv_block(op, p.BlockPhiRequest(t, a, V1, wl.tol, ss))
    W2 = p.phimv_block(op, p.BlockPhiRequest(t, a, V2, wl.tol, ss)).W
    W12 = p.phimv_block(op, p.BlockPhiRequest(t, a, V1 + V2, wl.tol, ss)).W
    assert W1.stats.s_effective > 1
    assert np.array_equal(W1.W[:, 0], W1.W[:, 1])
    lhs, rhs = W12, W1.W + W2
    rel = np.linalg.norm(lhs - rhs) / np.linalg.norm(lhs)
    assert rel <= 1e3 * wl.tol, rel


def test_kernel_actually_runs():
    p = P()
    before = p.kernel_launches()
    wl = p.workload(2, 32)
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(op, 61, wl.tol)
    p.phimv_block(op, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    assert p.kernel_launches() > before
    ms, steps = p.last_eval_stats()
    assert ms > 0 and steps >= 2


def _random_sparse(n, k, seed):
    """n x n CSR with k off-diagonal entries per row + a dominant diagonal."""
    rng = np.random.default_rng(seed)
    rp = [0]
    ci, av = [], []
    for i in range(n):
        cols = sorted(set(rng.integers(0, n, size=k).tolist()) | {i})
        vals = rng.standard_normal(len(cols))
        vals[cols.index(i)] = -(np.abs(vals).sum() + 2.0)
        ci += cols
        av += vals.tolist()
        rp.append(len(ci))
    return n, np.array(rp, dtype=np.int64), np.array(ci, dtype=np.int32), np.array(av)


@pytest.mark.parametrize("p,r", [(9, 8), (4, 7), (15, 16), (0, 5), (1, 1), (2, 40), (3, 33)])
def test_block_widths_bitwise(p, r):
    """Every evaluator variant: V = 1/2 columns per lane, Q = 1..8 column
    chunks, p = 0 (F width r) and wide F widths, with recovery sweeps."""
    P_ = P()
    n, rp, ci, av = _random_sparse(700, 4, 1000 + 17 * p + r)
    av = av * 25.0  # ||A|| large enough for recovery sweeps
    op = P_.CsrOperator(n, rp, ci, av)
    oop = O.csr_from_arrays(n, rp, ci, av)
    rng = O.Rng(31 + p + r)
    V = rng.matrix(n, p + 1)
    t = 0.05 + 0.4 * rng.uniforms(r)
    alpha = -1.0 + 2.0 * rng.uniforms(r)
    tol = 1e-12
    ss = O.select_parameters(oop, 61, tol)
    ss.s *= 4.0  # force recovery sweeps
    Wo, ro = O.phimv_block(oop, t, alpha, V, tol, ss)
    res = P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, P_.ScalingShift(*ss.astuple())))
    assert ro.s_effective > 1
    assert res.stats.series_len_S == ro.series_len_S
    assert res.stats.series_lens_F == ro.series_lens_F
    assert np.array_equal(res.W, Wo)


def test_single_variant_with_recovery_bitwise():
    P_ = P()
    wl = P_.workload(5, 3000)
    op = P_.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    ss = O.select_parameters(oop, 61, wl.tol)
    w, e0, tail, rec = O.phimv(oop, 2.0, 0.75, wl.V, wl.tol, ss)
    res = P_.phimv(op, P_.PhiRequest(2.0, 0.75, wl.V, wl.tol, P_.ScalingShift(*ss.astuple())))
    assert rec.s_effective > 1
    assert res.stats.series_lens_F == rec.series_lens_F
    assert np.array_equal(res.w, w) and np.array_equal(res.exp_v0, e0) and np.array_equal(res.tail, tail)


def test_irregular_csr_bitwise():
    """Legal but irregular CSR: unsorted columns, duplicate column entries,
    empty rows, explicit zeros, one dense row (> the staged-entry capacity,
    the global-memory gather path).  Rows accumulate in storage order on both
    sides, so selection, the run record and W stay bitwise the oracle's."""
    P_ = P()
    rng = np.random.default_rng(77)
    n = 900
    rows = []
    for i in range(n):
        if i % 37 == 5:
            rows.append([])                                        # empty row
            continue
        k = int(rng.integers(1, 7))
        cols = list(rng.integers(0, n, size=k))
        if i % 11 == 0:
            cols.append(cols[0])                                   # duplicate entry
        cols.append(i)
        rng.shuffle(cols)                                          # unsorted
        rows.append(cols)
    rows[450] = list(rng.permutation(n)[:400]) + [450]             # one very long row
    rp = np.zeros(n + 1, dtype=np.int64)
    ci, av = [], []
    for i, cols in enumerate(rows):
        for c in cols:
            ci.append(int(c))
            av.append(0.0 if (len(av) % 53 == 7) else float(rng.standard_normal()) * (
                -8.0 if c == i else 1.0))
        rp[i + 1] = len(ci)
    ci = np.array(ci, dtype=np.int32)
    av = np.array(av)
    op = P_.CsrOperator(n, rp, ci, av)
    oop = O.csr_from_arrays(n, rp, ci, av)
    X = O.Rng(5).matrix(n, 3)
    assert np.array_equal(op.apply(X), O.apply(oop, X))
    tol = 1e-12
    ss = P_.select_parameters(op, 61, tol)
    sso = O.select_parameters(oop, 61, tol)
    assert ss.astuple() == sso.astuple()
    V = O.Rng(6).matrix(n, 3)
    t = np.array([0.1, 0.7, 1.3])
    alpha = np.array([1.0, -0.5, 2.0])
    Wo, ro = O.phimv_block(oop, t, alpha, V, tol, sso)
    res = P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, ss))
    assert (res.stats.s_effective, res.stats.series_len_S) == (ro.s_effective, ro.series_len_S)
    assert res.stats.series_lens_F == ro.series_lens_F
    assert np.array_equal(res.W, Wo)


@pytest.mark.parametrize("n", [1, 2, 3, 31, 33, 257, 4099])
def test_tiny_and_ragged_operators_bitwise(n):
    """Operators smaller than one tile, one row past a tile, and sizes that
    leave a partial last tile (latency mode below the SM count, the
    persistent grid above): selection, run record and W stay the oracle's."""
    P_ = P()
    n_, rp, ci, av = _random_sparse(n, min(3, n), 4242 + n)
    op = P_.CsrOperator(n_, rp, ci, av)
    oop = O.csr_from_arrays(n_, rp, ci, av)
    tol = 1e-12
    ss = P_.select_parameters(op, 61, tol)
    sso = O.select_parameters(oop, 61, tol)
    assert ss.astuple() == sso.astuple()
    rng = O.Rng(9 + n)
    V = rng.matrix(n_, 3)
    t = np.array([0.3, 1.1, 2.5])
    alpha = np.array([0.5, 1.0, -1.5])
    Wo, ro = O.phimv_block(oop, t, alpha, V, tol, sso)
    res = P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, ss))
    assert (res.stats.s_effective, res.stats.series_len_S) == (ro.s_effective, ro.series_len_S)
    assert res.stats.series_lens_F == ro.series_lens_F
    assert np.array_equal(res.W, Wo)


def test_block_width_limit():
    """(p+1)*r above the widest variant is rejected with the documented error,
    before any device work."""
    P_ = P()
    n, rp, ci, av = _random_sparse(64, 3, 5)
    op = P_.CsrOperator(n, rp, ci, av)
    ss = P_.ScalingShift(1.0, 0.0, 1.0, 0.0, 61, 0)
    r = 40
    p = 12  # w = 520 > 512
    V = np.ones((n, p + 1))
    with pytest.raises(ValueError, match="not supported"):
        P_.phimv_block(op, P_.BlockPhiRequest(np.full(r, 0.1), np.ones(r), V, 1e-10, ss))


@pytest.mark.parametrize("n,p,r", [(10007, 3, 4), (12011, 1, 4), (6007, 3, 8), (20011, 0, 6)])
def test_short_row_grid_kernel_bitwise(n, p, r):
    """Operators with 3-5 entries per row and more tiles than SMs: the static
    gather-batch-5 kernel with its lean S-term body (grid-stride warp tiles,
    shared-memory column coefficients), at sizes that leave a ragged last
    warp tile."""
    P_ = P()
    rng = np.random.default_rng(n + 7 * p + r)
    rp = [0]
    ci, av = [], []
    for i in range(n):
        k = int(rng.integers(2, 5))
        cols = sorted(set(rng.integers(max(0, i - 300), min(n, i + 300), size=k).tolist()) | {i})
        vals = rng.standard_normal(len(cols))
        vals[cols.index(i)] = -(np.abs(vals).sum() + 1.0)
        ci += cols
        av += (vals * 50.0).tolist()
        rp.append(len(ci))
    rp, ci, av = np.array(rp, dtype=np.int64), np.array(ci, dtype=np.int32), np.array(av)
    op = P_.CsrOperator(n, rp, ci, av)
    oop = O.csr_from_arrays(n, rp, ci, av)
    tol = 1e-10
    ss = P_.select_parameters(op, 61, tol)
    sso = O.select_parameters(oop, 61, tol)
    assert ss.astuple() == sso.astuple()
    V = O.Rng(n).matrix(n, p + 1)
    t = np.linspace(0.2, 1.0, r) * (2.0 / sso.s)
    alpha = np.linspace(-1.0, 1.5, r)
    Wo, ro = O.phimv_block(oop, t, alpha, V, tol, sso)
    res = P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, ss))
    assert (res.stats.s_effective, res.stats.series_len_S) == (ro.s_effective, ro.series_len_S)
    assert res.stats.series_lens_F == ro.series_lens_F
    assert np.array_equal(res.W, Wo)
    assert P_.last_eval_mode() == 0
    var = P_.last_eval_variant()
    assert (var["Q"], var["V"], var["R"]) == (1, 2, 1)
    assert (var["dynamic_tail"], var["latency_mode"], var["short_batch"]) == (0, 0, 1)


@pytest.mark.parametrize("p,r,k", [(3, 4, 8), (4, 6, 7), (2, 3, 9), (7, 8, 4), (15, 8, 3),
                                   (3, 8, 1), (0, 5, 6)])
def test_grid_kernel_layouts_bitwise(p, r, k):
    """The persistent grid kernel (not latency mode) for every lane layout:
    Q = 1..8 column chunks, V = 1 / 2 columns per lane, R = 1 / 2 rows per lane
    group, default and short gather batches, with recovery sweeps."""
    P_ = P()
    n = 40000
    n_, rp, ci, av = _random_sparse(n, k, 300 + 13 * p + r + k)
    av = av * 20.0
    op = P_.CsrOperator(n_, rp, ci, av)
    oop = O.csr_from_arrays(n_, rp, ci, av)
    tol = 1e-10
    ss = O.select_parameters(oop, 61, tol)
    rng = O.Rng(77 + p + r)
    V = rng.matrix(n_, p + 1)
    t = (0.5 + rng.uniforms(r)) * (1.5 / ss.s)
    alpha = -1.0 + 2.0 * rng.uniforms(r)
    Wo, ro = O.phimv_block(oop, t, alpha, V, tol, ss)
    res = P_.phimv_block(op, P_.BlockPhiRequest(t, alpha, V, tol, P_.ScalingShift(*ss.astuple())))
    var = P_.last_eval_variant()
    assert var["latency_mode"] == 0 and var["grid"] > 148
    assert res.stats.series_len_S == ro.series_len_S
    assert res.stats.series_lens_F == ro.series_lens_F
    assert np.array_equal(res.W, Wo)


def test_single_variant_grid_kernel_bitwise():
    """phimv (Alg. 2: exp_v0 and the phi tail beside w) through the persistent
    grid kernel at n = 40,000, with recovery sweeps."""
    P_ = P()
    n, rp, ci, av = _random_sparse(40000, 5, 4711)
    av = av * 20.0
    op = P_.CsrOperator(n, rp, ci, av)
    oop = O.csr_from_arrays(n, rp, ci, av)
    tol = 1e-12
    ss = O.select_parameters(oop, 61, tol)
    V = O.Rng(12).matrix(n, 4)
    t = 3.5 / ss.s
    w, e0, tail, rec = O.phimv(oop, t, 0.75, V, tol, ss)
    res = P_.phimv(op, P_.PhiRequest(t, 0.75, V, tol, P_.ScalingShift(*ss.astuple())))
    assert rec.s_effective > 1
    assert P_.last_eval_variant()["latency_mode"] == 0
    assert res.stats.series_lens_F == rec.series_lens_F
    assert np.array_equal(res.w, w)
    assert np.array_equal(res.exp_v0, e0) and np.array_equal(res.tail, tail)


def test_c5_dynamic_tail_variant_bitwise(monkeypatch):
    """C5's production variant of k_phimv_block at full size -- the
    dynamic-tail (1, 2, 2) short-batch-2 kernel, chosen from ~1.8 M rows --
    forced (PHX_FORCE_DYN) at n = 2^14, where the oracle is quick: run record
    and W bitwise the oracle's through 420 recovery sweeps."""
    monkeypatch.setenv("PHX_BULK", "0")
    monkeypatch.setenv("PHX_FORCE_DYN", "1")
    p = P()
    wl = p.workload(5, 1 << 14)
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    ss = O.select_parameters(oop, 61, wl.tol)
    Wo, ro = O.phimv_block(oop, wl.t, wl.alpha, wl.V, wl.tol, ss)
    res = p.phimv_block(op, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol,
                                              p.ScalingShift(*ss.astuple())))
    var = p.last_eval_variant()
    assert (var["Q"], var["V"], var["R"]) == (1, 2, 2)
    assert (var["dynamic_tail"], var["short_batch"], var["latency_mode"]) == (1, 1, 0)
    assert ro.s_effective > 400
    assert (res.stats.series_len_S, res.stats.series_lens_F) == (ro.series_len_S, ro.series_lens_F)
    assert np.array_equal(res.W, Wo)


@pytest.mark.parametrize("bulk", ["1", "0"])
def test_c5_production_size_bitwise(golden_dir, monkeypatch, bulk):
    """C5 at n = 2^21 (419 recovery sweeps, ~16,000 grid steps), the size from
    which both production kernels run it -- the bulk-copy kernel (merged
    window-only stages) and k_phimv_block's dynamic-tail (1, 2, 2) batch-2
    variant -- against the oracle's committed SHA-256 of W, sampled rows and
    run record (tests/golden/full_cfg5_s2097152, make_golden.py c5big)."""
    name = "full_cfg5_s2097152"
    if not os.path.exists(os.path.join(golden_dir, name + ".json")):
        pytest.skip("C5 2^21 fixture not generated")
    monkeypatch.setenv("PHX_BULK", bulk)
    meta, arr = load(golden_dir, name)
    wl = P().workload(5, 1 << 21)
    p = P()
    op = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.ScalingShift(*meta["params"])
    res = p.phimv_block(op, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    var = p.last_eval_variant()
    if bulk == "1":
        assert var["dynamic_tail"] == 2
    else:
        assert (var["dynamic_tail"], var["short_batch"], var["R"]) == (1, 1, 2)
    st = res.stats
    assert (st.s_effective, st.series_len_S, st.series_lens_F, st.matvecs) == (
        meta["s_effective"], meta["series_len_S"], meta["series_lens_F"], meta["matvecs"])
    assert np.array_equal(res.W[arr["sample_rows"]], arr["sample_W"])
    assert sha(res.W) == meta["W_sha256"]


@pytest.mark.parametrize("scales", [(0.0, 1e-310, 1.0, 0.0), (1e-300, 0.0, 1e300, 1e-5),
                                    (0.0, 0.0, 0.0, 3.0), (5e-324, 2.0, 1e-320, 1e10)])
def test_selection_stablenorm_branches_bitwise(scales):
    """select_parameters on diagonal operators whose 4096-row chunks carry very
    different magnitudes (all-zero chunks, subnormal and huge entries): the
    stableNorm's per-chunk invScale comes from the device's parallel prefix
    scan and the fold from the host; ScalingShift bitwise the oracle's."""
    p = P()
    rng = np.random.default_rng(11)
    n = 4096 * len(scales)
    d = np.concatenate([s * (1.0 + rng.random(4096)) for s in scales]) * -1.0
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int32)
    op = p.CsrOperator(n, rp, ci, d)
    oop = O.csr_from_arrays(n, rp, ci, d)
    for tol in (2.0 ** -53, 1e-8):
        try:
            ss = p.select_parameters(op, 61, tol).astuple()
        except Exception as e:  # the same rejection as the oracle's
            with pytest.raises(type(e)):
                O.select_parameters(oop, 61, tol)
            continue
        assert ss == O.select_parameters(oop, 61, tol).astuple()
