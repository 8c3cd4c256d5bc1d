"""Row-partitioned evaluation in its single-GPU emulation:
every part is processed by its own CTA group of ONE cooperative launch with
its own buffers; other parts' block rows are read through the part table and
the per-term maxima are combined through the cross-part mailboxes — the
exact protocol of the multi-GPU run.  The result must be bitwise the
unpartitioned one (rows are independent given the previous term; maxima
are order-free)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def P():
    import paper_2509_26475_b200 as mod
    return mod


@pytest.mark.parametrize("cfg,size,parts", [(1, 0, 2), (1, 0, 3), (2, 64, 2), (2, 64, 4),
                                            (3, 12, 3), (4, 1024, 4), (5, 2000, 2),
                                            (5, 2000, 7)])
def test_partitioned_bitwise(cfg, size, parts):
    p = P()
    wl = p.workload(cfg, size)
    whole = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(whole, 61, wl.tol)
    ref = p.phimv_block(whole, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    part = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=parts)
    assert part.parts == parts
    p.set_trace(3 * 100000)
    res = p.phimv_block(part, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    tr = p.get_trace(3 * 100000)
    p.set_trace(0)
    assert res.stats.series_len_S == ref.stats.series_len_S
    assert res.stats.series_lens_F == ref.stats.series_lens_F
    assert res.stats.matvecs == ref.stats.matvecs
    assert np.array_equal(res.W, ref.W)
    oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    _, _, otr = O.phimv_block(oop, wl.t, wl.alpha, wl.V, wl.tol, O.ScalingShift(*ss.astuple()),
                              trace=True)
    assert np.array_equal(tr, otr)


@pytest.mark.parametrize("cfg,size,parts", [(1, 0, 8), (1, 0, 16), (2, 24, 8), (3, 8, 8),
                                            (4, 512, 16), (5, 1000, 16), (1, 300, 3)])
def test_cluster_mode_bitwise(cfg, size, parts, monkeypatch):
    """Parts on one device that fit in shared memory run as ONE thread-block
    cluster (opt-in PHX_CLUSTER=1: DSMEM gathers, cluster barrier): bitwise the
    unpartitioned run, term by term."""
    monkeypatch.setenv("PHX_CLUSTER", "1")
    p = P()
    wl = p.workload(cfg, size)
    whole = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(whole, 61, wl.tol)
    ref = p.phimv_block(whole, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    part = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=parts)
    res = p.phimv_block(part, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    assert p.last_eval_mode() == 2
    assert res.stats.series_len_S == ref.stats.series_len_S
    assert res.stats.series_lens_F == ref.stats.series_lens_F
    assert np.array_equal(res.W, ref.W)
    p.set_trace(3 * 100000)
    p.phimv_block(part, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    tr = p.get_trace(3 * 100000)
    p.set_trace(0)
    oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    _, _, otr = O.phimv_block(oop, wl.t, wl.alpha, wl.V, wl.tol, O.ScalingShift(*ss.astuple()),
                              trace=True)
    assert np.array_equal(tr, otr)


def test_partitioned_full_c2_bitwise():
    p = P()
    wl = p.workload(2, 0)
    whole = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(whole, 61, wl.tol)
    ref = p.phimv_block(whole, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)).W
    part = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=8)
    W = p.phimv_block(part, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)).W
    assert np.array_equal(W, ref)


@pytest.mark.parametrize("cfg,size,parts", [(2, 32, 2), (3, 12, 3), (5, 2000, 7)])
def test_partitioned_selection_is_the_whole_operators(cfg, size, parts):
    """select_parameters / apply on a partitioned operator run on its selection
    replica (the whole CSR on part 0's device): bitwise the unpartitioned
    ScalingShift, and the evaluation with it matches end to end."""
    p = P()
    wl = p.workload(cfg, size)
    whole = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    part = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=parts)
    ss_w = p.select_parameters(whole, 61, wl.tol)
    ss_p = p.select_parameters(part, 61, wl.tol)
    assert ss_p.astuple() == ss_w.astuple()
    X = np.asfortranarray(wl.V[:, :2])
    assert np.array_equal(part.apply(X), whole.apply(X))
    req = p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss_p)
    assert np.array_equal(p.phimv_block(part, req).W, p.phimv_block(whole, req).W)


@pytest.mark.parametrize("cfg,size,parts", [(1, 0, 2), (2, 64, 3), (3, 12, 3), (3, 20, 8),
                                            (5, 2000, 2), (5, 3000, 7), (2, 160, 16)])
def test_partitioned_bulk_bitwise(cfg, size, parts, monkeypatch):
    """The bulk-copy kernel's partitioned instantiation (forced with
    PHX_BULK=1): each part stages its tiles' gathers -- rows of other parts
    included, cut at the part boundaries and copied from the owner's buffers
    -- and the parts combine their maxima through the mailboxes.  Bitwise the
    unpartitioned evaluation, term by term against the oracle's trace."""
    monkeypatch.setenv("PHX_BULK", "1")
    p = P()
    wl = p.workload(cfg, size)
    whole = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(whole, 61, wl.tol)
    ref = p.phimv_block(whole, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    part = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=parts)
    res = p.phimv_block(part, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    assert p.last_eval_mode() == 1 and p.last_eval_variant()["dynamic_tail"] == 2
    assert res.stats.series_len_S == ref.stats.series_len_S
    assert res.stats.series_lens_F == ref.stats.series_lens_F
    assert res.stats.matvecs == ref.stats.matvecs
    assert np.array_equal(res.W, ref.W)
    p.set_trace(3 * 100000)
    p.phimv_block(part, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    tr = p.get_trace(3 * 100000)
    p.set_trace(0)
    oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    _, _, otr = O.phimv_block(oop, wl.t, wl.alpha, wl.V, wl.tol, O.ScalingShift(*ss.astuple()),
                              trace=True)
    assert np.array_equal(tr, otr)


@pytest.mark.parametrize("parts", [2, 8])
def test_partitioned_full_c3_bulk_bitwise(golden_dir, parts):
    """Full-size C3 (n = 2^24) row-partitioned into 2 / 8 parts -- the
    multi-GPU configuration of SURVEY.md §8e in its single-GPU emulation --
    runs the partitioned bulk kernel and reproduces the oracle's committed
    SHA-256 of W (tests/golden/full_cfg3.json)."""
    import hashlib
    import json
    import os
    p = P()
    with open(os.path.join(golden_dir, "full_cfg3.json")) as f:
        meta = json.load(f)
    wl = p.workload(3, 0)
    part = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=parts)
    ss = p.ScalingShift(*meta["params"])
    res = p.phimv_block(part, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    assert p.last_eval_variant()["dynamic_tail"] == 2
    assert res.stats.series_len_S == meta["series_len_S"]
    h = hashlib.sha256(np.asfortranarray(res.W).tobytes(order="F")).hexdigest()
    assert h == meta["W_sha256"]


@pytest.mark.parametrize("cfg,size,bulk", [(3, 20, "1"), (2, 64, "0"), (5, 3000, "1")])
def test_multi_device_partition_bitwise(cfg, size, bulk, monkeypatch):
    """Parts on DISTINCT devices (one launch per device, peer gathers / peer
    bulk copies over NVLink, system-scope mailboxes): bitwise the one-GPU
    evaluation.  Needs >= 2 GPUs (skipped on a one-GPU box)."""
    import torch
    ndev = torch.cuda.device_count()
    if ndev < 2:
        pytest.skip("needs >= 2 GPUs")
    monkeypatch.setenv("PHX_BULK", bulk)
    p = P()
    wl = p.workload(cfg, size)
    whole = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = p.select_parameters(whole, 61, wl.tol)
    ref = p.phimv_block(whole, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    parts = min(ndev, 4)
    part = p.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=parts, devices=list(range(parts)))
    res = p.phimv_block(part, p.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    assert res.stats.series_len_S == ref.stats.series_len_S
    assert res.stats.series_lens_F == ref.stats.series_lens_F
    assert np.array_equal(res.W, ref.W)
