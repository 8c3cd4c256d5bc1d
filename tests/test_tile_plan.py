"""The bulk-copy evaluator's tile plan (csrc/phx_plan.cpp), checked on the
host: every CSR entry's one-byte slot must lead, through its tile's copy
descriptors, back to exactly the column it gathers -- the inspector half of
the bulk kernel's gather.  No device needed."""
import numpy as np
import pytest

import paper_2509_26475_b200 as P

T = P.tile_plan(1, [0, 1], [0])[0]["T"]  # rows per tile (kPlanT)


def check_plan(n, rp, ci):
    info, desc, slot, sgl = P.tile_plan(n, rp, ci)
    assert info["ok"] == 1
    assert info["tiles"] == (n + T - 1) // T
    scap = info["singles_cap"]
    gbase = T + 2 + scap
    assert info["rows"] <= 256 and (info["rows"] - gbase) % T == 0
    ngmax = (info["rows"] - gbase) // T
    order = desc[:, 5]
    assert sorted(order.tolist()) == list(range(info["tiles"]))  # a permutation of the tiles
    for d in desc:
        t = int(d[5])
        base = t * T
        rows = min(T, n - base)
        wlo, whi = max(base - 1, 0), min(base + rows + 1, n)
        ng, nsgl, s0, e_lo, e_hi = (int(x) for x in d[:5])
        assert (e_lo, e_hi) == (rp[base], rp[base + rows])
        assert ng <= ngmax and nsgl <= scap
        groups = []
        for g in range(ng):
            src0, cnt, dst = int(d[8 + g]), int(d[12 + g]) & 0xFFFF, int(d[12 + g]) >> 16
            assert 0 <= src0 and src0 + cnt <= n and 1 <= cnt <= T
            assert gbase + g * T <= dst and dst + cnt <= gbase + (g + 1) * T
            groups.append((src0, cnt, dst))
        for e in range(e_lo, e_hi):
            s = int(slot[e])
            if s < T + 2:
                src = wlo + s
                assert src < whi
            elif s < gbase:
                q = s - (T + 2)
                assert q < nsgl
                src = sgl[s0 + q]
            else:
                hit = [src0 + (s - dst) for (src0, cnt, dst) in groups if dst <= s < dst + cnt]
                assert len(hit) == 1
                src = hit[0]
            assert src == ci[e], (t, e, s)
    return info


def test_stencil_3d_four_groups():
    wl = P.workload(3, 20, with_V=False)  # 20^3 7-point stencil
    info = check_plan(wl.n, wl.rp, wl.ci)
    assert info["rows"] == T + 2 + 4 * T and info["singles"] == 0


def test_lattice_tile_order():
    """A 3D lattice (strides 256, 256^2 -> here 64, 64^2 with 64 z-planes) is
    swept in y-blocks of 32 lines: for each block, for z, for y, for x."""
    wl = P.workload(3, 128, with_V=False)  # 128^3 (>= 2 x 32 y-lines)
    info, desc, _, _ = P.tile_plan(wl.n, wl.rp, wl.ci)
    order = desc[:, 5]
    xt = 128 // T
    want = [(z * 128 * 128 + y * 128) // T + x for yb in range(0, 128, 32) for z in range(128)
            for y in range(yb, yb + 32) for x in range(xt)]
    assert order.tolist() == want


def test_stencil_2d_two_groups():
    wl = P.workload(2, 96, with_V=False)
    info = check_plan(wl.n, wl.rp, wl.ci)
    assert info["rows"] == T + 2 + 2 * T and info["singles"] == 0


def test_bidiagonal_window_only():
    wl = P.workload(5, 5000, with_V=False)
    info = check_plan(wl.n, wl.rp, wl.ci)
    assert info["rows"] == T + 2 and info["singles"] == 0


def test_random_far_entries_as_singles():
    rng = np.random.default_rng(3)
    n = 3001
    rp, ci = [0], []
    for i in range(n):
        cols = {i, max(0, i - 1)}
        if rng.random() < 0.3:
            cols.add(int(rng.integers(0, n)))
        ci += sorted(cols)
        rp.append(len(ci))
    info = check_plan(n, np.array(rp), np.array(ci, dtype=np.int32))
    assert info["singles"] > 0


def test_unsorted_duplicates_and_empty_rows():
    rng = np.random.default_rng(4)
    n = 777
    rp, ci = [0], []
    for i in range(n):
        if i % 13 == 3:
            rp.append(len(ci))
            continue
        cols = [i, min(n - 1, i + 50), max(0, i - 50), i]  # duplicate diagonal
        rng.shuffle(cols)
        ci += cols
        rp.append(len(ci))
    check_plan(n, np.array(rp), np.array(ci, dtype=np.int32))


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 65])
def test_tiny_operators(n):
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int32)
    check_plan(n, rp, ci)


def test_plan_rejects_what_the_stage_cannot_hold():
    n = 64
    rp, ci = [0], []
    for i in range(n):  # every row touches 40 scattered columns: > 32 singles per tile
        ci += sorted({i} | {(i * 37 + 11 * k) % n for k in range(40)})
        rp.append(len(ci))
    ci = np.array(ci, dtype=np.int32)
    rp = np.array(rp)
    n2 = 4096
    rp2 = np.concatenate([[0], np.full(n2, 1300)]).cumsum()  # > 1024 entries per tile
    ci2 = np.tile(np.arange(1300, dtype=np.int32), n2)
    info2, *_ = P.tile_plan(n2, rp2, ci2)
    assert info2["ok"] == 0
