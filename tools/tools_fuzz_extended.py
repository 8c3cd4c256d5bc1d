"""Developer run: a longer randomized parity sweep of the bulk evaluator than the
test suite's (tests/test_bulk_fuzz.py), plus draws aimed at the specialised
consumers: S-term shapes with 16 < w <= 32 and r even on banded operators with
offset groups, and window-only (tri/bidiagonal) operators with 8 < 2r <= 16 and
recovery sweeps.  Every case: ScalingShift, RunRecord and W bitwise the oracle's.
python tools/tools_fuzz_extended.py [n_general] [n_targeted]"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
os.environ["PHX_BULK"] = "1"
import oracle as O  # noqa: E402
import paper_2509_26475_b200 as P  # noqa: E402
import test_bulk_fuzz as F  # noqa: E402

n_general = int(sys.argv[1]) if len(sys.argv) > 1 else 300
n_targeted = int(sys.argv[2]) if len(sys.argv) > 2 else 120

S_SHAPES = [(2, 6), (3, 6), (4, 6), (2, 8), (3, 8), (4, 4), (5, 4), (6, 4), (7, 4), (2, 10), (1, 12), (1, 16)]
F_SHAPES = [(1, 5), (3, 5), (0, 6), (1, 6), (2, 6), (1, 7), (3, 7), (0, 8), (1, 8), (3, 8)]


def banded(rng, n, offs, scale):
    rp, ci, av = [0], [], []
    for i in range(n):
        cols = sorted({i} | {i + o for o in offs if 0 <= i + o < n})
        vals = rng.standard_normal(len(cols)) * scale
        vals[cols.index(i)] = -(np.abs(vals).sum() + scale)
        ci += cols
        av += vals.tolist()
        rp.append(len(ci))
    return n, np.array(rp, dtype=np.int64), np.array(ci, dtype=np.int32), np.array(av)


def run(n, rp, ci, av, p, r, rng, want_sweeps):
    op = P.CsrOperator(n, rp, ci, av)
    oop = O.csr_from_arrays(n, rp, ci, av)
    tol = float(rng.choice([1e-8, 1e-11, 2.0 ** -53]))
    sso = O.select_parameters(oop, 61, tol)
    ss = P.select_parameters(op, 61, tol)
    assert ss.astuple() == sso.astuple()
    V = O.Rng(int(rng.integers(1, 1 << 30))).matrix(n, p + 1)
    t = (0.3 + rng.random(r)) * ((4.5 if want_sweeps else 0.9) / sso.s)
    alpha = rng.uniform(-2, 2, size=r)
    Wo, ro = O.phimv_block(oop, t, alpha, V, tol, sso)
    res = P.phimv_block(op, P.BlockPhiRequest(t, alpha, V, tol, ss))
    assert P.last_eval_variant()["dynamic_tail"] == 2
    assert (res.stats.s_effective, res.stats.series_len_S, res.stats.series_lens_F) == \
        (ro.s_effective, ro.series_len_S, ro.series_lens_F)
    assert np.array_equal(res.W, Wo)
    op.close()
    return ro.s_effective, sso.xi != 0.0


ok = 0
for seed in range(n_general):
    F._case(50000 + seed, 1 if seed % 4 else 2 + seed % 3)
    ok += 1
print(f"general draws bitwise: {ok}", flush=True)
ns = nf = sweeps = 0
for seed in range(n_targeted):
    rng = np.random.default_rng(70000 + seed)
    n = int(rng.choice([333, 1000, 2500, 4097, 9001]))
    if seed % 2 == 0:
        p, r = S_SHAPES[int(rng.integers(len(S_SHAPES)))]
        offs = sorted({int(o) for o in rng.choice([-97, -40, -1, 1, 40, 97], size=int(rng.integers(2, 6)))})
        s_eff, xi = run(*banded(rng, n, offs, 10.0 ** rng.uniform(-1, 2)), p, r, rng, seed % 4 == 0)
        ns += 1
    else:
        p, r = F_SHAPES[int(rng.integers(len(F_SHAPES)))]
        offs = [[-1, 1], [1], [-1]][int(rng.integers(3))]
        s_eff, xi = run(*banded(rng, n, offs, 10.0 ** rng.uniform(-1, 2)), p, r, rng, True)
        nf += 1
    sweeps += s_eff > 1
print(f"targeted draws bitwise: S-term shapes {ns}, window-only recovery shapes {nf} "
      f"({sweeps} with recovery sweeps)", flush=True)
