"""Developer experiment: DRAM traffic of the S series vs the z-plane distance
of a 7-point stencil (C3 parameters; same n, different grid shapes)."""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_2509_26475_b200 as P  # noqa: E402


def grid3(nx, ny, nz, eps=1e-2):
    h = 1.0 / 257.0  # C3 coefficients for every shape
    v = 1.0 / np.sqrt(3.0)
    d = eps / (h * h)
    a = v / h
    n = nx * ny * nz
    idx = np.arange(n, dtype=np.int64)
    i, j, k = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    cols, vals, rows = [], [], []
    P_ = nx * ny
    for (cond, off, val) in [(k > 0, -P_, d + a), (j > 0, -nx, d + a), (i > 0, -1, d + a),
                             (np.ones(n, bool), 0, -6 * d - 3 * a), (i < nx - 1, 1, d),
                             (j < ny - 1, nx, d), (k < nz - 1, P_, d)]:
        rows.append(idx[cond])
        cols.append(idx[cond] + off)
        vals.append(np.full(int(cond.sum()), val))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    return n, np.cumsum(rp), cols.astype(np.int32), vals


def run(shape):
    n, rp, ci, av = grid3(*shape)
    op = P.CsrOperator(n, rp, ci, av)
    c = np.array([0.5, 0.5, 1 / 3, 5 / 6, 1 / 3, 1.0])
    V = np.random.default_rng(3).standard_normal((n, 5))
    tol = 2.0 ** -53
    sel = P.select_parameters(op, 61, tol)
    req = P.BlockPhiRequest(1e-3 * c, c, V, tol, sel)
    P.phimv_block(op, req)
    t0 = time.time()
    res = P.phimv_block(op, req)
    ms, steps = P.last_eval_stats()
    print(shape, "kernel ms", round(ms, 2), "L_S", res.stats.series_len_S, flush=True)


if __name__ == "__main__":
    for s in sys.argv[1:]:
        run(tuple(int(x) for x in s.split("x")))
