import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2509_26475_b200 as P
N = 1024; n = N * N
wl = P.workload(2, 0)
for label, (rp, ci, av) in [("c2", (wl.rp, wl.ci, wl.av))]:
    pass
# the microbench's stencil: 1 (down), 1.5 (left), -4, 0.5 (right), 1 (up)
rows = []
idx = np.arange(n)
i = idx % N; j = idx // N
cols_list, vals_list = [], []
for dj, di, v in [(-1, 0, 1.0), (0, -1, 1.5), (0, 0, -4.0), (0, 1, 0.5), (1, 0, 1.0)]:
    ok = (i + di >= 0) & (i + di < N) & (j + dj >= 0) & (j + dj < N)
    cols_list.append(np.where(ok, idx + di + dj * N, -1)); vals_list.append(np.where(ok, v, 0.0))
C = np.stack(cols_list, 1); Vv = np.stack(vals_list, 1)
mask = C >= 0
cnt = mask.sum(1)
rp = np.zeros(n + 1, dtype=np.int64); rp[1:] = np.cumsum(cnt)
ci = C[mask].astype(np.int32); av = Vv[mask] * 1e4
for label, (rp_, ci_, av_) in [("mbstencil", (rp, ci, av)), ("c2", (wl.rp, wl.ci, wl.av))]:
    op = P.CsrOperator(n, rp_, ci_, av_)
    ss = P.select_parameters(op, 61, wl.tol)
    req = P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)
    for _ in range(3):
        res = P.phimv_block(op, req)
    ms, steps = P.last_eval_stats()
    print(label, f"{ms:.3f} ms", steps, "L_S", res.stats.series_len_S, "s_eff", res.stats.s_effective, flush=True)
    op.close()
