import os, sys
sys.path.insert(0, "/root/repo")
import paper_2509_26475_b200 as P
wl = P.workload(3, 0)
for parts in (1, 2):
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=parts) if parts > 1 else P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = P.select_parameters(op, 61, wl.tol)
    for it in range(2):
        res = P.phimv_block(op, P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    print("parts", parts, "kernel_ms", P.last_eval_stats(), res.stats.series_len_S, file=sys.stderr, flush=True)
    op.close()
