import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2509_26475_b200 as P
cfg, size = int(sys.argv[1]), int(sys.argv[2])
wl = P.workload(cfg, size)
whole = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
ss = P.select_parameters(whole, 61, wl.tol)
ref = P.phimv_block(whole, P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)).W
for parts in [int(x) for x in sys.argv[3:]]:
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=parts)
    for rep in range(2):
        W = P.phimv_block(op, P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)).W
        bad = np.nonzero(np.any(W != ref, axis=1))[0]
        bnd = [q * wl.n // parts for q in range(parts + 1)]
        print(f"parts={parts} rep={rep} bad_rows={len(bad)} first={bad[:12].tolist()} bounds={bnd}", flush=True)
