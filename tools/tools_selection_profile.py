import sys, time
sys.path.insert(0, "/root/repo")
import paper_2509_26475_b200 as P
for cfg in (2, 3):
    wl = P.workload(cfg, 0, with_V=False)
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    P.select_parameters(op, 61, wl.tol)
    t0 = time.perf_counter(); ss = P.select_parameters(op, 61, wl.tol); t1 = time.perf_counter()
    print(f"cfg{cfg}: select {1e3*(t1-t0):.2f} ms", flush=True)
    op.close()
