"""Developer script: cluster mode (one thread-block cluster, blocks in shared
memory) vs the grid-wide launch on small operators."""
import sys

sys.path.insert(0, "/root/repo")
import paper_2509_26475_b200 as P  # noqa: E402

for cfg, size, parts in [(1, 1000, 8), (1, 1000, 16), (1, 1000, 12), (5, 2000, 16), (2, 32, 16)]:
    wl = P.workload(cfg, size)
    whole = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = P.select_parameters(whole, 61, wl.tol)
    req = P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)
    P.phimv_block(whole, req)
    r0 = P.phimv_block(whole, req)
    ms0, steps = P.last_eval_stats()
    part = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=parts)
    P.phimv_block(part, req)
    r1 = P.phimv_block(part, req)
    ms1, _ = P.last_eval_stats()
    print(f"cfg{cfg} n={wl.n} steps={steps} grid {ms0:.2f} ms ({1e3 * ms0 / steps:.2f} us/step) | "
          f"cluster x{parts} mode={P.last_eval_mode()} {ms1:.2f} ms ({1e3 * ms1 / steps:.2f} us/step) "
          f"equal={bool((r0.W == r1.W).all())}", flush=True)
