"""Developer check: per-step durations (PHX_STEP_TIMES=1) of the bulk and the
register-gather evaluators on full-size configs."""
import os
import sys

sys.path.insert(0, "/root/repo")
import paper_2509_26475_b200 as P  # noqa: E402

cfgs = [(int(a.split(":")[0]), int(a.split(":")[1])) for a in sys.argv[1:]] or [(3, 0)]
for cfg, size in cfgs:
    wl = P.workload(cfg, size)
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = P.select_parameters(op, 61, wl.tol)
    for mode in ("1", "0"):
        os.environ["PHX_BULK"] = mode
        res = P.phimv_block(op, P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
        print(f"cfg{cfg} n={wl.n} PHX_BULK={mode} kernel_ms={P.last_eval_stats()[0]:.2f} "
              f"steps={P.last_eval_stats()[1]}", file=sys.stderr, flush=True)
