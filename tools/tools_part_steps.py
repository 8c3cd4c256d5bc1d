"""Developer diagnostic: per-step durations (PHX_STEP_TIMES=1) of one config
unpartitioned and row-partitioned on one device (the partitioned path stamps
part 0's steps after each mailbox barrier)."""
import os
import sys

os.environ["PHX_STEP_TIMES"] = "1"
sys.path.insert(0, "/root/repo")
import paper_2509_26475_b200 as P  # noqa: E402

cfg, size = map(int, sys.argv[1].split(":"))
wl = P.workload(cfg, size)
for parts in [int(x) for x in sys.argv[2:]] or [1, 2, 8]:
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=parts) if parts > 1 else \
        P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = P.select_parameters(op, 61, wl.tol)
    req = P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)
    for _ in range(2):
        P.phimv_block(op, req)
    print(f"cfg{cfg} parts={parts} kernel_ms={P.last_eval_stats()[0]:.2f}", file=sys.stderr, flush=True)
    op.close()
