"""Developer script: kernel time of a row-partitioned operator emulated on one
GPU (all parts in one cooperative launch) against the unpartitioned kernel --
the cost of the part tables and the mailbox step barrier."""
import json
import os
import sys

sys.path.insert(0, "/root/repo")
if os.environ.get("AB_HEAD"):  # another build under abtest/<AB_HEAD>
    sys.path.insert(0, "/root/repo/abtest/" + os.environ["AB_HEAD"])
import paper_2509_26475_b200 as P  # noqa: E402

for arg in sys.argv[1:]:
    cfg, size = map(int, arg.split(":"))
    wl = P.workload(cfg, size)
    base = None
    for parts in (1, 2, 4, 8):
        op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=parts) if parts > 1 else \
            P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
        ss = P.select_parameters(op, 61, wl.tol)
        req = P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)
        ts = []
        for _ in range(4):
            res = P.phimv_block(op, req)
            ts.append(P.last_eval_stats()[0])
        ms = min(ts[1:])
        steps = P.last_eval_stats()[1]
        base = base or ms
        print(json.dumps({"cfg": cfg, "n": wl.n, "parts": parts, "kernel_ms": ms, "grid_steps": steps,
                          "vs_unpartitioned": ms / base,
                          "us_per_step_extra": (ms - base) * 1e3 / steps}), flush=True)
        op.close()
