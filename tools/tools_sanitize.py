"""Small evaluations for compute-sanitizer runs (memcheck / racecheck /
synccheck, one tool per process): every kernel family on small operators --
the register-gather persistent kernel (latency mode and grid mode), the
bulk-copy kernel (offset groups, merged window-only stages, recovery sweeps),
the partitioned emulation (mailbox barrier), selection kernels -- each
checked bitwise against the oracle so a silent corruption also fails."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
import oracle as O  # noqa: E402
import paper_2509_26475_b200 as P  # noqa: E402


def check(cfg, size, bulk, parts=1):
    os.environ["PHX_BULK"] = bulk
    wl = P.workload(cfg, size)
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, parts=parts) if parts > 1 else \
        P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    ss = P.select_parameters(op, 61, wl.tol)
    sso = O.select_parameters(oop, 61, wl.tol)
    assert ss.astuple() == sso.astuple()
    res = P.phimv_block(op, P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    Wo, ro = O.phimv_block(oop, wl.t, wl.alpha, wl.V, wl.tol, sso)
    ok = np.array_equal(res.W, Wo)
    var = P.last_eval_variant() if parts == 1 else {"parts": parts}
    print(f"cfg{cfg} size {size} PHX_BULK={bulk} parts={parts}: bitwise={ok} variant={var}",
          flush=True)
    assert ok
    op.close()


check(1, 200, "0")                 # latency mode, recovery sweeps
check(2, 64, "0")                  # C2 small
check(2, 160, "0")                 # grid kernel (more tiles than SMs)
check(3, 12, "1")                  # bulk kernel, offset groups
check(3, 20, "1")
check(5, 3000, "1")                # bulk kernel, merged window-only stages, sweeps
check(2, 48, "0", parts=3)         # partitioned emulation (mailbox barrier)
print("sanitize cases done", flush=True)
