"""Developer script: kernel-time distribution of repeated evaluations of one
configuration (A/B of runtime knobs: run twice with different env)."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
if os.environ.get("AB_HEAD"):  # another build under abtest/<AB_HEAD>
    sys.path.insert(0, "/root/repo/abtest/" + os.environ["AB_HEAD"])
import paper_2509_26475_b200 as P  # noqa: E402

cfg, size, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
wl = P.workload(cfg, size)
op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
ss = P.select_parameters(op, 61, wl.tol)
req = P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)
ts = []
for _ in range(reps):
    P.phimv_block(op, req)
    ts.append(P.last_eval_stats()[0])
ts = np.array(ts[2:])
print(f"cfg{cfg} {P.__file__.split('/')[-3]} {' '.join(sys.argv[4:])}: min {ts.min():.3f} med {np.median(ts):.3f} ms over {ts.size}",
      flush=True)
