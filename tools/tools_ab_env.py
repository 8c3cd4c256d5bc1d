"""Developer A/B: kernel time of repeated evaluations of one config under
several environment settings (same process, interleaved):
python tools/tools_ab_env.py cfg:size reps VAR=a,b,c"""
import os
import statistics
import sys

sys.path.insert(0, "/root/repo")
import paper_2509_26475_b200 as P  # noqa: E402

cfg, size = map(int, sys.argv[1].split(":"))
reps = int(sys.argv[2])
var, vals = sys.argv[3].split("=")
vals = vals.split(",")
wl = P.workload(cfg, size)
op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
ss = P.select_parameters(op, 61, wl.tol)
req = P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)
res = {v: [] for v in vals}
W = {}
for i in range(reps):
    for v in vals:
        os.environ[var] = v
        r = P.phimv_block(op, req)
        res[v].append(P.last_eval_stats()[0])
        W.setdefault(v, r.W)
for v in vals:
    print(f"cfg{cfg} {var}={v}: median {statistics.median(res[v]):.3f} ms  min {min(res[v]):.3f}  "
          f"all {[round(x, 2) for x in res[v]]}", flush=True)
import numpy as np  # noqa: E402
print("bitwise equal across settings:", all(np.array_equal(W[vals[0]], W[v]) for v in vals))
