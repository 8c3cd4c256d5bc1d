"""Developer script: run one full-size configuration several times and compare
W bitwise across runs (SHA-256 of W, run records, kernel times)."""
import hashlib
import json
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_2509_26475_b200 as P  # noqa: E402

cfg, size, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
wl = P.workload(cfg, size)
op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
ss = P.select_parameters(op, 61, wl.tol)
req = P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)
for it in range(reps):
    res = P.phimv_block(op, req)
    ms, steps = P.last_eval_stats()
    W = np.ascontiguousarray(res.W)
    print(json.dumps({"cfg": cfg, "n": wl.n, "run": it, "kernel_ms": ms, "grid_steps": steps,
                      "s_eff": res.stats.s_effective, "L_S": res.stats.series_len_S,
                      "sweeps": len(res.stats.series_lens_F), "matvecs": res.stats.matvecs,
                      "finite": bool(np.isfinite(W).all()),
                      "max_abs": float(np.max(np.abs(W[np.isfinite(W)]))) if np.isfinite(W).any() else None,
                      "sha256_W": hashlib.sha256(W.tobytes()).hexdigest()}), flush=True)
