"""Developer check: the bulk-copy evaluator (PHX_BULK=1) against the
register-gather kernel (PHX_BULK=0) and the oracle, then full-size timings."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
import oracle as O  # noqa: E402
import paper_2509_26475_b200 as P  # noqa: E402


def run(op, wl, ss, mode):
    os.environ["PHX_BULK"] = mode
    res = P.phimv_block(op, P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    return res, P.last_eval_variant(), P.last_eval_stats()[0]


for cfg, size in [(3, 16), (3, 40), (2, 128), (5, 1 << 13), (2, 300)]:
    wl = P.workload(cfg, size)
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = P.select_parameters(op, 61, wl.tol)
    r0, v0, _ = run(op, wl, ss, "0")
    r1, v1, _ = run(op, wl, ss, "1")
    oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    Wo, ro = O.phimv_block(oop, wl.t, wl.alpha, wl.V, wl.tol, O.ScalingShift(*ss.astuple()))
    print(f"cfg{cfg} n={wl.n} bulk_var={v1['dynamic_tail']} grid={v1['grid']} "
          f"L_S={r1.stats.series_len_S}/{ro.series_len_S} sweeps={len(r1.stats.series_lens_F)} "
          f"bitwise_vs_old={np.array_equal(r0.W, r1.W)} bitwise_vs_oracle={np.array_equal(r1.W, Wo)} "
          f"lensF_eq={r1.stats.series_lens_F == ro.series_lens_F}", flush=True)

for cfg, size in [(3, 0), (2, 0), (5, 1 << 21)]:
    wl = P.workload(cfg, size)
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = P.select_parameters(op, 61, wl.tol)
    for mode in ("0", "1", "0", "1"):
        res, var, ms = run(op, wl, ss, mode)
        print(f"cfg{cfg} n={wl.n} PHX_BULK={mode} kernel_ms={ms:.2f} var={var} L_S={res.stats.series_len_S}",
              flush=True)
        if mode == "1":
            W1 = res.W
        else:
            W0 = res.W
    print(f"cfg{cfg} full bitwise bulk==old: {np.array_equal(W0, W1)}", flush=True)
