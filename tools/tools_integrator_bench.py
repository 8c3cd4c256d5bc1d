"""Integrator timing (developer script, run on the GPU box):
the reference's ADR order study (bench.cpp:131-179: 50x50 grid, tol 1e-7, T = 1/32,
h0 = T/128 .. h0/8) through the product, the oracle beside it on one core, and a
large grid for the device path.  Prints one JSON object per line."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
import oracle as O  # noqa: E402  (CPU baseline of the study)
import paper_2509_26475_b200 as P  # noqa: E402


def study(nx, ny, tol, t_end, hs, cpu=True):
    prob = P.adr_build(nx, ny)
    sel = P.select_parameters(prob.op, 61, tol)
    csr = O.csr_from_arrays(prob.op.n, *P.adr_csr(nx, ny)[:3])
    ss = O.ScalingShift(*sel.astuple())
    for h in hs:
        P.integrate(prob, h, h, tol, sel, keep_records=False)  # warm
        t0 = time.perf_counter()
        res = P.integrate(prob, h, t_end, tol, sel, keep_records=False)
        gpu_s = time.perf_counter() - t0
        steps = int(round(t_end / h))
        row = {"grid": nx, "h": h, "steps": steps, "gpu_s": gpu_s,
               "gpu_steps_per_s": steps / gpu_s}
        if cpu:
            t0 = time.perf_counter()
            uo, _, _ = O.integrate(csr, prob.gamma, prob.u0, h, t_end, tol, ss, keep_records=False)
            cpu_s = time.perf_counter() - t0
            row.update({"oracle_1core_s": cpu_s, "bitwise_equal": bool(np.array_equal(uo, res.u))})
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    T = 0.5 / 16.0
    h0 = T / 128.0
    study(50, 50, 1e-7, T, [h0, h0 / 2.0, h0 / 4.0, h0 / 8.0])
    study(1024, 1024, 1e-7, 8 * h0, [h0], cpu=False)
