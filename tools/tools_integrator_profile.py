"""Developer script: a short 50x50 ADR integration for an ncu launch list
(per-kernel device time of one integrator step vs its wall time)."""
import sys
import time

sys.path.insert(0, "/root/repo")
import paper_2509_26475_b200 as P  # noqa: E402

prob = P.adr_build(50, 50)
sel = P.select_parameters(prob.op, 61, 1e-7)
h = 0.5 / 16.0 / 128.0
P.integrate(prob, h, h, 1e-7, sel, keep_records=False)
t0 = time.perf_counter()
res = P.integrate(prob, h, 8 * h, 1e-7, sel, keep_records=True)
print(f"8 steps: {(time.perf_counter() - t0) / 8 * 1e6:.1f} us/step")
for c in res.steps[0].calls:
    print("call", c.s_effective, c.series_len_S, c.series_lens_F, c.matvecs)
