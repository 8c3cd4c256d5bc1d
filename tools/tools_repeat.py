import sys, numpy as np
sys.path.insert(0, '/root/repo')
import oracle as O, paper_2509_26475_b200 as P
cfg, size, trace = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
wl = P.workload(cfg, size)
op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
ss = P.select_parameters(op, 61, wl.tol)
oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
Wo, ro = O.phimv_block(oop, wl.t, wl.alpha, wl.V, wl.tol, O.ScalingShift(*ss.astuple()))
if trace: P.set_trace(3*200000)
for it in range(5):
    res = P.phimv_block(op, P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss))
    d = np.abs(res.W - Wo)
    print(f"cfg{cfg} trace={trace} it{it}: L_S={res.stats.series_len_S} bitwise={np.array_equal(res.W, Wo)} maxdiff={d.max():.3e} |W|={np.linalg.norm(res.W):.9e} |Wo|={np.linalg.norm(Wo):.9e} argmax={np.unravel_index(d.argmax(), d.shape)}", flush=True)
