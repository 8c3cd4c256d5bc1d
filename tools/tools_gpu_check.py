"""Quick GPU-vs-oracle parity probe (developer script)."""
import sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
import oracle as O
import paper_2509_26475_b200 as P

def cmp(name, a, b):
    a = np.asarray(a); b = np.asarray(b)
    same = np.array_equal(a, b)
    den = np.linalg.norm(b)
    rel = np.linalg.norm(a - b) / (den if den > 0 else 1)
    print(f"  {name}: bitwise={same} rel={rel:.3e}")
    return same

def run(cfg, size):
    wl = P.workload(cfg, size)
    oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    gop = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    t0 = time.time(); so = O.select_parameters(oop, 61, wl.tol); t1 = time.time()
    sg = P.select_parameters(gop, 61, wl.tol); t2 = time.time()
    print(f"cfg{cfg} n={wl.n} oracle_sel={t1-t0:.3f}s gpu_sel={t2-t1:.3f}s")
    print("  oracle", so.astuple()); print("  gpu   ", sg.astuple())
    ss = O.ScalingShift(*so.astuple())
    t0 = time.time(); Wo, ro, tro = O.phimv_block(oop, wl.t, wl.alpha, wl.V, wl.tol, ss, trace=True); t1 = time.time()
    P.set_trace(3 * 200000)
    res = P.phimv_block(gop, P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, P.ScalingShift(*so.astuple())))
    t2 = time.time()
    trg = P.get_trace()
    ms, steps = P.last_eval_stats()
    print(f"  eval oracle={t1-t0:.3f}s gpu={t2-t1:.3f}s kernel={ms:.3f}ms steps={steps}")
    print("  rec oracle", ro.s_effective, ro.series_len_S, ro.series_lens_F[:6], ro.matvecs)
    print("  rec gpu   ", res.stats.s_effective, res.stats.series_len_S, res.stats.series_lens_F[:6], res.stats.matvecs)
    ok = cmp("W", res.W, Wo)
    if tro.shape != trg.shape or not np.array_equal(tro, trg):
        k = min(len(tro), len(trg))
        bad = np.nonzero(np.any(tro[:k] != trg[:k], axis=1))[0]
        print("  trace mismatch: lens", len(tro), len(trg), "first bad", bad[:3], tro[bad[:1]], trg[bad[:1]])
    else:
        print("  trace identical", len(tro))
    return ok

cases = [(1, 0), (2, 64), (3, 12), (4, 1024), (5, 2000)]
if len(sys.argv) > 1:
    cases = [tuple(map(int, a.split(':'))) for a in sys.argv[1:]]
for c in cases:
    try:
        run(*c)
    except Exception as e:
        import traceback; traceback.print_exc()
print("launches", P.kernel_launches())
