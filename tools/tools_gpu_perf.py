"""GPU-only timing of full-size configs (developer script)."""
import sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
import paper_2509_26475_b200 as P
for a in sys.argv[1:]:
    cfg, size = map(int, a.split(':'))
    t0 = time.time(); wl = P.workload(cfg, size); t1 = time.time()
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    t2 = time.time(); ss = P.select_parameters(op, 61, wl.tol); t3 = time.time()
    res = P.phimv_block(op, P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)); t4 = time.time()
    ms, steps = P.last_eval_stats()
    res = P.phimv_block(op, P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)); t5 = time.time()
    ms2, _ = P.last_eval_stats()
    st = res.stats
    print(f"cfg{cfg} n={wl.n} nnz={wl.nnz} gen={t1-t0:.2f}s sel={t3-t2:.3f}s eval1={t4-t3:.3f}s eval2={t5-t4:.3f}s kernel={ms:.2f}/{ms2:.2f}ms steps={steps}")
    print(f"   params={ss.astuple()} s_eff={st.s_effective} L_S={st.series_len_S} sweeps={len(st.series_lens_F)} lensF[:4]={st.series_lens_F[:4]} matvecs={st.matvecs} |W|={np.linalg.norm(res.W):.6e}", flush=True)
    op.close()
