"""Developer script: kernel time, algorithmic bytes (bench.algorithmic_bytes)
and achieved GB/s of one evaluation per config (cfg:size arguments).  Run it
plain for the numbers, and under `ncu --set full -k regex:k_phimv_block -c 1`
for the DRAM traffic of the same launch."""
import json
import sys

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
import paper_2509_26475_b200 as P  # noqa: E402

for arg in [x for x in sys.argv[1:] if not x.startswith("--")]:
    cfg, size = map(int, arg.split(":"))
    wl = P.workload(cfg, size)
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = P.select_parameters(op, 61, wl.tol)
    req = P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)
    res = P.phimv_block(op, req)
    ms, steps = P.last_eval_stats()
    if "--once" not in sys.argv:
        res = P.phimv_block(op, req)
        ms, steps = P.last_eval_stats()
    bulk = P.last_eval_variant()["dynamic_tail"] == 2
    b = bench.algorithmic_bytes(wl, res.stats, bulk)
    print(json.dumps({"cfg": cfg, "n": wl.n, "nnz": wl.nnz, "p": wl.p, "r": wl.r, "kernel": "k_phimv_bulk" if bulk else "k_phimv_block", "kernel_ms": ms,
                      "grid_steps": steps, "s_eff": res.stats.s_effective,
                      "L_S": res.stats.series_len_S, "sweeps": len(res.stats.series_lens_F),
                      "alg_bytes": b, "alg_GBps": b / (ms * 1e-3) / 1e9,
                      "frac_of_6547.5": b / (ms * 1e-3) / 1e9 / 6547.5}), flush=True)
    op.close()
