mkdir -p gpurun_out
compute-sanitizer --version 2>&1 | head -3
timeout 300 compute-sanitizer --tool memcheck --print-limit 10 python -c "
import sys; sys.path.insert(0,'.')
import paper_2509_26475_b200 as P
wl=P.workload(1,200); op=P.CsrOperator(wl.n,wl.rp,wl.ci,wl.av)
ss=P.select_parameters(op,61,wl.tol); r=P.phimv_block(op,P.BlockPhiRequest(wl.t,wl.alpha,wl.V,wl.tol,ss)); print('ok',r.stats.series_len_S)
" > gpurun_out/san_probe.log 2>&1; echo "san rc=$?"; tail -15 gpurun_out/san_probe.log
