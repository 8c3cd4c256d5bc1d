"""Developer script: host overhead of one phimv_block call on a small
operator (wall time per call vs the kernel's event time)."""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_2509_26475_b200 as P  # noqa: E402

for cfg, size in [(2, 50), (1, 300), (2, 16)]:
    wl = P.workload(cfg, size)
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = P.select_parameters(op, 61, wl.tol)
    req = P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)
    for _ in range(5):
        P.phimv_block(op, req)
    N = 200
    t0 = time.perf_counter()
    for _ in range(N):
        P.phimv_block(op, req)
    wall = (time.perf_counter() - t0) / N * 1e6
    ms, steps = P.last_eval_stats()
    print(f"cfg{cfg} n={wl.n} steps={steps}: wall {wall:.1f} us/call, kernel {ms * 1e3:.1f} us, "
          f"host+copies {wall - ms * 1e3:.1f} us", flush=True)

# device-resident buffers: no V/W copies, no numpy conversions of the block
import torch  # noqa: E402

for cfg, size in [(2, 50), (2, 16)]:
    wl = P.workload(cfg, size)
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = P.select_parameters(op, 61, wl.tol)
    V = np.asfortranarray(wl.V)
    dV = torch.from_numpy(V.T.copy()).cuda()  # column-major n x (p+1)
    dW = torch.empty(len(np.atleast_1d(wl.t)), wl.n, dtype=torch.float64, device="cuda")
    args = (op, wl.t, wl.alpha, V.shape[1] - 1, dV.data_ptr(), wl.tol, ss, dW.data_ptr())
    for _ in range(5):
        P.phimv_block_device(*args)
    N = 200
    t0 = time.perf_counter()
    for _ in range(N):
        P.phimv_block_device(*args)
    wall = (time.perf_counter() - t0) / N * 1e6
    ms, steps = P.last_eval_stats()
    print(f"device cfg{cfg} n={wl.n} steps={steps}: wall {wall:.1f} us/call, kernel {ms * 1e3:.1f} us, "
          f"host {wall - ms * 1e3:.1f} us", flush=True)
