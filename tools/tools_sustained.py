"""Developer A/B under sustained load (the bench's condition): back-to-back
device-resident evaluations of one config per setting, with NVML clock and
power samples.  python tools/tools_sustained.py cfg:size reps VAR=a,b [VAR2=c,d]
(VAR*_AT_CREATE: set before the operator is created)."""
import os
import statistics
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2509_26475_b200 as P  # noqa: E402

cfg, size = map(int, sys.argv[1].split(":"))
reps = int(sys.argv[2])
settings = [[]]
for arg in sys.argv[3:]:
    var, vals = arg.split("=")
    settings = [s + [(var, v)] for s in settings for v in vals.split(",")]
wl = P.workload(cfg, size)
import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for st in settings:
    for var, v in st:
        os.environ[var.replace("_AT_CREATE", "")] = v
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = P.select_parameters(op, 61, wl.tol)
    dV = torch.from_numpy(np.ascontiguousarray(wl.V.T)).cuda()
    dW = torch.empty((wl.r, wl.n), dtype=torch.float64, device="cuda")
    samples = []
    stop = threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            stop.wait(0.02)
    th = threading.Thread(target=sampler)
    th.start()
    ms = []
    for _ in range(reps):
        P.phimv_block_device(op, wl.t, wl.alpha, wl.p, dV.data_ptr(), wl.tol, ss, dW.data_ptr())
        ms.append(P.last_eval_stats()[0])
    stop.set()
    th.join()
    tail = ms[len(ms) // 3:]
    clk = [c for c, _ in samples[len(samples) // 3:]]
    pw = [p for _, p in samples[len(samples) // 3:]]
    print(f"cfg{cfg} {st}: median {statistics.median(tail):.2f} ms (first {ms[0]:.2f}) "
          f"sm_mhz median {statistics.median(clk) if clk else 0} power median "
          f"{statistics.median(pw) if pw else 0:.0f} W  var {P.last_eval_variant()['dynamic_tail']}",
          flush=True)
    op.close()
