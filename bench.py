#!/usr/bin/env python
"""Benchmark of the B200 phi-combination hot path (BASELINE.json metric).

A step is one phimv_block evaluation (Alg. 3, phi_block.cpp:48-157) of the
configs[1] workload — 2D advection-diffusion, n = 1,048,576, FP64 CSR, p=3,
r=4, tol 1e-10 — with ScalingShift selected once beforehand and reused (as
the paper prescribes).  `value` = phi-combination blocks/s over
the whole job with V already resident in HBM; `e2e` = the same through the
C-ABI host-buffer call (pinned V in, W out, copies inside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: one process per GPU (torchrun); each rank evaluates its own
independent block (phi blocks are independent units, weak scaling, no
data-path collective); timing is the max over ranks.  --impl reference times
the CPU oracle (the reference cannot be compiled here: no Eigen) on the host
cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "φ-combination blocks/s"
UNIT = "blocks/s"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def measured_peak():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(cfg):
    """dram read+write bytes per launch of k_phimv_block from the committed
    ncu --set full capture summary (profiles/), or None."""
    p = os.path.join(HERE, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(f"cfg{cfg}")
        return float(e["dram_bytes_per_launch"]) if e else None
    except Exception:
        return None


class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML during the timed region."""

    def __init__(self, dev_index):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def max_over_ranks(x: float, dist=None, device="cpu") -> float:
    """Max of a per-rank timing over all ranks (the contract's max-over-ranks
    clock); identity without a process group."""
    if dist is None:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def algorithmic_bytes(wl, rec):
    """Algorithmic HBM bytes of one k_phimv_block launch,
    counting only bytes the kernel moves: init 16n(p+1) (V read, V row-major
    write -- Vw_1 = D_1 = S_1 is recomputed, not stored); the first S term
    CSR + 8n(p+1) + 24wn (V rows gathered, Vw/D'/S written), each further
    S term B_S = CSR + 48wn; promotion+assembly CSR + 8n(3r+1); each
    recovery term B_F = CSR + 32 fc n; each sweep end 8n(2fc + 2pr)."""
    n, p, r = wl.n, wl.p, wl.r
    w = (p + 1) * r
    fc = r if p == 0 else 2 * r
    csr = 12 * wl.nnz + 4 * (n + 1)
    b = 16 * n * (p + 1)
    if rec.series_len_S >= 2:
        b += csr + 8 * n * (p + 1) + 24 * w * n
    b += max(0, rec.series_len_S - 2) * (csr + 48 * w * n)
    b += csr + 8 * n * (3 * r + 1)
    for lf in rec.series_lens_F:
        b += lf * (csr + 32 * fc * n)
    b += len(rec.series_lens_F) * 8 * n * (2 * fc + 2 * p * r)
    return b


def run_reference(args):
    """CPU reference arm: the oracle (C++ restatement of the reference path;
    the reference needs Eigen, absent here) on the host cores."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    import oracle as O
    import paper_2509_26475_b200 as P  # workload generator only (input setup)
    wl = P.workload(args.config, args.size)
    op = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    ss = O.select_parameters(op, 61, wl.tol)
    # one untimed full evaluation calibrates the per-block cost in S terms
    t0 = time.perf_counter()
    _, rec = O.phimv_block(op, wl.t, wl.alpha, wl.V, wl.tol, ss)
    t_full1 = time.perf_counter() - t0
    w = (wl.p + 1) * wl.r
    full_units = (rec.series_len_S - 1) * w + wl.r + sum(2 * wl.r * lf for lf in rec.series_lens_F)
    k_cap = max(1, min(args.ref_terms, rec.series_len_S - 1))
    sample_units = k_cap * w
    # all host threads the memory allows (each evaluation holds ~10 n x w blocks)
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 64 << 30
    per = 12 * 8 * wl.n * w + (1 << 28)
    cores = os.cpu_count() or 1
    threads = max(1, min(cores, int(avail * 0.6 // per)))

    def one_step():
        done = [0] * threads

        def work(i):
            done[i] = O.phimv_block_prefix(op, wl.t, wl.alpha, wl.V, wl.tol, ss, k_cap)

        ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        one_step()
    tot = 0.0
    for _ in range(args.steps):
        tot += one_step()
    per_step = tot / args.steps
    # each step: `threads` concurrent samples of k_cap S terms; a full block
    # costs full_units/sample_units samples
    block_time = per_step * full_units / sample_units
    value = threads / block_time
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(wl, args),
        "cpu_baseline": {
            "value": value, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"{threads} concurrent single-thread oracle evaluations per step, each the "
                       f"first {k_cap} S-series terms of the block; block cost extrapolated by "
                       f"matvec units ({full_units}/{sample_units}); one untimed full "
                       f"evaluation took {t_full1:.2f} s on 1 core"),
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(wl, args):
    names = {1: "C1 1D Dirichlet Laplacian", 2: "C2 2D advection-diffusion 1024^2",
             3: "C3 3D convection-diffusion 256^3", 4: "C4 random sparse stiff",
             5: "C5 nonnormal upper bidiagonal"}
    return {"workload": names.get(wl.cfg, str(wl.cfg)) + (f" (size {wl.size})" if args.size else ""),
            "n": wl.n, "nnz": wl.nnz, "p": wl.p, "r": wl.r, "tol": wl.tol,
            "block_width": (wl.p + 1) * wl.r, "parallelism": f"replicas x{args.gpus}",
            "l2": "working set (Vw, D, D', S: 4 x n x w x 8 B) larger than the 126 MB L2; no flush"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--size", type=int, default=0)
    ap.add_argument("--ref-terms", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_2509_26475_b200 as P

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    wl = P.workload(args.config, args.size)
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av, device=local)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    params = P.select_parameters(op, 61, wl.tol)
    sel_s = time.perf_counter() - t0

    stream = torch.cuda.ExternalStream(op.stream_ptr(), device=torch.device("cuda", local))
    dV = torch.from_numpy(np.ascontiguousarray(wl.V.T)).to(f"cuda:{local}")  # (p+1, n) = col-major V
    dW = torch.empty((wl.r, wl.n), dtype=torch.float64, device=f"cuda:{local}")
    torch.cuda.synchronize()

    def step():
        return P.phimv_block_device(op, wl.t, wl.alpha, wl.p, dV.data_ptr(), wl.tol, params,
                                    dW.data_ptr())

    for _ in range(max(args.warmup, 0)):
        rec = step()
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches0 = P.kernel_launches()
    kms = []
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            rec = step()
            kms.append(P.last_eval_stats()[0])
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = P.kernel_launches() - launches0
    elapsed = ev0.elapsed_time(ev1) / 1e3
    barrier()
    elapsed_max = max_over_ranks(elapsed, dist, f"cuda:{local}")
    value = args.steps * world / elapsed_max

    # ---- e2e through the C-ABI host-buffer call: pinned V in, W out ----
    L = P.lib()
    hV = torch.from_numpy(np.ascontiguousarray(wl.V.T)).pin_memory()
    hW = torch.empty((wl.r, wl.n), dtype=torch.float64).pin_memory()
    tt = np.ascontiguousarray(wl.t)
    aa = np.ascontiguousarray(wl.alpha)
    ss = params._c()
    lens = np.zeros(max(1, rec.s_effective), dtype=np.int32)
    crec = P._Rec(0, 0, 0, lens.ctypes.data_as(P.i32p), lens.size, 0)
    dp = C.POINTER(C.c_double)

    def e2e_step():
        code = L.phx_phimv_block(op._h, wl.r, tt.ctypes.data_as(dp), aa.ctypes.data_as(dp), wl.p,
                                 C.cast(hV.data_ptr(), dp), wl.n, wl.tol, C.byref(ss),
                                 C.cast(hW.data_ptr(), dp), wl.n, C.byref(crec))
        P._check(code)

    e2e_steps = max(5, args.steps // 2)
    for _ in range(2):
        e2e_step()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_el = e0.elapsed_time(e1) / 1e3
    e2e_value = e2e_steps * world / max_over_ranks(e2e_el, dist, f"cuda:{local}")

    # ---- roofline of the dominant (only) kernel, k_phimv_block ----
    peak, peak_src = measured_peak()
    prec = P.RunRecord(rec.s_effective, rec.series_len_S, rec.series_lens_F, rec.matvecs)
    alg = algorithmic_bytes(wl, prec)
    kernel_s = statistics.mean(kms) / 1e3
    achieved = alg / kernel_s / 1e9
    traffic = ncu_traffic(args.config)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle as O
        oop = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
        oss = O.ScalingShift(*params.astuple())
        t0 = time.perf_counter()
        Wo, ro = O.phimv_block(oop, wl.t, wl.alpha, wl.V, wl.tol, oss)
        dt = time.perf_counter() - t0
        same = bool(np.array_equal(Wo, dW.cpu().numpy().T))
        cpu = {"value": 1.0 / dt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": (f"one full oracle phimv_block of the same block (1 thread, "
                          f"{dt:.2f} s); GPU W bitwise-equal to it: {same}")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, csrc/workloads.cpp)",
            "config": config_dict(wl, args),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_phimv_block", "peak_source": peak_src,
                         "alg_bytes_per_launch": alg, "kernel_ms": kernel_s * 1e3},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int(wl.n * (wl.p + 1) * 8),
                    "d2h_bytes_per_step": int(wl.n * wl.r * 8)},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "selection_s": sel_s,
            "run_record": {"s_effective": rec.s_effective, "series_len_S": rec.series_len_S,
                           "n_sweeps": len(rec.series_lens_F), "matvecs": rec.matvecs},
            "params": {"s": params.s, "xi": params.xi, "s0": params.s0, "r": params.r},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    op.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
