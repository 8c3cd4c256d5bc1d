"""Generate the golden fixtures under tests/golden/ from the CPU oracle.

The reference itself cannot be built or run here (it needs Eigen3, absent
from the image), so the fixtures pin the oracle restatement: every fixture is
(a) a bitwise record of the oracle's output on a seeded BASELINE workload
(ScalingShift, RunRecord, W or its SHA-256) and, where n + p <= 2000, (b) the
long-double augmented-matrix reference (reference_w, oracle.cpp:53-91
restated) that the oracle's W must match within the user tolerance.

Usage:  python tests/golden/make_golden.py [small] [highprec] [full2] [full4] [full3] [c5big]

c5big: C5 at n = 2^21 (419 recovery sweeps) -- the size from which the
production kernel variants run C5 -- with the oracle's row-parallel loops on
all host cores (bitwise those of one thread).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2509_26475_b200 as P  # noqa: E402  (workload generators only)

SMALL = [(1, 0), (2, 64), (3, 12), (4, 1024), (5, 2000), (1, 200)]
HIGHPREC = [(1, 0), (2, 44), (3, 12), (4, 1024), (5, 1990)]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.asfortranarray(a, dtype=np.float64).tobytes(order="F")).hexdigest()


def run_oracle(cfg, size):
    wl = P.workload(cfg, size)
    op = O.csr_from_arrays(wl.n, wl.rp, wl.ci, wl.av)
    t0 = time.time()
    ss = O.select_parameters(op, 61, wl.tol)
    t1 = time.time()
    W, rec, tr = O.phimv_block(op, wl.t, wl.alpha, wl.V, wl.tol, ss, trace=True)
    t2 = time.time()
    return wl, ss, W, rec, tr, (t1 - t0, t2 - t1)


def save_record(name, cfg, size, ss, W, rec, tr, store_W):
    meta = {
        "cfg": cfg, "size": size, "params": list(ss.astuple()),
        "s_effective": rec.s_effective, "series_len_S": rec.series_len_S,
        "series_lens_F": rec.series_lens_F, "matvecs": rec.matvecs,
        "W_sha256": sha(W), "trace_sha256": sha(tr), "n": int(W.shape[0]), "r": int(W.shape[1]),
    }
    idx = np.unique(np.linspace(0, W.shape[0] - 1, 64).astype(np.int64))
    arrays = {"sample_rows": idx, "sample_W": W[idx]}
    if store_W:
        arrays["W"] = W
        arrays["trace"] = tr
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)
    with open(os.path.join(HERE, name + ".json"), "w") as f:
        json.dump(meta, f, indent=1)


def small():
    for cfg, size in SMALL:
        wl, ss, W, rec, tr, dt = run_oracle(cfg, size)
        save_record(f"cfg{cfg}_s{wl.size}", cfg, size, ss, W, rec, tr, store_W=True)
        print(f"cfg{cfg} size {wl.size}: sel {dt[0]:.2f}s eval {dt[1]:.2f}s L_S={rec.series_len_S} "
              f"s_eff={rec.s_effective}", flush=True)


def dense_of(wl):
    A = np.zeros((wl.n, wl.n))
    for i in range(wl.n):
        A[i, wl.ci[wl.rp[i]:wl.rp[i + 1]]] += wl.av[wl.rp[i]:wl.rp[i + 1]]
    return A


def highprec():
    for cfg, size in HIGHPREC:
        wl = P.workload(cfg, size)
        A = dense_of(wl)
        t0 = time.time()
        Wref = np.empty((wl.n, wl.r))
        done = {}
        for i in range(wl.r):
            key = (float(wl.t[i]), float(wl.alpha[i]))
            if key not in done:
                done[key] = O.reference_w(A, wl.V, wl.t[i], wl.alpha[i])
            Wref[:, i] = done[key]
        np.savez_compressed(os.path.join(HERE, f"hp_cfg{cfg}_s{wl.size}.npz"), W_ref=Wref,
                            t=wl.t, alpha=wl.alpha)
        print(f"highprec cfg{cfg} size {wl.size}: {time.time() - t0:.1f}s", flush=True)


def full(cfg):
    wl, ss, W, rec, tr, dt = run_oracle(cfg, 0)
    save_record(f"full_cfg{cfg}", cfg, 0, ss, W, rec, tr, store_W=False)
    print(f"full cfg{cfg}: sel {dt[0]:.1f}s eval {dt[1]:.1f}s L_S={rec.series_len_S} "
          f"s_eff={rec.s_effective}", flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["small", "highprec"]
    for w in what:
        if w == "small":
            small()
        elif w == "highprec":
            highprec()
        elif w.startswith("full"):
            full(int(w[4:]))
        elif w == "c5big":
            O.set_threads(os.cpu_count() or 1)
            wl, ss, W, rec, tr, dt = run_oracle(5, 1 << 21)
            save_record("full_cfg5_s2097152", 5, 1 << 21, ss, W, rec, tr, store_W=False)
            print(f"c5big: sel {dt[0]:.1f}s eval {dt[1]:.1f}s L_S={rec.series_len_S} "
                  f"s_eff={rec.s_effective} sweeps={len(rec.series_lens_F)}", flush=True)
