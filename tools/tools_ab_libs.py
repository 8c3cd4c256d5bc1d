"""Developer A/B across builds and runtime knobs on one box: for each
(PHX_LIB, env) setting a fresh process runs `reps` device-resident evaluations
of one config; settings are visited round-robin `rounds` times, so box drift
hits all of them alike.  Prints the per-setting median kernel time and checks
W bitwise across settings.
python tools/tools_ab_libs.py cfg:size reps rounds 'LIB[,VAR=v...]' ..."""
import hashlib
import json
import os
import statistics
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, "/root/repo")
    import numpy as np
    import paper_2509_26475_b200 as P
    cfg, size = map(int, sys.argv[2].split(":"))
    reps = int(sys.argv[3])
    wl = P.workload(cfg, size)
    op = P.CsrOperator(wl.n, wl.rp, wl.ci, wl.av)
    ss = P.select_parameters(op, 61, wl.tol)
    req = P.BlockPhiRequest(wl.t, wl.alpha, wl.V, wl.tol, ss)
    ts = []
    for _ in range(reps):
        r = P.phimv_block(op, req)
        ts.append(P.last_eval_stats()[0])
    h = hashlib.sha256(np.asfortranarray(r.W).tobytes(order="F")).hexdigest()[:16]
    print(json.dumps({"ts": ts[1:], "sha": h, "var": P.last_eval_variant(),
                      "L_S": r.stats.series_len_S}), flush=True)
    sys.exit(0)

cfgsize, reps, rounds = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
settings = sys.argv[4:]
res = {s: [] for s in settings}
shas = {}
for _ in range(rounds):
    for s in settings:
        parts = s.split(",")
        env = dict(os.environ)
        if parts[0] and parts[0] != "default":
            env["PHX_LIB"] = parts[0]
        for kv in parts[1:]:
            k, v = kv.split("=")
            env[k] = v
        out = subprocess.run([sys.executable, __file__, "--child", cfgsize, str(reps)], env=env,
                             capture_output=True, text=True)
        line = [x for x in out.stdout.splitlines() if x.startswith("{")]
        if not line:
            print(s, "FAILED", out.stderr[-2000:], flush=True)
            continue
        d = json.loads(line[-1])
        res[s] += d["ts"]
        shas[s] = d["sha"]
        print(s, [round(x, 2) for x in d["ts"]], d["sha"], d["var"], flush=True)
for s in settings:
    if res[s]:
        print(f"{cfgsize} {s}: median {statistics.median(res[s]):.3f} ms min {min(res[s]):.3f} "
              f"(n={len(res[s])}) sha {shas.get(s)}", flush=True)
print("bitwise equal across settings:", len(set(shas.values())) == 1, flush=True)
