"""Summarise an ncu --set full report of k_phimv_block (run here, no GPU):
python profiles/ncu_extract.py <report.ncu-rep> [label]"""
import csv
import io
import json
import subprocess
import sys
from collections import Counter

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def sass_mix(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    idx = {n: i for i, n in enumerate(h)}
    ops, stall = Counter(), Counter()
    tot = samp = 0
    for r in rows[2:]:
        try:
            ex = int(r[idx["Instructions Executed"]])
            s = int(r[idx["Warp Stall Sampling (All Samples)"]])
        except (ValueError, KeyError, IndexError):
            continue
        t = r[idx["Source"]].strip().split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        op = op.split(".")[0]
        ops[op] += ex
        stall[op] += s
        tot += ex
        samp += s
    return {op: (round(c / tot * 100, 1), round(stall[op] / max(samp, 1) * 100, 1))
            for op, c in ops.most_common(12)}


if __name__ == "__main__":
    rep = sys.argv[1]
    r = raw(rep)
    d = {k: r[k][0] + " " + r[k][1] for k in KEYS if k in r}
    rb = float(r["dram__bytes_read.sum"][0]) * {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[r["dram__bytes_read.sum"][1]]
    wb = float(r["dram__bytes_write.sum"][0]) * {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[r["dram__bytes_write.sum"][1]]
    d["dram_bytes_per_launch"] = rb + wb
    d["sass_mix_pct_instr_pct_stall"] = sass_mix(rep)
    print(json.dumps(d, indent=1))
