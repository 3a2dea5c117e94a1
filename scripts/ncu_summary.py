#!/usr/bin/env python
"""Summarise an ncu --set full report (.ncu-rep) of one kernel into a small
JSON record + markdown table for profiles/.

    python scripts/ncu_summary.py gpurun_out/prof_x.ncu-rep --label atomic \
        --bytes-per-launch 2.4e9 [--json profiles/ncu_construct_summary.json]
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

METRICS = {
    "Duration": "duration",
    "DRAM Throughput": "dram_pct",
    "L2 Cache Throughput": "l2_pct",
    "L1/TEX Cache Throughput": "l1_pct",
    "Compute (SM) Throughput": "sm_pct",
    "Executed Ipc Active": "ipc_active",
    "Issue Slots Busy": "issue_busy_pct",
    "Warp Cycles Per Issued Instruction": "cycles_per_issue",
    "Executed Instructions": "instructions",
    "Avg. Active Threads Per Warp": "active_threads",
    "L1/TEX Hit Rate": "l1_hit_pct",
    "L2 Hit Rate": "l2_hit_pct",
    "Achieved Active Warps Per SM": "warps_per_sm",
    "Theoretical Active Warps per SM": "theoretical_warps_per_sm",
    "Registers Per Thread": "registers",
    "Grid Size": "grid",
    "Block Size": "block",
}


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def details(rep):
    rows = ncu_csv(rep, "--page", "details")
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    out = {"kernel": rows[1][ix["Kernel Name"]] if len(rows) > 1 else ""}
    for r in rows[1:]:
        name = r[ix["Metric Name"]]
        if name in METRICS:
            val = r[ix["Metric Value"]].replace(",", "")
            try:
                val = float(val)
            except ValueError:
                pass
            key = METRICS[name]
            unit = r[ix["Metric Unit"]]
            if key == "duration":
                val = val * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}.get(unit, 1.0)
            out[key] = val
    return out


def raw(rep):
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units = rows[0], rows[1]
    vals = rows[2]
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active"]
    out = {}
    for i, h in enumerate(hdr):
        if h in want:
            v = vals[i].replace(",", "")
            mult = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(units[i], 1.0)
            try:
                out[h] = float(v) * mult
            except ValueError:
                out[h] = v
    return out


def stalls(rep, top=12):
    rows = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = defaultdict(int)
    allsum = 0
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        allsum += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        for k in reasons:
            tot[k[6:]] += int(r[ix[k]] or 0)
    return {k: round(v / max(allsum, 1) * 100, 1) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--label", required=True)
    ap.add_argument("--bytes-per-launch", type=float, default=None,
                    help="algorithmic bytes per launch (SURVEY 8(d)) for the achieved-GB/s figure")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    d = details(a.rep)
    d.update(raw(a.rep))
    d["stall_pct"] = stalls(a.rep)
    rd = d.get("dram__bytes_read.sum", 0) or 0
    wr = d.get("dram__bytes_write.sum", 0) or 0
    d["dram_bytes_per_launch"] = rd + wr
    if a.bytes_per_launch and d.get("duration"):
        d["algorithmic_bytes_per_launch"] = a.bytes_per_launch
        d["achieved_gbs"] = a.bytes_per_launch / d["duration"] / 1e9
    d["source"] = os.path.basename(a.rep)
    print(json.dumps(d, indent=1))
    if a.json:
        db = {}
        if os.path.exists(a.json):
            db = json.load(open(a.json))
        db[a.label] = d
        json.dump(db, open(a.json, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
