"""Paper m-sweep / k-sweep tables (budget 1000 n solutions) vs this build (scripts/quality_paper_tables.sh output).
usage: python scripts/paper_tables_report.py <dir with qp_*.json>"""
import json
import os
import sys

D = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
# PAPER.md:1170-1186 (ACS-GPU-Alt, m = 256) and PAPER.md:1136-1146 (Alt, k = 1, m sweep): mean / min %
ALT_K = {"nrw1379": {1: (4.189, 3.019), 2: (4.266, 3.321), 4: (4.223, 3.060), 8: (4.474, 3.395), 16: (4.718, 3.464)},
         "pr2392": {1: (5.290, 3.374), 2: (6.249, 3.413), 4: (7.077, 3.798), 8: (8.331, 4.797), 16: (8.404, 4.801)}}
ALT_M = {"nrw1379": {128: (4.351, 3.476), 512: (4.332, 3.282), 1024: (4.289, 2.949)},
         "pr2392": {128: (6.174, 4.209), 512: (5.631, 3.904), 1024: (6.609, 4.245)}}
SPM_K16 = {"nrw1379": 3.72, "pr2392": 4.66}  # PAPER.md:1235-1238 (figure; only k = 16 quoted)


def rec(path, key):
    p = os.path.join(D, path)
    if not os.path.exists(p):
        return None
    return json.load(open(p))["results"].get(key)


rows = []
print("| instance | setting | paper Alt mean / min | relaxed (ours) mean / min | paper SPM | spm (ours) mean / min |")
print("|---|---|---|---|---|---|")
for inst in ("nrw1379", "pr2392"):
    for k in (1, 2, 4, 8, 16):
        r = rec(f"qb_{inst}_m256_k{k}.json", f"{inst}/relaxed")
        s = rec(f"qb_{inst}_m256_k{k}.json", f"{inst}/spm")
        pa = ALT_K[inst][k]
        ps = f"{SPM_K16[inst]:.2f}" if k == 16 else "(figure)"
        fr = f"{r['mean_pct']:.2f} / {r['min_pct']:.2f}" if r else "—"
        fs = f"{s['mean_pct']:.2f} / {s['min_pct']:.2f}" if s else "—"
        print(f"| {inst} | m=256, k={k} | {pa[0]:.2f} / {pa[1]:.2f} | {fr} | {ps} | {fs} |")
        rows.append({"instance": inst, "m": 256, "k": k, "paper_alt": pa, "relaxed": r and [r["mean_pct"], r["min_pct"]],
                     "paper_spm_mean": SPM_K16[inst] if k == 16 else None, "spm": s and [s["mean_pct"], s["min_pct"]]})
    for m in (128, 512, 1024):
        r = rec(f"qb_{inst}_m{m}_k1.json", f"{inst}/relaxed")
        pa = ALT_M[inst][m]
        fr = f"{r['mean_pct']:.2f} / {r['min_pct']:.2f}" if r else "—"
        print(f"| {inst} | m={m}, k=1 | {pa[0]:.2f} / {pa[1]:.2f} | {fr} | | |")
        rows.append({"instance": inst, "m": m, "k": 1, "paper_alt": pa, "relaxed": r and [r["mean_pct"], r["min_pct"]]})
if len(sys.argv) > 2:
    json.dump(rows, open(sys.argv[2], "w"), indent=1)
