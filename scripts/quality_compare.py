#!/usr/bin/env python
"""Quality parity table: GPU variant vs the CPU oracle's matching mode.

Each row pairs a GPU result (tools/quality.py JSON) with an oracle result
(tests/studies/oracle_quality.py JSON) on the same instance and settings and
reports mean / min % over optimum, the difference of means, the two-sided
Wilcoxon rank-sum p-value (the paper's test) and whether the pair is within
the stated tolerance:  |mean_gpu - mean_oracle| <= TOL_PP percentage points
OR the rank-sum test does not reject equality at 0.05.

    python scripts/quality_compare.py --pair d198/atomic=gpu.json:d198/oracle-relaxed=orc.json ... \
        --out profiles/quality_parity_r01.json
"""
import argparse
import json

from scipy.stats import mannwhitneyu

TOL_PP = 0.5


def load(spec):
    key, path = spec.split("=", 1)
    rec = json.load(open(path))["results"][key]
    return key, path, rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pair", action="append", required=True,
                    help="GPUKEY=gpu.json:ORACLEKEY=oracle.json[:label]")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for spec in a.pair:
        parts = spec.split(":")
        (gk, gp, g), (ok, op, o) = load(parts[0]), load(parts[1])
        label = parts[2] if len(parts) > 2 else ""
        p = float(mannwhitneyu(g["lengths"], o["lengths"], alternative="two-sided").pvalue)
        d = g["mean_pct"] - o["mean_pct"]
        rows.append({"label": label, "gpu": gk, "gpu_file": gp, "oracle": ok, "oracle_file": op,
                     "gpu_mean": g["mean_pct"], "gpu_min": g["min_pct"], "gpu_runs": len(g["lengths"]),
                     "oracle_mean": o["mean_pct"], "oracle_min": o["min_pct"], "oracle_runs": len(o["lengths"]),
                     "diff_pp": round(d, 3), "p": round(p, 4),
                     "within": abs(d) <= TOL_PP or p >= 0.05})
    print("| setting | GPU | oracle | GPU mean / min | oracle mean / min | diff (pp) | rank-sum p | within |")
    print("|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['label']} | {r['gpu']} ({r['gpu_runs']}) | {r['oracle']} ({r['oracle_runs']}) | "
              f"{r['gpu_mean']:.2f} / {r['gpu_min']:.2f} | {r['oracle_mean']:.2f} / {r['oracle_min']:.2f} | "
              f"{r['diff_pp']:+.2f} | {r['p']:.3f} | {'yes' if r['within'] else 'NO'} |")
    if a.out:
        json.dump({"tolerance": f"|diff| <= {TOL_PP} pp or rank-sum p >= 0.05", "rows": rows},
                  open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
