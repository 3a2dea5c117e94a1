"""Merge tools/quality.py result files run on disjoint seed ranges (same
instance/variant/settings) into one, recomputing mean / min % over optimum.
usage: python scripts/merge_quality.py out.json a.json b.json ..."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_02669_b200 as P  # noqa: E402

out, files = sys.argv[1], sys.argv[2:]
merged = {"params": [], "results": {}}
for f in files:
    d = json.load(open(f))
    merged["params"].append(d["params"])
    for key, r in d["results"].items():
        m = merged["results"].setdefault(key, {"lengths": [], "optimum": P.load_instance(key.split("/")[0]).optimum})
        m["lengths"] += r["lengths"]
for key, m in merged["results"].items():
    opt = m.get("optimum")
    m["best_len"] = int(min(m["lengths"]))
    m["mean_len"] = float(np.mean(m["lengths"]))
    m["runs"] = len(m["lengths"])
    if opt:
        err = [100.0 * (x - opt) / opt for x in m["lengths"]]
        m["mean_pct"] = round(float(np.mean(err)), 3)
        m["min_pct"] = round(float(np.min(err)), 3)
json.dump(merged, open(out, "w"), indent=1)
