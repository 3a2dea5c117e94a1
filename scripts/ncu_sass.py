"""Top SASS instructions by warp-stall samples with the dominant stall reasons.
usage: ncu_sass.py sass.csv [top]   (ncu --page source --csv --print-source sass)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
tot = {r: 0 for r in reasons}
all_samples = 0
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    all_samples += s
    rs = {k: int(r[ix[k]] or 0) for k in reasons}
    for k, v in rs.items():
        tot[k] += v
    data.append((s, r[ix["Address"]][-5:], r[ix["Source"]].strip()[:60], rs, r[ix["Instructions Executed"]]))
print("total stall samples", all_samples)
print("by reason:", ", ".join(f"{k[6:]} {v / max(all_samples, 1) * 100:.1f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]))
for s, a, src, rs, ex in sorted(data, key=lambda d: -d[0])[:top]:
    rr = ", ".join(f"{k[6:]}:{v}" for k, v in sorted(rs.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{s / max(all_samples, 1) * 100:5.1f}% {a} {src:60s} ex={ex} [{rr}]")
