"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line:
instructions executed and warp-stall samples.  usage: ncu_lines.py mix.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg, cur, hdr, fname = {}, None, None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1][:70])
        continue
    try:
        ex = int(r[hdr.index("Instructions Executed")] or 0)
        st = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0])
    a[0] += ex
    a[1] += st
tot_ex = sum(v[0] for v in agg.values()) or 1
tot_st = sum(v[1] for v in agg.values()) or 1
print(f"total inst {tot_ex}  stall samples {tot_st}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[1] / tot_st * 100:5.1f}% stall {v[0] / tot_ex * 100:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")
