"""Executed-instruction mix per SASS opcode of one kernel, from an ncu source
page (--page source --csv --print-source cuda,sass).
usage: ncu_opmix.py src.csv [units]   (units: divide counts, e.g. steps per launch)"""
import collections
import csv
import sys


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
ops, seen, tot = collections.Counter(), set(), 0.0
for r in rows:
    if len(r) < 8 or r[0] == "Line No" or not r[2]:
        continue
    if r[2] in seen:  # the same SASS address is listed under several CUDA lines
        continue
    seen.add(r[2])
    words = r[3].split()
    if not words:
        continue
    op = words[1] if words[0].startswith("@") and len(words) > 1 else words[0]
    c = num(r[7])
    ops[op.split(".")[0]] += c
    tot += c
for op, c in ops.most_common(30):
    print(f"{op:12s} {c / units:8.2f} {100 * c / tot:5.1f}%")
print(f"{'total':12s} {tot / units:8.2f}")
