"""Static check of the construction loop's row prefetch: for every
LDG.E.128.CONSTANT (packed row load) in the dense/SPM construction kernels,
print how many instructions issue before the first one that reads its
destination registers.  A consumer right after the load (a phi copy) makes
the warp wait on L2 there instead of overlapping the step's bookkeeping.
usage: sass_loaduse.py lib.so"""
import re
import subprocess
import sys

lib = sys.argv[1]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
fn, insts = None, []
funcs = {}
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        fn = m.group(1)
        funcs[fn] = []
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
    if m and fn:
        funcs[fn].append(m.group(1).strip())
for fn, ins in funcs.items():
    if "construct" not in fn and "k_deferred" not in fn:
        continue
    short = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()[:70]
    for i, s in enumerate(ins):
        m = re.match(r"(@!?P\d\s+)?LDG\.E\.(128|64|)\.?CONSTANT R(\d+),", s)
        if not m:
            continue
        base = int(m.group(3))
        regs = {f"R{base + j}" for j in range({"128": 4, "64": 2, "": 1}[m.group(2)])}
        dist = None
        for j in range(i + 1, min(i + 400, len(ins))):
            srcs = ins[j].split(",", 1)[1] if "," in ins[j] else ""
            toks = set(re.findall(r"\bR\d+", srcs))
            if "STG" in ins[j] or "RED" in ins[j] or "ATOM" in ins[j]:
                toks |= set(re.findall(r"\bR\d+", ins[j]))
            if toks & regs:
                dist = j - i
                break
        print(f"{short:72s} load@{i:5d}  first use after {dist} instr: {ins[i + dist] if dist else '-'}")
