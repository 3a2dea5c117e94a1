#!/bin/bash
# SPEC acceptance criteria 6-9 on the GPU through the
# bench-cli; reports land in gpurun_out/acc_*.{csv,json}.
mkdir -p gpurun_out
B=build/acs-bench
CAT=data/tsplib/optima.txt.gz
T=data/tsplib
[ -x $B ] || make -s tools
# 6: hit-ratio trend over s in {1,2,4,8}, 5 seeded RELAXED (spm) runs on a280
$B sweep --instance $T/a280.tsp.gz --optima $CAT --variant spm --iterations 200 --reps 5 \
  --sweep "s=1,2,4,8" --out gpurun_out/acc6_hit_ratio > /dev/null
# 7: update period on nrw1379, m=256, 15 runs at k=1 and k=4 (relaxed, ACS-GPU-Alt)
$B sweep --instance $T/nrw1379.tsp.gz --optima $CAT --variant relaxed --ants 256 --iterations 1000 \
  --reps 15 --sweep "k=1,4" --out gpurun_out/acc7_period > /dev/null
# 7b: the same at m = n (the paper's Table freq-quality, where k=4 is significantly better at nrw1379)
$B sweep --instance $T/nrw1379.tsp.gz --optima $CAT --variant relaxed --iterations 1000 \
  --reps 15 --sweep "k=1,4" --out gpurun_out/acc7b_period_mn > /dev/null
# 8: selective vs dense under equal wall-clock limits on a280, m=256, k=4, 15 runs each
$B compare --instance $T/a280.tsp.gz --optima $CAT --ants 256 --update-period 4 --time-limit-ms 1000 \
  --reps 15 --a "memory=dense,consistent=0" --b "memory=selective" --out gpurun_out/acc8_compare > /dev/null
# 9: RELAXED vs SEQ wall-clock at identical budget on rat783
$B solve --instance $T/rat783.tsp.gz --optima $CAT --mode seq --iterations 10 --format json \
  > gpurun_out/acc9_seq.json
$B solve --instance $T/rat783.tsp.gz --optima $CAT --mode relaxed --consistent 0 --iterations 10 --format json \
  > gpurun_out/acc9_relaxed.json
python - <<'PY'
import json
h = json.load(open("gpurun_out/acc6_hit_ratio.json"))
print("acc6 hit ratio by s:", [(p["point"], round(sum(r["hit_ratio"] for r in p["reports"]) / len(p["reports"]), 4)) for p in h])
for f in ("acc7_period", "acc7b_period_mn"):
    k = json.load(open(f"gpurun_out/{f}.json"))
    print(f, [(p["point"], p["mean_err_pct"], p["p_vs_baseline"], p["mark"]) for p in k])
c = json.load(open("gpurun_out/acc8_compare.json"))
print("acc8: dense", c["A"]["mean_err_pct"], "selective", c["B"]["mean_err_pct"], "p", c["p_value"], "winner", c["winner"])
s = json.loads(open("gpurun_out/acc9_seq.json").read().splitlines()[0])
r = json.loads(open("gpurun_out/acc9_relaxed.json").read().splitlines()[0])
print("acc9: seq total_ms", s["total_ms"], "relaxed total_ms", r["total_ms"], "speedup", round(s["total_ms"] / r["total_ms"], 1))
PY
