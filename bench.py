#!/usr/bin/env python
"""Benchmark: constructed tours/sec at pr2392 (ACS, 2392 ants, cl=32, k=1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--variant atomic]
    python bench.py --impl reference ...      # CPU reference arm (oracle port, all host threads)

One step = one ACS iteration of the colony: m = n = 2392 tours constructed
(warp per ant, whole tour per launch), iteration best, global-best update.
Under torchrun (N > 1) every rank runs its own colony on its own GPU (island
model); colonies exchange the global best through NCCL every
--exchange-every iterations inside the timed region.  value = all tours built
by all ranks / max over ranks of the device time.  L2 is flushed (256 MiB
write) before every timed step; each step is timed with CUDA events on the
colony stream (acs_gpu_last_timing).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "constructed tours/sec at pr2392 (1/2/4/8 B200); mean % over optimum"
PAPER_ACS_GPU_PR2392 = 4942.0  # ACS-GPU (atomic) pr2392, GK104


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--instance", default="pr2392")
    ap.add_argument("--variant", default="atomic")
    ap.add_argument("--ants", type=int, default=0)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--rng", default="auto", choices=["auto", "philox", "xoshiro"],
                    help="per-ant stream of the GPU arm; auto = philox (counter-based, 32 draws per "
                         "warp evaluation) for atomic/relaxed, xoshiro (the reference RngStream) otherwise")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--exchange-every", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    return ap.parse_args()


def data_desc(name: str) -> str:
    if name.startswith("rnd"):
        return f"synthetic {name}: uniform integer coordinates in [0,1e6)^2 from RngStream(20161017)"
    return f"TSPLIB {name} (real instance, data/tsplib)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5:  # first sample before timing starts
                time.sleep(0.02)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic_bytes_per_tour(n: int, L: int, k: int, variant: str, slots: int = 8) -> int:
    """B = n*(cl*(4+S) + 4) + ceil(n/k)*4S (dense) with S = 8;
    selective: n*(cl*(4+S) + s*(4+S) + 8) + ceil(n/k)*2*(s*4 + S + 4).
    The fallback term F is added from the device counter by the caller."""
    S = 8
    upd = -(-n // k)
    if variant in ("spm", "spm-seq", "spm-sync"):
        return n * (L * (4 + S) + slots * (4 + S) + 8) + upd * 2 * (slots * 4 + S + 4)
    return n * (L * (4 + S) + 4) + upd * 4 * S


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


def ncu_record(variant: str) -> dict:
    """The committed ncu --set full summary of this variant's construct kernel."""
    path = os.path.join(REPO, "profiles", "ncu_construct_summary.json")
    try:
        with open(path) as f:
            return json.load(f).get(variant, {})
    except (OSError, ValueError):
        return {}


def ncu_traffic(variant: str):
    """dram bytes per construct launch from the committed ncu --set full capture."""
    return ncu_record(variant).get("dram_bytes_per_launch")


def cpu_baseline_seq(name: str, m: int, k: int):
    """oracle SEQ (ACS-SEQ restated) on one host core, bounded sample."""
    import oracle as O
    I = O.load(name)
    # bounded sample (~10-20 s of one core): 7 full iterations up to pr2392,
    # one iteration of a 1000-ant colony beyond
    iters, m_s = (7, m) if I.n <= 4096 else (1, min(m, 1000))
    o = O.Oracle().run(I, m=m_s, iterations=iters, seed=0, mode=O.SEQ, k=k, want_routes=False)
    tps = m_s * iters / (o["loop_ms"] / 1e3)
    return {"value": round(tps, 1), "unit": "tours/s", "cores": 1, "kind": "port",
            "sample": f"oracle SEQ (ant-major, immediate updates) on {name}, m={m_s}, k={k}, "
                      f"{iters} iterations = {m_s * iters} tours, {o['loop_ms'] / 1e3:.1f} s"}


def run_reference(args):
    """--impl reference: the CPU port of the reference path on all host threads."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O
    I = O.load(args.instance)
    m = args.ants or I.n
    threads = os.cpu_count() or 1
    mode = O.SEQ if args.variant in ("seq", "spm-seq") else (
        O.SYNC if args.variant in ("deferred", "spm-sync") else O.RELAXED)
    memory = O.SELECTIVE if args.variant in ("spm", "spm-seq", "spm-sync") else O.DENSE
    consistent = 1 if args.variant == "atomic" else 0
    orc = O.Oracle()
    # Each step is one ACS iteration of a bounded sample of the colony
    # (min(m, 1024) ants) so that --steps K --warmup W stays within minutes;
    # the metric is per tour, so the sample does not bias it.  The oracle keeps
    # no state across calls: every step is a fresh single-iteration colony.
    m_step = min(m, 1024)
    for w in range(args.warmup):
        orc.run(I, m=m_step, iterations=1, seed=args.seed + 1000 + w, mode=mode, memory=memory,
                consistent=consistent, threads=threads, k=args.k, want_routes=False)
    loop_ms = []
    for st in range(args.steps):
        o = orc.run(I, m=m_step, iterations=1, seed=args.seed + st, mode=mode, memory=memory,
                    consistent=consistent, threads=threads, k=args.k, want_routes=False)
        loop_ms.append(o["loop_ms"])
    total_s = sum(loop_ms) / 1e3
    value = m_step * args.steps / total_s
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "tours/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sum(loop_ms) / args.steps * m / m_step, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": data_desc(args.instance),
        "config": {"workload": f"{args.instance} ACS, {m} ants, cl=32, k={args.k}, {args.variant}",
                   "variant": args.variant, "mode": ["seq", "sync", "relaxed"][mode],
                   "memory": ["dense", "selective"][memory], "consistent": consistent},
        "cpu_baseline": {"value": round(value, 1), "unit": "tours/s", "cores": threads, "kind": "port",
                         "sample": f"oracle/acs_oracle.c OpenMP on {threads} host threads, "
                                   f"{args.steps} iterations x {m_step} of {m} ants per step"},
        "e2e": {"value": round(value, 1), "unit": "tours/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def rng_for(variant: str, rng: str) -> str:
    if rng != "auto":
        return rng
    return "philox" if variant in ("atomic", "relaxed") else "xoshiro"


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)

    rank, world, local = dist_env()
    import numpy as np
    import torch
    import paper_1605_02669_b200 as P

    # one GPU per rank; if the ranks outnumber the visible GPUs (a test of the
    # multi-rank path on one device) they share GPUs and exchange on the host
    # over gloo (NCCL refuses two ranks on one device)
    ndev = max(1, torch.cuda.device_count())
    shared = world > ndev
    local = local % ndev
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    inst = P.load_instance(args.instance)
    opt = inst.optimum
    m = args.ants or inst.n
    # P11: colony c uses seed + c * golden -> colony 0 == the single-GPU run
    seed = (args.seed + rank * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    params = P.AcsParams(variant=args.variant, m=m, k=args.k, seed=seed, rng=rng_for(args.variant, args.rng))
    col = P.Colony(inst, params, device=local)
    exchange = None
    if world > 1:
        if shared:
            exchange = "host (gloo; ranks share a GPU)"
        else:
            uid = [P.Colony.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            col.island_init(uid[0], world, rank)
            exchange = "device (NCCL inside libacs_b200)"

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    # our kernels per iteration: construction (1 launch; deferred = 1 cooperative
    # launch) + k_best + global update (+ k_fold_counts for atomic)
    launches_per_iter = 3 + (1 if args.variant == "atomic" else 0)

    def step(i):
        flush.fill_(i & 0xFF)  # evict L2 (126 MB) before the step
        torch.cuda.synchronize()
        col.iterate(1)
        tot, con = col.last_timing()
        ex = 0
        if world > 1 and (i + 1) % args.exchange_every == 0:
            t0 = time.perf_counter()
            if shared:
                P.island.exchange_host(col, dist)
            else:
                col.island_exchange()
            ex = (time.perf_counter() - t0) * 1e3
        return tot + ex, con

    for i in range(args.warmup):
        step(i)
    c0 = col.counters()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        per = [step(args.warmup + i) for i in range(args.steps)]
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    c1 = col.counters()
    total_ms = sum(p[0] for p in per)
    construct_ms = sum(p[1] for p in per)
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cpu" if shared else f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * m * args.steps / (total_ms / 1e3)
    order, best_len = col.best()

    # roofline of the dominant kernel (construction): algorithmic bytes / launch time
    fb_elems = c1.get("fallback_elems", 0) - c0.get("fallback_elems", 0)
    B_tour = algorithmic_bytes_per_tour(inst.n, col.info.list_len, args.k, args.variant)
    alg_bytes_launch = B_tour * m + fb_elems * 12 / max(args.steps, 1)
    construct_s = construct_ms / 1e3 / args.steps
    peaks, src = measured_peaks()
    achieved = alg_bytes_launch / construct_s / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": ncu_traffic(args.variant),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src})",
                "kernel": "k_construct_dense" if args.variant != "spm" else "k_construct_spm",
                "construct_ms_per_launch": round(construct_s * 1e3, 4),
                "bytes_per_tour": B_tour,
                "note": "latency-bound dependent-load chain; L2-resident working set"}
    # the working set is L2-resident: the same bytes against the
    # measured L2 read bandwidth, and the ncu L2 read traffic per launch
    l2_gbs = P._native.l2_read_bandwidth(local, 48 << 20)
    rec = ncu_record(args.variant)
    sectors = rec.get("lts__t_sectors_srcunit_tex_op_read.sum")
    roofline["l2"] = {"peak": round(l2_gbs, 1), "unit": "GB/s", "achieved": round(achieved, 1),
                      "frac": round(achieved / l2_gbs, 4),
                      "peak_source": "acs_gpu_l2_read_bandwidth: ld.global.cg stream over a 48 MiB "
                                     "L2-resident buffer, measured in this run",
                      "ncu_l2_read_bytes_per_launch": sectors * 32 if sectors else None}

    # The construction loop is a dependent chain per ant, so its practical
    # ceiling is instruction issue (one warp instruction per SM sub-partition
    # per cycle), not bytes: executed warp instructions per launch (committed
    # ncu capture) / measured launch time, against 4 x SMs x SM clock.
    n_inst = rec.get("instructions")
    clk_mhz = clk.summary().get("sm_mhz")
    if n_inst and clk_mhz:
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        peak_ips = 4 * sms * clk_mhz * 1e6
        roofline["issue"] = {"achieved": round(n_inst / construct_s / 1e12, 4), "peak": round(peak_ips / 1e12, 4),
                             "unit": "T warp-inst/s", "frac": round(n_inst / construct_s / peak_ips, 4),
                             "inst_per_launch": n_inst,
                             "source": "ncu --set full 'Executed Instructions' of this variant's construct kernel "
                                       "(profiles/ncu_construct_summary.json) / this run's launch time; peak = "
                                       "4 schedulers x SMs x median SM clock under load"}
    # Latency bound: every ant is a chain of n-1 dependent steps, so no colony
    # can construct faster than ONE isolated ant's tour.  A 128-ant colony
    # (< 1 ant per SM, no issue contention) of the same variant measures that
    # chain in this run; frac = its construct time / the full colony's.
    p_lat = P.AcsParams(variant=args.variant, m=128, k=args.k, seed=args.seed, rng=rng_for(args.variant, args.rng))
    with P.Colony(inst, p_lat, device=local) as lc:
        lc.iterate(2)
        lat = []
        for i in range(5):
            flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            lc.iterate(1)
            lat.append(lc.last_timing()[1])
    lat_ms = statistics.median(lat)
    roofline["latency"] = {"bound_ms": round(lat_ms, 4), "achieved_ms": round(construct_s * 1e3, 4),
                           "frac": round(lat_ms / (construct_s * 1e3), 4),
                           "source": "construct time of a 128-ant colony (same variant, < 1 ant per SM: the "
                                     "isolated dependent chain of n-1 steps), median of 5, measured in this run"}
    col.close()
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "tours/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": round(value / PAPER_ACS_GPU_PR2392, 2) if args.instance == "pr2392" and args.variant == "atomic" else None,
        "vs_baseline_ref": "paper ACS-GPU (atomic) pr2392 4942 tours/s on GK104 (BASELINE.md, PAPER.md:920)",
        "dtype": "f64", "data": data_desc(args.instance),
        "config": {"workload": f"{args.instance} ACS, {m} ants, cl=32, k={args.k}, {args.variant} dense"
                   if args.variant != "spm" else f"{args.instance} ACS-SPM, {m} ants, s=8",
                   "instance": args.instance, "n": inst.n, "ants_per_gpu": m, "variant": args.variant,
                   "cl": 32, "k": args.k, "beta": 3.0, "alpha": 0.2, "rho": 0.01,
                   "q0": round(col.info.q0, 6), "rng": rng_for(args.variant, args.rng), "l2": "flushed (256 MiB write) before every timed step",
                   "parallelism": f"island x{world}" if world > 1 else "single colony",
                   "exchange_every": args.exchange_every if world > 1 else None, "exchange": exchange},
        "roofline": roofline,
        "gpu_launches": launches_per_iter * args.steps,
        "clocks": clk.summary(),
        "counters_per_step": {k: round((c1[k] - c0[k]) / args.steps, 1) for k in c1 if k != "iterations"},
        "quality": {"best_len": int(best_len), "optimum": opt,
                    "pct_over_opt": round(100.0 * (best_len - opt) / opt, 3) if opt else None,
                    "iterations": args.warmup + args.steps, "seeds": 1,
                    "note": "single run; 30-seed study in profiles/quality_*.json"},
    }
    if rank == 0 and not args.no_variants:
        line["variants"] = other_variants(P, inst, args, local)
    if not args.no_e2e:  # every rank: whole-job figure from the max wall time over ranks
        e = e2e(P, inst, params, args, world, dist, local, shared)
        if rank == 0:
            line["e2e"] = e
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_seq(args.instance, m, args.k)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def other_variants(P, inst, args, device):
    """Secondary numbers: the other pheromone memories on the same workload
    (same flush + per-step event timing, 5 steps each)."""
    import torch
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{device}")
    out = {}
    for v in ("atomic", "relaxed", "spm", "deferred"):
        if v == args.variant:
            continue
        p = P.AcsParams(variant=v, m=args.ants or inst.n, k=args.k, seed=args.seed, rng=rng_for(v, args.rng))
        with P.Colony(inst, p, device=device) as col:
            col.iterate(2)
            ms = []
            for i in range(5):
                flush.fill_(i)
                torch.cuda.synchronize()
                col.iterate(1)
                ms.append(col.last_timing()[0])
        t = sum(ms) / len(ms)
        out[v] = {"ms_per_step": round(t, 4), "tours_per_s": round(col.m / (t / 1e3), 1)}
    return out


def e2e(P, inst, params, args, world, dist=None, device=0, shared=False):
    """Same metric through the public C-ABI with HOST buffers: create (host
    coordinates H2D, setup kernels), then every step one acs_gpu_iterate(ctx,
    1, &stats) with that step's result (iteration best, L_gb: 24 B) read back
    to the host, then the best tour D2H and destroy -- all inside the timed
    region.  Every rank runs its own colony at the same time; the whole-job
    value uses the max wall time over ranks.  Repeated 3 times (host wall
    clocks on the box jitter by tens of ms); the median is reported."""
    import ctypes as C
    import numpy as np
    from paper_1605_02669_b200 import _native as N
    K = args.steps
    d = inst.desc()
    p = params.to_c(inst.n)
    order = np.empty(inst.n, np.uint32)
    bl = C.c_int64()
    stat = N.IterStats()
    lib = N.lib()

    def one(k):
        h = C.c_void_p()
        N.check(lib.acs_gpu_create(C.byref(d), C.byref(p), device, C.byref(h)), "acs_gpu_create")
        try:
            for _ in range(k):
                N.check(lib.acs_gpu_iterate(h, 1, C.byref(stat)), "acs_gpu_iterate")
            N.check(lib.acs_gpu_get_best(h, order.ctypes.data_as(C.c_void_p), C.byref(bl)), "acs_gpu_get_best")
        finally:
            lib.acs_gpu_destroy(h)

    one(1)  # untimed: lazy CUDA module loading of the setup kernels
    walls = []
    for _ in range(3):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        one(K)
        dt = time.perf_counter() - t0
        if dist:
            import torch
            t = torch.tensor([dt], dtype=torch.float64, device="cpu" if shared else f"cuda:{device}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        walls.append(dt)
    dt = statistics.median(walls)
    m = p.ants
    return {"value": round(world * m * K / dt, 1), "unit": "tours/s",
            "h2d_bytes_per_step": round(2 * 8 * inst.n / K, 1),
            "d2h_bytes_per_step": round(C.sizeof(N.IterStats) + (4 * inst.n + 8) / K, 1),
            "api": f"acs_gpu_create + K x acs_gpu_iterate(ctx, 1, &stats) (per-step result D2H) + "
                   f"acs_gpu_get_best + acs_gpu_destroy, host buffers, on each of {world} rank(s); "
                   f"max wall over ranks, median of 3 runs",
            "wall_s": round(dt, 4), "wall_s_runs": [round(w, 4) for w in walls]}


if __name__ == "__main__":
    sys.exit(main())
