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


def resident_ants(P, device: int, m: int) -> int:
    """Ants constructing at once (one warp each): 20 per SM with the 96-register
    build (5 warps per sub-partition), 28 with the 72-register build the
    launcher picks for colonies larger than one wave (k_colony.cu kWideRegs)."""
    import torch
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    return sms * 20 if m <= sms * 20 else sms * 28


def construct_kernel(variant: str, k: int) -> str:
    """The construction kernel the library launches for this workload (cl = 32)."""
    if variant == "deferred":
        return "k_deferred"
    if variant == "spm-sync":
        return "k_ssync_select"
    lean = k == 1
    if variant in ("spm", "spm-seq"):
        return "k_spm_lean" if lean and variant == "spm" else "k_construct_spm"
    return "k_tour_lean" if lean and variant in ("atomic", "relaxed") else "k_construct_dense"


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
    """--impl reference: the reference's path on the host cores, SAME workload
    as the GPU arm: one persistent colony of m ants on the same instance, the
    same variant semantics (SPEC mode x memory x contract) and the same per-ant
    RNG engine, W warm-up and K timed iterations of that one colony.  The
    oracle (oracle/acs_oracle.c, the CPU restatement of the reference path,
    OpenMP over all host threads) times every iteration itself (iter_ms)."""
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
    rng = rng_for(args.variant, args.rng)
    o = O.Oracle().run(I, m=m, iterations=args.warmup + args.steps, seed=args.seed, mode=mode,
                       memory=memory, consistent=consistent, threads=threads, k=args.k,
                       rng=O.PHILOX if rng == "philox" else O.XOSHIRO, want_routes=False)
    timed_ms = float(o["iter_ms"][args.warmup:].sum())
    value = m * args.steps / (timed_ms / 1e3)
    cfg = bench_config(args, I.n, m, world)
    cfg["reference_mode"] = {"mode": ["seq", "sync", "relaxed"][mode], "memory": ["dense", "selective"][memory],
                             "consistent": consistent}
    cpu = host_cpu_model()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "tours/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(timed_ms / args.steps, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": data_desc(args.instance),
        "config": cfg,
        "cpu_baseline": {"value": round(value, 1), "unit": "tours/s", "cores": threads, "kind": "port",
                         "cpu": cpu,
                         "sample": f"oracle/acs_oracle.c (OpenMP, {threads} threads on {cpu}): one persistent "
                                   f"{m}-ant colony, {args.warmup} warm-up + {args.steps} timed iterations "
                                   f"(per-iteration wall time), best L_gb {int(o['best_len'])}"},
        "e2e": {"value": round(value, 1), "unit": "tours/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def rng_for(variant: str, rng: str) -> str:
    if rng != "auto":
        return rng
    return "philox" if variant in ("atomic", "relaxed", "spm") else "xoshiro"


def default_q0(n: int) -> float:
    """SPEC D6 default q0 = (n - 20) / n (capi.cu default_q0)."""
    return 0.0 if n <= 20 else (n - 20) / n


def bench_config(args, n: int, m: int, world: int, exchange=None) -> dict:
    """The workload both arms run (the reference arm prints the same dict)."""
    return {"workload": f"{args.instance} ACS, {m} ants, cl=32, k={args.k}, {args.variant} dense"
            if args.variant not in ("spm", "spm-seq", "spm-sync") else f"{args.instance} ACS-SPM, {m} ants, s=8",
            "instance": args.instance, "n": n, "ants_per_gpu": m, "variant": args.variant,
            "cl": 32, "k": args.k, "beta": 3.0, "alpha": 0.2, "rho": 0.01,
            "q0": round(default_q0(n), 6), "rng": rng_for(args.variant, args.rng),
            "l2": "flushed (256 MiB write) before every timed step",
            "parallelism": f"island x{world}" if world > 1 else "single colony",
            "exchange_every": args.exchange_every if world > 1 else None, "exchange": exchange}


def host_cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
        if not shared:  # NCCL's own init lines carry the communicator size (nRanks), on stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
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
            print(f"[acs] island NCCL communicator: rank {rank} of nranks {world} on cuda:{local}",
                  file=sys.stderr, flush=True)

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

    # Roofline of the dominant kernel (construction).  Its working set is
    # L2-resident: the bound is the L2, with the L2 read
    # bandwidth measured in this run as the peak; the HBM figure is kept
    # alongside.  Algorithmic bytes = the per-tour term x m
    # + F, the fallback term, reported separately: F counts n - t nodes x
    # 12 B for every fallback step as if it scanned all unvisited nodes,
    # which the pruned pass mostly does not.
    fb_elems = c1.get("fallback_elems", 0) - c0.get("fallback_elems", 0)
    B_tour = algorithmic_bytes_per_tour(inst.n, col.info.list_len, args.k, args.variant)
    F_launch = fb_elems * 12 / max(args.steps, 1)
    alg_bytes_launch = B_tour * m + F_launch
    construct_s = construct_ms / 1e3 / args.steps
    peaks, src = measured_peaks()
    achieved = alg_bytes_launch / construct_s / 1e9
    l2_gbs = P._native.l2_read_bandwidth(local, 48 << 20)
    rec = ncu_record(args.variant)
    sectors = rec.get("lts__t_sectors_srcunit_tex_op_read.sum")
    l2_read = sectors * 32 if sectors else None
    roofline = {"bound": "l2", "achieved": round(achieved, 1), "peak": round(l2_gbs, 1), "unit": "GB/s",
                "frac": round(achieved / l2_gbs, 4), "traffic": ncu_traffic(args.variant),
                "traffic_note": "dram bytes per launch (ncu --set full, committed capture); the working set "
                                "is L2-resident, so DRAM traffic is the cold fill only",
                "peak_source": "acs_gpu_l2_read_bandwidth: ld.global.cg stream over a 48 MiB L2-resident "
                               "buffer, measured in this run",
                "kernel": construct_kernel(args.variant, args.k),
                "construct_ms_per_launch": round(construct_s * 1e3, 4),
                "bytes_per_tour": B_tour,
                "algorithmic_bytes_per_launch": round(alg_bytes_launch),
                "fallback_bytes_per_launch": round(F_launch),
                "l2_read_bytes_per_launch": l2_read,
                "l2_traffic_ratio": round(l2_read / (B_tour * m), 3) if l2_read else None,
                "l2_traffic_ratio_note": "ncu L2 read bytes per launch / the per-tour algorithmic bytes x m "
                                         "(without F): >1 means bytes read that the algorithm does not need",
                "hbm": {"peak": peaks["hbm_gbs"], "frac": round(achieved / peaks["hbm_gbs"], 4),
                        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src})"},
                "note": "latency-bound dependent-load chain; L2-resident working set"}

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
                             "inst_per_step": round(n_inst / (m * (inst.n - 1)), 1),
                             "source": "ncu --set full 'Executed Instructions' of this variant's construct kernel "
                                       "(profiles/ncu_construct_summary.json) / this run's launch time; peak = "
                                       "4 schedulers x SMs x median SM clock under load"}
    # Latency floor (hardware, not this kernel): acs_gpu_l2_latency measures
    # the L2 load-to-use latency (pointer chase) and one warp's MINIMAL
    # selection step over L2-resident rows (row + trail load, visited test,
    # score, exact argmax, next row = the winner's).  Every ant is a chain of
    # n - 1 such steps, so ns per step of the colony = launch time / (n - 1)
    # cannot go below floor_ns_per_step.
    load_ns, step_ns = P._native.l2_latency(local, 48 << 20)
    ach_step_ns = construct_s * 1e9 / ((inst.n - 1) * max(1, -(-m // resident_ants(P, local, m))))
    roofline["latency"] = {"floor_ns_per_step": round(step_ns, 1), "l2_load_ns": round(load_ns, 1),
                           "achieved_ns_per_step": round(ach_step_ns, 1),
                           "frac": round(step_ns / ach_step_ns, 4),
                           "source": "acs_gpu_l2_latency in this run: L2 pointer chase (ld.global.cg, 48 MiB) and "
                                     "one warp's minimal selection step over L2-resident rows; achieved = launch "
                                     "time / (n - 1) steps / waves"}
    # the isolated ant of THIS kernel (128-ant colony, < 1 ant per SM)
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
    roofline["latency"]["isolated_ant"] = {
        "ms": round(lat_ms, 4), "ns_per_step": round(lat_ms * 1e6 / (inst.n - 1), 1),
        "frac_colony": round(lat_ms / (construct_s * 1e3), 4),
        "source": "construct time of a 128-ant colony of the same kernel, median of 5: the colony's time "
                  "over one ant's chain (issue contention)"}
    col.close()
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "tours/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": round(value / PAPER_ACS_GPU_PR2392, 2) if args.instance == "pr2392" and args.variant == "atomic" else None,
        "vs_baseline_ref": "paper ACS-GPU (atomic) pr2392 4942 tours/s on GK104 (BASELINE.md, PAPER.md:920)",
        "dtype": "f64", "data": data_desc(args.instance),
        "config": bench_config(args, inst.n, m, world, exchange),
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
    region.  At N > 1 every rank runs its own colony at the same time and the
    colonies exchange their best every --exchange-every steps inside the timed
    region (acs_gpu_island_exchange over NCCL; host exchange over gloo when
    ranks share a GPU); the NCCL communicator setup (acs_gpu_island_init, the
    analogue of init_process_group) is excluded from the wall time.  The
    whole-job value uses the max wall time over ranks.  Repeated 5 times (host
    wall clocks on the box jitter by tens of ms); the median is reported."""
    import ctypes as C
    import numpy as np
    from paper_1605_02669_b200 import _native as N
    K = args.steps
    d = inst.desc()
    p = params.to_c(inst.n)
    order = np.empty(inst.n, np.uint32)
    bl = C.c_int64()
    stat = N.IterStats()
    gbl = C.c_int64()
    lib = N.lib()
    nccl = world > 1 and not shared
    exchanges = [0]

    def one(k):
        if nccl:  # the unique id travels over the process group, before the clock starts
            uid = [P.Colony.nccl_unique_id() if dist.get_rank() == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            ubuf = C.create_string_buffer(uid[0], 128)
        h = C.c_void_p()
        t0 = time.perf_counter()
        N.check(lib.acs_gpu_create(C.byref(d), C.byref(p), device, C.byref(h)), "acs_gpu_create")
        excluded = 0.0
        try:
            if nccl:
                ti = time.perf_counter()
                N.check(lib.acs_gpu_island_init(h, ubuf, world, dist.get_rank()), "acs_gpu_island_init")
                excluded = time.perf_counter() - ti
            n_ex = 0
            for i in range(k):
                N.check(lib.acs_gpu_iterate(h, 1, C.byref(stat)), "acs_gpu_iterate")
                if world > 1 and (i + 1) % args.exchange_every == 0:
                    n_ex += 1
                    if nccl:
                        N.check(lib.acs_gpu_island_exchange(h, C.byref(gbl)), "acs_gpu_island_exchange")
                    else:
                        P.island.exchange_host(_CtxView(lib, h, inst.n), dist)
            N.check(lib.acs_gpu_get_best(h, order.ctypes.data_as(C.c_void_p), C.byref(bl)), "acs_gpu_get_best")
            exchanges[0] = n_ex
        finally:
            lib.acs_gpu_destroy(h)
        return time.perf_counter() - t0 - excluded

    one(1)  # untimed: lazy CUDA module loading of the setup kernels
    walls = []
    for _ in range(5):
        if dist:
            dist.barrier()
        dt = one(K)
        if dist:
            import torch
            t = torch.tensor([dt], dtype=torch.float64, device="cpu" if shared else f"cuda:{device}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        walls.append(dt)
    dt = statistics.median(walls)
    m = p.ants
    ex_bytes = exchanges[0] * (8 if nccl else 8 + 4 * inst.n) / K  # L_gb read back per exchange (host path: + tour)
    return {"value": round(world * m * K / dt, 1), "unit": "tours/s",
            "h2d_bytes_per_step": round(2 * 8 * inst.n / K, 1),
            "d2h_bytes_per_step": round(C.sizeof(N.IterStats) + (4 * inst.n + 8) / K + ex_bytes, 1),
            "api": f"acs_gpu_create + K x acs_gpu_iterate(ctx, 1, &stats) (per-step result D2H)"
                   + (f" + island exchange every {args.exchange_every} steps ({exchanges[0]} per run, "
                      + ("acs_gpu_island_exchange over NCCL" if nccl else "host exchange over gloo") + ")"
                      if world > 1 else "")
                   + f" + acs_gpu_get_best + acs_gpu_destroy, host buffers, on each of {world} rank(s); "
                   f"max wall over ranks, median of 5 runs",
            "nccl_comm_nranks": world if nccl else None,
            "wall_s": round(dt, 4), "wall_s_runs": [round(w, 4) for w in walls]}


class _CtxView:
    """best()/set_best() of a raw C-ABI context, for island.exchange_host."""

    def __init__(self, lib, h, n):
        self.lib, self.h, self.n = lib, h, n

    def best(self):
        import ctypes as C
        import numpy as np
        from paper_1605_02669_b200 import _native as N
        order = np.empty(self.n, np.uint32)
        ln = C.c_int64()
        N.check(self.lib.acs_gpu_get_best(self.h, order.ctypes.data_as(C.c_void_p), C.byref(ln)), "get_best")
        return order, ln.value

    def set_best(self, order, length):
        import ctypes as C
        import numpy as np
        from paper_1605_02669_b200 import _native as N
        order = np.ascontiguousarray(order, np.uint32)
        N.check(self.lib.acs_gpu_set_best(self.h, order.ctypes.data_as(C.c_void_p), int(length)), "set_best")


if __name__ == "__main__":
    sys.exit(main())
