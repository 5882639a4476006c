#!/usr/bin/env python
"""bench.py -- candidate (task set, partition, allocation) evals/s on B200.

Default workload: C3 (BASELINE.json configs[2], the largest enumeration
config): M = 20 SMs, n = 6 tasks, 10 utilisation bins x 1,000 task sets per
GPU per step (weak scaling: every rank adds its own 10,000 sets), all
694,755 canonical candidates of every set evaluated exactly.  One step = the
whole hot path: gp_generate -> gp_sched_ratio(EXHAUSTIVE) (enumerate + WCET +
EDF fused) -> gp_allocate x {1G, SMS_ACT, SMS_INA, BF_ACT, BF_INA} ->
gp_sched_ratio(FROM_VERDICTS) -> NCCL all-reduce of the integer counts.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--reps R]
  python bench.py --impl reference ...   # the CPU oracle arm (rank 0 only)

Timing: CUDA events on the launching stream around each step (an L2 flush --
a 256 MiB memset -- runs between steps outside the events), barrier +
synchronize on both sides of the K timed steps, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gp_workloads as W  # noqa: E402

METRIC = "candidate (taskset,partition,alloc) evals/sec at 1/2/4/8 B200; % INT/HBM roofline"
UNIT = "candidate evals/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
B200_SMS, SMSP_PER_SM, LANES = 148, 4, 32
FALLBACK_SM_MHZ = 1965.0  # clocks.max.sm of B200 (B200_PROFILING.md)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c2", "c3"])
    ap.add_argument("--reps", type=int, default=1000, help="sets per (bin) group per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-sets", type=int, default=0, help="0 = auto (~15 s)")
    return ap.parse_args()


def workload_config(key, reps, world):
    wl = W.WORKLOADS[key]
    n_cand = _count(wl["M"], wl["n"])
    return wl, n_cand


def _count(M, n):
    from math import comb

    def s2(n_, k):
        from math import factorial
        return sum((-1) ** j * comb(k, j) * (k - j) ** n_ for j in range(k + 1)) // factorial(k)
    return sum(s2(n, k) * comb(M, k) for k in range(1, min(M, n) + 1))


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    wl, n_cand = workload_config(args.config, args.reps, 1)
    cores = os.cpu_count() or 1
    gen = wl["gen"](R=args.reps)
    sample_reps = 2  # 2 sets per bin = 20 sets per step: ~1-3 s of CPU work per step
    sets = oracle.generate(gen, W.SEED, 0, sample_reps)
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        s = oracle.generate(gen, W.SEED, (it % 50) * sample_reps, sample_reps)
        oracle.exhaustive(s, threads=cores)
        for v in W.VARIANT_NAMES:
            oracle.allocate(s, v, threads=cores)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    per_step = sets.n_sets * n_cand
    value = per_step * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "config": {"workload": wl["name"], "M": wl["M"], "n": wl["n"],
                                        "sets_per_step": sets.n_sets, "candidates_per_set": n_cand},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{sets.n_sets} sets ({sample_reps} per bin) of {wl['name']} "
                                   "per step: generate + exhaustive + 5 heuristics, C oracle, "
                                   f"{cores} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- cpu baseline
def cpu_baseline(key, reps, n_cand, target_s=15.0):
    import oracle
    wl = W.WORKLOADS[key]
    gen = wl["gen"](R=reps)
    cores = os.cpu_count() or 1
    probe = oracle.generate(gen, W.SEED, 0, 1)  # one set per bin, all bins
    t0 = time.perf_counter()
    oracle.exhaustive(probe, threads=cores)
    dt = time.perf_counter() - t0
    per_rep = max(dt, 1e-3)
    k = int(max(1, min(reps, target_s / per_rep)))
    s = oracle.generate(gen, W.SEED, 0, k)
    t0 = time.perf_counter()
    oracle.exhaustive(s, threads=cores)
    dt = time.perf_counter() - t0
    return {"value": s.n_sets * n_cand / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {k} sets of each of the 10 bins ({s.n_sets} sets, "
                      f"{s.n_sets * n_cand} candidates) of {wl['name']}, exhaustive verdicts, "
                      f"{dt:.1f} s on {cores} threads"}


# --------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_2105_10312_b200 import gpart as G
    from paper_2105_10312_b200.pipeline import Pipeline, allreduce_counts

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl, n_cand = workload_config(args.config, args.reps, world)
    pipe = Pipeline(args.config, reps=args.reps, rank=rank, world=world)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    exh_ev = []

    def step(i, timed):
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        G.gp_generate(pipe.gens[0], pipe.seed, pipe.rep_begin, pipe.reps, pipe.ts, stream)
        if timed:
            e0.record(stream)
        G.gp_sched_ratio(pipe.ts, G.GP_EXHAUSTIVE, pipe.counts, slot0=0, n_slots=pipe.n_slots,
                         setting=0, per_set=pipe.per_set, work_counter=pipe.work,
                         stats=pipe.stats, stream=stream)
        if timed:
            e1.record(stream)
            exh_ev.append((e0, e1))
        for vi, v in enumerate(pipe.variants):
            G.gp_allocate(pipe.ts, v, pipe.alloc[vi], stream)
        G.gp_sched_ratio(pipe.ts, G.GP_FROM_VERDICTS, pipe.counts, verdicts=pipe.verdicts,
                         slot0=1, n_slots=pipe.n_slots, setting=0, stream=stream)
        allreduce_counts(pipe.counts)

    for i in range(args.warmup):
        step(i, False)
    torch.cuda.synchronize()
    pipe.reset_counts()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    evs = []
    for i in range(args.steps):
        flush.zero_()  # L2 flush between steps, outside the events
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        step(i, True)
        s1.record(stream)
        evs.append((s0, s1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    exh_ms = [a.elapsed_time(b) for a, b in exh_ev]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    cand_step_rank = pipe.candidates_per_step()
    value = cand_step_rank * world * args.steps / (total_ms / 1e3)
    stats = pipe.stats.cpu().numpy() / args.steps  # per launch (deterministic)
    tests = pipe.heuristic_tests()

    # ---- roofline of the dominant kernel (exhaustive evaluator): essential
    # integer ops per launch: 3 per task of every tested
    # block (W lookup, C<=D compare, U multiply-add), 4 per deadline examined
    # (min-select, add, compare, advance), 4 per candidate (successor, verdict).
    ops = 3 * stats[3] + 4 * stats[2] + 4 * stats[0]
    exh_avg_s = statistics.mean(exh_ms) / 1e3
    peak_mhz = FALLBACK_SM_MHZ
    peak_src = "B200 clocks.max.sm 1965 MHz (B200_PROFILING.md)"
    try:
        with open(PEAKS) as fh:
            pk = json.load(fh)
        peak_mhz = float(pk.get("sm_max_mhz", peak_mhz))
        peak_src = f"MEASURED_PEAKS.json sm_max_mhz {peak_mhz:.0f}"
    except (OSError, ValueError):
        pass
    peak_ops = B200_SMS * SMSP_PER_SM * LANES * peak_mhz * 1e6  # 1 warp-inst/clk/SMSP
    roof = {"bound": "alu", "achieved": ops / exh_avg_s / 1e12, "peak": peak_ops / 1e12,
            "unit": "Tops/s (int32 lane-ops)", "frac": (ops / exh_avg_s) / peak_ops,
            "traffic": None, "kernel": "k_exhaustive<6>",
            "ops_per_launch": float(ops), "ops_per_candidate": float(ops / max(stats[0], 1)),
            "launch_ms": exh_avg_s * 1e3, "kernel_share_of_step": statistics.mean(exh_ms) /
            statistics.mean(step_ms), "peak_source": peak_src + " x 148 SM x 4 SMSP x 32 lanes",
            "events_per_candidate": float(stats[2] / max(stats[0], 1))}

    # ---- e2e: the same metric through the C ABI from HOST buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(G, pipe, stream, args, world, n_cand)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": wl["name"], "M": wl["M"], "n": wl["n"],
                   "sets_per_gpu": pipe.ts.n_sets, "global_sets": pipe.ts.n_sets * world,
                   "candidates_per_set": n_cand, "candidates_per_step": cand_step_rank * world,
                   "heuristic_edf_tests_per_step": tests * world,
                   "variants": list(pipe.variants), "parallelism": f"dp{world}",
                   "l2": "flushed between steps (256 MiB memset outside the events)",
                   "seed": W.SEED},
        "roofline": roof,
        "gpu_launches": launches_per_step(pipe) * args.steps,
        "clocks": clk,
    }
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, args.reps, n_cand)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def launches_per_step(pipe):
    # gp_generate 1 + EXHAUSTIVE (init, main, finalize) 3 + gp_allocate x V + ratio 1
    return 1 + 3 + len(pipe.variants) + 1


def run_e2e(G, pipe, stream, args, world, n_cand):
    """Host task sets (pinned) -> H2D -> exhaustive + allocate + ratio -> D2H."""
    import torch
    host = {f: getattr(pipe.ts, f).cpu().pin_memory() for f in
            ("T", "D", "B", "cn", "cc", "fn", "fc", "type", "valid", "group")}
    dev = G.TaskSets(pipe.ts.n_sets, pipe.ts.n_tasks, pipe.ts.M, pipe.ts.n_groups)
    out_per = torch.empty((pipe.ts.n_sets, 4), dtype=torch.int64).pin_memory()
    out_cnt = torch.empty(tuple(pipe.counts.shape), dtype=torch.int64).pin_memory()
    out_ver = torch.empty(tuple(pipe.verdicts.shape), dtype=torch.uint8).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in host.values())
    d2h = sum(t.numel() * t.element_size() for t in (out_per, out_cnt, out_ver))

    def one():
        for f, t in host.items():
            getattr(dev, f).copy_(t, non_blocking=True)
        pipe.counts.zero_()
        G.gp_sched_ratio(dev, G.GP_EXHAUSTIVE, pipe.counts, slot0=0, n_slots=pipe.n_slots,
                         per_set=pipe.per_set, work_counter=pipe.work, stream=stream)
        for vi, v in enumerate(pipe.variants):
            G.gp_allocate(dev, v, pipe.alloc[vi], stream)
        G.gp_sched_ratio(dev, G.GP_FROM_VERDICTS, pipe.counts, verdicts=pipe.verdicts, slot0=1,
                         n_slots=pipe.n_slots, stream=stream)
        out_per.copy_(pipe.per_set, non_blocking=True)
        out_cnt.copy_(pipe.counts, non_blocking=True)
        out_ver.copy_(pipe.verdicts, non_blocking=True)

    for _ in range(2):
        one()
    torch.cuda.synchronize()
    evs = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        one()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": pipe.ts.n_sets * n_cand * world * args.steps / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": ms / args.steps,
            "path": "pinned host task sets -> H2D -> gp_sched_ratio(EXHAUSTIVE) + gp_allocate x5 "
                    "+ gp_sched_ratio -> D2H per-set results, verdicts, counts"}


if __name__ == "__main__":
    sys.exit(main())
