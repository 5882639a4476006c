#!/usr/bin/env python
"""bench.py -- candidate (task set, partition, allocation) evals/s on B200.

Default workload: C3 (BASELINE.json configs[2], the largest enumeration
config, its scaling size): M = 20 SMs, n = 6 tasks, 10 utilisation bins x
10,000 task sets per GPU per step (weak scaling: every rank adds its own
100,000 sets), all
694,755 canonical candidates of every set evaluated exactly.  One step = the
whole hot path: gp_generate -> gp_sched_ratio(EXHAUSTIVE) (enumerate + WCET +
EDF fused) -> gp_allocate x {1G, SMS_ACT, SMS_INA, BF_ACT, BF_INA} ->
gp_sched_ratio(FROM_VERDICTS) -> NCCL all-reduce of the integer counts.
Heuristic-only configs (--config c4 / c5) count one candidate eval per
EDF-PDC test the heuristics run.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--reps R]
  python bench.py --impl reference ...   # the CPU oracle arm (rank 0 only)

Timing: CUDA events on the launching stream around each step (an L2 flush --
a 256 MiB memset -- runs between steps outside the events), barrier +
synchronize on both sides of the K timed steps, max over ranks.
"""
from __future__ import annotations

import argparse
import math
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import gp_workloads as W  # noqa: E402

METRIC = "candidate (taskset,partition,alloc) evals/sec at 1/2/4/8 B200; % INT/HBM roofline"
UNIT = "candidate evals/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
B200_SMS, SMSP_PER_SM, LANES = 148, 4, 32
FALLBACK_SM_MHZ = 1965.0  # clocks.max.sm of B200 (B200_PROFILING.md)
DEFAULT_REPS = {"c2": 10000, "c3": 10000, "c4": 20000, "c5": 10000}  # SURVEY §8(d) sizes


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--reps", type=int, default=0,
                    help="sets per (prm, bin) group: per GPU (--split weak) or global")
    ap.add_argument("--split", default="weak", choices=["weak", "sets", "ranks"],
                    help="multi-GPU sharding (SURVEY 8(e)): weak = R sets/group per GPU; "
                         "sets = R global sets/group split by set range (strong); ranks = all "
                         "R global sets on every GPU, candidate-rank windows + per-set merge")
    ap.add_argument("--strong", action="store_true", help="alias of --split sets")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-memo-heuristics", action="store_true",
                    help="the heuristics run their own EDF tests instead of looking up the "
                         "bit-sliced evaluator's memoised block verdicts (A/B)")
    ap.add_argument("--exh-flags", type=int, default=0,
                    help="extra gp_exhaustive_opts flags for the timed call (A/B of test hooks)")
    ap.add_argument("--variants-in-order", action="store_true",
                    help="A/B: launch the parallel variant kernels in list order, not longest first")
    ap.add_argument("--serial-variants", action="store_true",
                    help="launch the heuristic variants one after the other on one stream "
                         "(default: parallel streams for sets of <= 8 tasks)")
    ap.add_argument("--no-graph", action="store_true",
                    help="issue every launch of the timed steps from the host instead of "
                         "replaying the step's CUDA graphs")
    ap.add_argument("--no-direct", action="store_true",
                    help="skip timing the per-candidate (direct) evaluator beside the headline")
    ap.add_argument("--f3", action="store_true",
                    help="use the subset-threshold evaluator (SURVEY §8(f) f3, a different work "
                         "unit, reported separately) instead of the direct per-candidate path")
    ap.add_argument("--per-candidate", action="store_true",
                    help="time the per-candidate EXHAUSTIVE evaluator instead of the bit-sliced one")
    ap.add_argument("--f3-hash", action="store_true",
                    help="with --f3, also enumerate the schedulable candidates for the verdict "
                         "hash (parity check; counts and ratios do not need it)")
    a = ap.parse_args()
    a.reps = a.reps or DEFAULT_REPS[a.config]
    if a.strong:
        a.split = "sets"
    return a


def n_candidates(M, n):
    from math import comb, factorial

    def s2(n_, k):
        return sum((-1) ** j * comb(k, j) * (k - j) ** n_ for j in range(k + 1)) // factorial(k)
    return sum(s2(n, k) * comb(M, k) for k in range(1, min(M, n) + 1))


def ncu_entry(workload):
    """The latest committed ncu --set full capture of the dominant kernel
    (profiles/rNN/ncu_metrics.json): (entry dict, source path) or (None, None)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_metrics.json")),
                       reverse=True):
        try:
            with open(path) as fh:
                m = json.load(fh)
        except (OSError, ValueError):
            continue
        e = m.get(workload)
        if isinstance(e, dict) and e.get("dram_bytes") is not None:
            return e, os.path.relpath(path, ROOT)
    return None, None


def stirling2(n, k):
    """Stirling numbers of the second kind (number of allocations with k blocks)."""
    row = [1] + [0] * k
    for i in range(1, n + 1):
        row = [0] + [row[j - 1] + j * (row[j] if j < len(row) else 0) for j in range(1, k + 1)]
    return row[k]


def peak_lane_ops():
    """Issue ceiling in int32 lane-ops/s: 148 SM x 4 SMSP x 32 lanes x clock."""
    mhz, src = FALLBACK_SM_MHZ, "B200 clocks.max.sm 1965 MHz (B200_PROFILING.md fallback)"
    try:
        with open(PEAKS) as fh:
            pk = json.load(fh)
        mhz = float(pk.get("sm_max_mhz", mhz))
        src = f"MEASURED_PEAKS.json sm_max_mhz {mhz:.0f}"
    except (OSError, ValueError):
        pass
    return B200_SMS * SMSP_PER_SM * LANES * mhz * 1e6, src + " x 148 SM x 4 SMSP x 32 lanes"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event reasons sampled DURING the timed region: NVML
    polled every 2 ms from a thread (so even a ~30 ms region gets samples);
    nvidia-smi -lms 200 as the fallback when pynvml is missing."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.rows, self.p, self.thread = [], None, None
        try:
            import threading

            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
            self.stop_ev = threading.Event()

            def poll():
                while True:
                    sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((sm, [bool(r & b) for b in bits]))
                    if self.stop_ev.wait(0.002):
                        break

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:  # noqa: BLE001 -- fall back to nvidia-smi
            self.thread = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.thread is not None:
            self.stop_ev.set()
            self.thread.join(timeout=5)
            rows = self.rows
            if not rows:
                return None
            sm = [r[0] for r in rows]
            mx = self.mx
            reasons = sorted({self.NAMES[i] for r in rows for i in range(4) if r[1][i]})
            src = "nvml 2 ms"
        else:
            if self.p is None:
                return None
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()
            self.f.flush()
            raw = []
            with open(self.f.name) as fh:
                for line in fh:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                        raw.append(parts)
            os.unlink(self.f.name)
            if not raw:
                return None
            sm = [float(r[1]) for r in raw]
            mx = max(float(r[2]) for r in raw)
            reasons = sorted({self.NAMES[i] for r in raw for i in range(4) if r[5 + i].lower() == "active"})
            src = "nvidia-smi 200 ms"
        loaded = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(sm), "source": src}


# --------------------------------------------------------------------------- CPU oracle
def oracle_step(oracle, wl, gen_list, rep_begin, reps, cores, exhaustive):
    """One oracle step on a sample: generate + [exhaustive] + 5 heuristics.
    Returns (candidate evals, seconds)."""
    t0 = time.perf_counter()
    evals = 0
    for gi, gen in enumerate(gen_list):
        s = oracle.generate(gen, W.SEED, rep_begin, reps)
        if exhaustive and gi == 0:
            oracle.exhaustive(s, threads=cores)
            evals += s.n_sets * n_candidates(wl["M"], wl["n"])
        for v in W.VARIANT_NAMES:
            r = oracle.allocate(s, v, threads=cores)
            if not exhaustive:
                evals += int(r["n_tests"].clip(min=0).sum())
    return evals, time.perf_counter() - t0


def gens_for(key, R):
    wl = W.WORKLOADS[key]
    if key == "c5":
        return [wl["gen"](R=R, kc=kc, km=km) for kc, km in W.C5_SETTINGS]
    return [wl["gen"](R=R)]


def run_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    import oracle
    wl = W.WORKLOADS[args.config]
    cores = os.cpu_count() or 1
    gens = gens_for(args.config, args.reps)
    n_groups0 = gens[0]["n_prm"] * gens[0]["n_bins"]
    # sets per (prm, bin) group per step: >= 4 sets per host thread so that every core
    # stays busy through the load imbalance between utilisation bins (C3 on 16 threads:
    # 7 per group = 70 sets, about 1 s of oracle work per step)
    sample = max(1, -(-4 * cores // n_groups0))
    if args.config == "c2":
        sample = max(sample, 20)
    if args.config == "c5":
        gens = gens[:4]  # 4 of the 16 coefficient settings per step
    evs, secs = [], []
    for it in range(args.warmup + args.steps):
        e, t = oracle_step(oracle, wl, gens, (it * sample) % max(1, args.reps - sample), sample,
                           cores, wl["exhaustive"])
        if it >= args.warmup:
            evs.append(e)
            secs.append(t)
    value = sum(evs) / sum(secs)
    n_groups = gens[0]["n_prm"] * gens[0]["n_bins"]
    desc = (f"{sample} sets per (prm,bin) group ({sample * n_groups} sets) of {wl['name']} per "
            f"step x {len(gens)} setting(s): generate + {'exhaustive + ' if wl['exhaustive'] else ''}"
            f"5 heuristics, C oracle on {cores} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(secs) / len(secs), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": wl["name"], "M": wl["M"], "n": wl["n"],
                   "sets_per_step": sample * n_groups},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(args, target_s=15.0):
    import oracle
    wl = W.WORKLOADS[args.config]
    cores = os.cpu_count() or 1
    gens = gens_for(args.config, args.reps)[:1]
    e, t = oracle_step(oracle, wl, gens, 0, 1, cores, wl["exhaustive"])  # probe: 1 set/group
    k = int(max(1, min(args.reps, target_s / max(t, 1e-3))))
    e, t = oracle_step(oracle, wl, gens, 0, k, cores, wl["exhaustive"])
    n_groups = gens[0]["n_prm"] * gens[0]["n_bins"]
    what = "exhaustive candidates" if wl["exhaustive"] else "heuristic EDF tests"
    return {"value": e / t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {k} sets of each of the {n_groups} groups of {wl['name']} "
                      f"({k * n_groups} sets, {e} {what}): generate + "
                      f"{'exhaustive + ' if wl['exhaustive'] else ''}5 heuristics, {t:.1f} s "
                      f"on {cores} threads"}


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
    # one rank per GPU; GP_BENCH_BACKEND=gloo lets several ranks share a GPU (a test of
    # the N > 1 code path on a one-GPU box; timings from such a run are not scaling data)
    backend = os.environ.get("GP_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    wl = W.WORKLOADS[args.config]
    pipe = Pipeline(args.config, reps=args.reps, rank=rank, world=world, split=args.split,
                    memo_heuristics=not args.no_memo_heuristics,
                    parallel_variants=False if args.serial_variants else None)
    pipe.longest_first = not args.variants_in_order
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    alloc_stats = torch.zeros(8, dtype=torch.int64, device="cuda")  # GP_AL_STATS_EXT layout
    exh_mode = G.GP_THRESHOLD if args.f3 else G.GP_EXHAUSTIVE
    exh_flags = G.GP_EX_NO_HASH if (args.f3 and not args.f3_hash) else 0
    if args.per_candidate:
        exh_flags |= G.GP_EX_PER_CANDIDATE
    exh_flags |= args.exh_flags
    if args.f3 and not pipe.exhaustive:
        raise SystemExit("--f3 needs an exhaustive config (c2, c3)")
    if args.f3 and args.split == "ranks":
        raise SystemExit("--f3 evaluates whole rank spaces: use --split weak|sets")
    dom_ev = []  # events around the dominant kernel's launches

    def step(timed, stats=False):
        """One full step (Pipeline.run).  The dominant kernel is the exhaustive evaluator
        when present, else the heuristics (gp_allocate); its launches are bracketed by CUDA
        events on the launching stream."""
        ev = []

        def hook(phase):
            if timed:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                ev.append(e)
        pipe.run(stream, mode=exh_mode, flags=exh_flags, stats=stats,
                 alloc_stats=alloc_stats if stats else None, on_dominant=hook)
        dom_ev.extend(zip(ev[0::2], ev[1::2]))

    for _ in range(args.warmup):
        step(False)
    # one instrumented, untimed step: per-step work figures (deterministic)
    pipe.reset_counts()
    alloc_stats.zero_()
    step(False, stats=True)
    torch.cuda.synchronize()
    exh_stats = pipe.stats.cpu().numpy().tolist() if pipe.exhaustive else [0] * 12
    al_stats = alloc_stats.cpu().numpy().tolist()
    # §8(d)'s per-candidate work (the direct evaluation's W lookups, utilisation
    # passes and demand-walk events), counted by the per-candidate evaluator on
    # the same sets (deterministic; untimed)
    direct_stats = exh_stats
    if pipe.exhaustive and not args.f3 and not args.per_candidate:
        pst = torch.zeros(4, dtype=torch.int64, device="cuda")
        G.gp_sched_ratio(pipe.ts, G.GP_EXHAUSTIVE, None, per_set=pipe.per_set,
                         work_counter=pipe.work, stats=pst, stream=stream,
                         flags=G.GP_EX_PER_CANDIDATE, rank_lo=pipe.rank_lo,
                         rank_hi=pipe.rank_hi)
        torch.cuda.synchronize()
        direct_stats = pst.cpu().numpy().tolist()
    # the timed step as CUDA graphs (the same launches, replayed with a few graph launches
    # per step, so host-side launch latency cannot starve the GPU); the dominant segments are
    # bracketed by events between graph launches
    graphs = None
    if not args.no_graph and args.split != "ranks":
        graphs = pipe.capture(mode=exh_mode, flags=exh_flags)
        for _ in range(2):  # warm replays
            for g in graphs:
                g.replay()
        torch.cuda.synchronize()

    def graph_step():
        for i, g in enumerate(graphs):
            if i % 2 == 1:  # a dominant segment
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g.replay()
                e1.record(stream)
                dom_ev.append((e0, e1))
            else:
                g.replay()
        allreduce_counts(pipe.counts)

    pipe.reset_counts()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    evs = []
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between steps, outside the events
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        if graphs is not None:
            graph_step()
        else:
            step(True)
        s1.record(stream)
        evs.append((s0, s1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    dom_ms = [a.elapsed_time(b) for a, b in dom_ev]
    t = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    if pipe.exhaustive:
        evals_rank = pipe.candidates_per_step()
        unit_def = "one canonical candidate's exact verdict (C.1.6-C.1.8)"
        if args.f3:
            unit_def = ("one canonical candidate's exact verdict, resolved by the subset-threshold "
                        "evaluator (f3: per-subset thresholds + closed-form counts; NOT one "
                        "EDF test per candidate -- reported separately from the direct path)")
    else:
        evals_rank = int(al_stats[0])
        unit_def = "one EDF-PDC test of a (task subset, size) pair run by the heuristics"
    # whole-job work: the sum over ranks (uneven strong splits differ per rank)
    ev_t = torch.tensor([evals_rank], dtype=torch.int64, device="cuda")
    if world > 1:
        dist.all_reduce(ev_t, op=dist.ReduceOp.SUM)
    evals_total = int(ev_t.item())
    value = evals_total * args.steps / (total_ms / 1e3)

    # ---- roofline of the dominant kernel: essential int32 lane-ops per launch
    # (DESIGN.md "Roofline"): 3 per task of every tested block (W lookup,
    # C<=D compare, U multiply-add) + 4 per deadline examined (min-select, add,
    # compare, advance) + 4 per candidate (successor, verdict) [exhaustive].
    peak, peak_src = peak_lane_ops()
    if pipe.exhaustive and args.f3:
        st = exh_stats  # {sets, threshold tests, deadlines, schedulable enumerated}
        ops = 3 * (pipe.n / 2) * st[1] + 4 * st[2] + 4 * st[3]
        launches = 1
        kname = "k_threshold"
        per_unit = ops / max(st[0], 1)
        extra = {"sets_per_launch": st[0], "threshold_tests_per_launch": st[1],
                 "deadlines_per_launch": st[2], "schedulable_enumerated_per_launch": st[3],
                 "ops_per_unit_is": "per set"}
    elif pipe.exhaustive:
        # roofline.achieved / frac = the timed evaluator's OWN essential work per step ÷ its
        # time ÷ peak (so ops / time <= peak holds by construction).  For the per-candidate
        # evaluator that is SURVEY 8(d)'s direct work (3/task tested + 4/deadline examined +
        # 4/candidate); for the bit-sliced evaluator it is the memo pass's EDF tests (3/task +
        # 4/deadline) + 2 ops per (set, run) walked (verdict word AND, zero test) + 6 per live
        # run (count, pi* min, first min, two hash-table reads, difference-add), all counted by
        # the kernels.  The direct work divided by the bit-sliced time is reported separately
        # as effective_vs_direct (a speed-up over the direct method's issue roofline, > 1
        # possible, NOT a roofline fraction).
        st = direct_stats
        direct_ops = 3 * st[3] + 4 * st[2] + 4 * st[0]
        launches = 1
        if args.per_candidate:
            kname = f"k_exhaustive_shaped<{pipe.n}> (per-candidate evaluator)"
            ops, runs = direct_ops, None
            ops_basis = ("SURVEY 8(d)'s direct per-candidate work (3/task tested + 4/deadline "
                         "examined + 4/candidate), counted by the evaluator itself")
        else:
            kname = "k_exh_memo + k_exh_bp (bit-sliced evaluator)"
            runs = pipe.ts.n_sets * sum(stirling2(pipe.n, k) * math.comb(pipe.M - 1, k - 1)
                                        for k in range(1, min(pipe.n, pipe.M) + 1))
            ops = (3 * exh_stats[3] + 4 * exh_stats[2] + 2 * exh_stats[4] + 6 * exh_stats[5]
                   + 12 * (exh_stats[6] - exh_stats[9]) + 12 * exh_stats[8]
                   + 5 * exh_stats[10] + 7 * exh_stats[11])
            ops_basis = ("the bit-sliced evaluator's own essential work, counted by its kernels: "
                         "memo-pass EDF tests (3/task + 4/deadline) + 2 per (set, run) walked + "
                         "6 per live run walked + 12 per (set, sweep) resolved in closed form "
                         "(count, pi*, first rank: 10 int ops; hash: 2 table reads) + 12 per "
                         "(set, block) resolved by one corner-table read (its sweeps not counted) + "
                         "per (set, allocation) resolved as one full corner 5 (count, pi*, first "
                         "rank, hash read and add) + 7 per block (first size, range check, prefix "
                         "sum, rank term)")
        per_unit = ops / max(pipe.candidates_per_step(), 1)
        extra = {"ops_basis": ops_basis, "candidates_per_launch": pipe.candidates_per_step(),
                 "memo_edf_tests": exh_stats[1], "memo_deadlines": exh_stats[2],
                 "runs_total": runs, "runs_walked": exh_stats[4], "live_runs": exh_stats[5],
                 "closed_sweeps": exh_stats[6], "closed_live_runs": exh_stats[7],
                 "corner_blocks": exh_stats[8], "corner_block_sweeps": exh_stats[9],
                 "full_corner_allocations": exh_stats[10], "full_corner_blocks": exh_stats[11],
                 "direct_ops_per_step": float(direct_ops),
                 "direct_events_per_candidate": st[2] / max(st[0], 1)}
    else:
        # the heuristics' own essential work, counted by the kernels: per EDF test actually
        # run 3 ops per task (W lookup, C <= D, U multiply-add) + 4 per deadline examined,
        # and per Algorithm 3 selection 2 mask ops per partition of par_list (eligibility
        # test, rank compare) -- SURVEY 8(d)'s "O(k) mask ops per selection"
        st = al_stats
        ops = 3 * st[1] + 4 * st[2] + 2 * st[6]
        launches = len(pipe.variants) * len(pipe.gens)
        kname = "k_allocate (5 variants)"
        per_unit = ops / max(st[4], 1)
        extra = {"ops_basis": "executed EDF tests (3/task + 4/deadline) + 2 per partition scanned "
                              "by each Algorithm 3 selection, counted by the kernels",
                 "edf_tests_per_step": st[0], "edf_tests_run_per_step": st[4],
                 "tasks_tested_per_step": st[1], "deadlines_per_step": st[2],
                 "sets_per_step": st[3], "selections_per_step": st[5],
                 "partitions_scanned_per_step": st[6], "partner_searches_per_step": st[7],
                 "ops_per_unit_is": "per EDF test run"}
    dom_s = sum(dom_ms) / args.steps / 1e3  # per step (sum of the dominant launches)
    if pipe.exhaustive and not args.f3 and not args.per_candidate:
        extra["effective_vs_direct"] = extra["direct_ops_per_step"] / dom_s / peak
    if pipe.exhaustive and not args.f3:
        prof, prof_src = ncu_entry(wl["name"] + ("_per_candidate" if args.per_candidate else ""))
    elif not pipe.exhaustive:
        prof, prof_src = ncu_entry(wl["name"] + "_allocate")
    else:
        prof, prof_src = None, None
    traffic = prof["dram_bytes"] if prof else None
    roof = {"bound": "alu", "achieved": ops / dom_s / 1e12, "peak": peak / 1e12,
            "unit": "T int32 lane-ops/s", "frac": (ops / dom_s) / peak, "traffic": traffic,
            "traffic_source": prof_src,
            "ncu_issue": ({k: prof.get(k) for k in ("inst_issued_pct", "alu_pipe_pct",
                                                    "fma_pipe_pct", "warp_inst_per_candidate",
                                                    "active_threads_per_inst", "duration_ms")}
                          | {"source": prof_src})
            if prof else None,
            "kernel": kname, "launches_per_step": launches, "ops_per_step": float(ops),
            "ops_per_unit": per_unit, "dominant_ms_per_step": dom_s * 1e3,
            "kernel_share_of_step": (sum(dom_ms) / args.steps) / (total_ms / args.steps),
            "peak_source": peak_src, **extra}

    if pipe.exhaustive and not args.f3 and not args.per_candidate and not args.no_direct:
        roof["direct"] = time_direct(G, pipe, stream, flush, args, peak, direct_stats, world)

    tables = None
    if (pipe.exhaustive and not args.f3 and not args.per_candidate and pipe.n <= 8
            and pipe.M <= 32 and pipe.workspace is not None):
        tables = time_tables(G, pipe, stream, exh_mode, exh_flags)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(G, pipe, stream, args, world, exh_mode, exh_flags)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.split == "weak" else "strong", "vs_baseline": None,
        "dtype": "int32", "data": "synthetic",
        "config": {"workload": wl["name"] + ("+f3_threshold" if args.f3 else "")
                   + ("_hash" if args.f3 and args.f3_hash else ""),
                   "M": wl["M"], "n": wl["n"],
                   "sets_per_gpu": pipe.ts.n_sets, "global_sets": pipe.ts.n_sets * world,
                   "coefficient_settings": len(pipe.gens),
                   "candidates_per_set": pipe.n_cand if pipe.exhaustive else None,
                   "evals_per_step": evals_total, "eval_unit": unit_def,
                   "split": args.split,
                   "heuristic_edf_tests_per_step": int(al_stats[0]) * world,
                   "variants": list(pipe.variants),
                   "parallelism": f"dp{world}" + ("" if args.split != "ranks"
                                                  else " (candidate-rank windows)"),
                   "l2": "flushed between steps (256 MiB memset outside the events)",
                   "launch": ("CUDA graphs: %d segments per step, dominant segments bracketed "
                              "by events" % len(graphs)) if graphs is not None else "eager",
                   "seed": W.SEED},
        "roofline": roof,
        "gpu_launches": launches_per_step(pipe, args) * args.steps,
        "clocks": clk,
    }
    if tables:
        line["tables"] = tables
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def time_direct(G, pipe, stream, flush, args, peak, direct_stats, world):
    """SURVEY 8(d)'s direct path, driver-measured in the same run: the per-candidate
    evaluator (every candidate's blocks tested one by one) timed on the same sets, with
    CUDA events on the launching stream around each launch and an L2 flush between
    launches (outside the events).  frac = its own counted work (3/task + 4/deadline +
    4/candidate) ÷ its time ÷ peak."""
    import torch
    k = max(1, min(args.steps, 3))
    ms = []
    for _ in range(k):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        G.gp_sched_ratio(pipe.ts, G.GP_EXHAUSTIVE, None, per_set=pipe.per_set,
                         work_counter=pipe.work, stream=stream, flags=G.GP_EX_PER_CANDIDATE,
                         rank_lo=pipe.rank_lo, rank_hi=pipe.rank_hi)
        e1.record(stream)
        ms.append((e0, e1))
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) for a, b in ms]
    tt = torch.tensor([sum(t) / k], dtype=torch.float64, device="cuda")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    avg_s = float(tt.item()) / 1e3
    st = direct_stats
    ops = 3 * st[3] + 4 * st[2] + 4 * st[0]
    return {"kernel": f"k_exhaustive_shaped<{pipe.n}> (per-candidate evaluator)",
            "value": pipe.candidates_per_step() * world / avg_s, "unit": UNIT,
            "ms_per_launch": avg_s * 1e3, "launches_timed": k,
            "ops_per_launch": float(ops), "achieved": ops / avg_s / 1e12,
            "frac": ops / avg_s / peak,
            "note": "the same candidates evaluated one by one (SURVEY 8(d)'s direct work); the "
                    "headline value uses the bit-sliced evaluator, which needs less work"}


def launches_per_step(pipe, args=None):
    """Our kernels per step: per setting gp_generate 1 + gp_allocate x V + ratio 1;
    + EXHAUSTIVE: per-candidate (init, main, finalize) or bit-sliced (init, memo, main,
    finalize); THRESHOLD (threshold, violations).  The bit-sliced evaluator's
    input-independent tables (RGS labels, hash prefix, run-prefix and corner
    tables) are built by the first call on the workspace, before the timed steps
    (gp_exhaustive_opts.tables_key; their build time is reported as `tables`)."""
    n = len(pipe.gens) * (2 + len(pipe.variants))
    if not pipe.exhaustive:
        return n
    if args is not None and args.f3:
        return n + 2  # k_threshold, k_thr_violations
    if (args is not None and args.per_candidate) or pipe.n > 8 or pipe.M > 32:
        return n + 3
    return n + 4


def time_tables(G, pipe, stream, exh_mode, exh_flags):
    """The bit-sliced evaluator's table build (functions of n, M only; built once per
    workspace): one exhaustive call that rebuilds them minus one that reuses them, CUDA
    events on the launching stream (median of 3 pairs)."""
    import torch

    def call_ms(rebuild):
        if rebuild:
            pipe.tables_key.value = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        G.gp_sched_ratio(pipe.ts, exh_mode, None, per_set=pipe.per_set, work_counter=pipe.work,
                         stream=stream, flags=exh_flags, workspace=pipe.workspace,
                         tables_key=pipe.tables_key, rank_lo=pipe.rank_lo, rank_hi=pipe.rank_hi)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    call_ms(False)
    d = sorted(call_ms(True) - call_ms(False) for _ in range(3))
    return {"build_ms": d[1], "built": "once per workspace, before the timed steps "
            "(gp_exhaustive_opts.tables_key): RGS labels, verdict-hash prefix P, run-prefix R, "
            "corner tables CT and FCT -- functions of (n, M) only, like an FFT plan's twiddles",
            "workspace_bytes": int(pipe.workspace.numel())}


def run_e2e(G, pipe, stream, args, world, exh_mode, exh_flags):
    """Host task sets (pinned) -> H2D -> evaluation -> D2H, through the C ABI.
    The host inputs are the first setting's task sets of this rank.  Every step copies
    its inputs H2D and its results D2H inside the timed region.  Two slots, each with its
    own device inputs, device outputs and pinned host outputs: the H2D of step k+1 (copy
    stream) and the D2H of step k-1 (a second copy stream) overlap the evaluation of step
    k; a slot is reused only after its D2H finished.  The evaluation is Pipeline.run on the
    uploaded sets (same calls and collectives as the device-only step, minus gp_generate)."""
    import torch
    fields = ("T", "D", "B", "cn", "cc", "fn", "fc", "type", "valid", "group")
    G.gp_generate(pipe.gens[0], pipe.seed, pipe.rep_begin, pipe.reps, pipe.ts, stream)
    host = {f: getattr(pipe.ts, f).cpu().pin_memory() for f in fields}
    devs = [G.TaskSets(pipe.ts.n_sets, pipe.ts.n_tasks, pipe.ts.M, pipe.ts.n_groups)
            for _ in range(2)]
    settings = pipe.settings
    pipe.settings = settings[:1]  # the host inputs are one setting's task sets
    # per-slot device outputs (the pipeline's own tensors for slot 0, copies for slot 1)
    orig = (pipe.counts, pipe.verdicts, pipe.per_set if pipe.exhaustive else None)

    def make_outs(first):
        if first:
            return orig
        return tuple(None if t is None else torch.zeros_like(t) for t in orig)

    slot_outs = [make_outs(True), make_outs(False)]

    def use_slot(b):
        """Point the pipeline's output tensors at slot b's (graphs capture the pointers)."""
        counts, verdicts, per_set = slot_outs[b]
        pipe.counts, pipe.verdicts = counts, verdicts
        for vi, out in enumerate(pipe.alloc):
            out.ok = verdicts[vi]
        if per_set is not None:
            pipe.per_set = per_set

    def out_list(b):
        return [t for t in slot_outs[b] if t is not None]

    host_out = [[torch.empty(tuple(t.shape), dtype=t.dtype).pin_memory() for t in out_list(b)]
                for b in range(2)]
    h2d = sum(t.numel() * t.element_size() for t in host.values())
    d2h = sum(t.numel() * t.element_size() for t in host_out[0])
    stats = torch.zeros(4, dtype=torch.int64, device="cuda")
    copy_stream, d2h_stream = torch.cuda.Stream(), torch.cuda.Stream()

    def upload(dev, s):
        with torch.cuda.stream(s):
            for f, t in host.items():
                getattr(dev, f).copy_(t, non_blocking=True)

    def compute_on(b, s, with_stats=False, collectives=True):
        """The step's ABI calls on stream `s` into slot b's outputs."""
        use_slot(b)
        with torch.cuda.stream(s):
            pipe.counts.zero_()
        pipe.run(s, mode=exh_mode, flags=exh_flags,
                 alloc_stats=stats if with_stats else None, ts=devs[b], collectives=collectives)

    # the compute of a step in either slot as a CUDA graph (as in the device-only timed
    # loop); the counts all-reduce and the copies stay outside
    egraphs = None
    if not args.no_graph and pipe.split != "ranks":
        compute_on(0, stream)  # warm (lazy module loading, workspaces)
        torch.cuda.synchronize()
        egraphs = []
        for b in range(2):
            side = torch.cuda.Stream()
            side.wait_stream(stream)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                g.capture_begin()
                compute_on(b, side, collectives=False)
                g.capture_end()
            stream.wait_stream(side)
            egraphs.append(g)

    def compute(b, with_stats=False):
        if egraphs is not None and not with_stats:
            egraphs[b].replay()
            from paper_2105_10312_b200.pipeline import allreduce_counts
            allreduce_counts(slot_outs[b][0])
        else:
            compute_on(b, stream, with_stats)

    def run(k_steps, with_stats=False):
        """k_steps pipelined steps; returns (start, end) events on `stream`."""
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        freed = [None, None]    # slot's inputs consumed (its compute finished)
        fetched = [None, None]  # slot's outputs copied to the host
        start.record(stream)
        copy_stream.wait_event(start)
        upload(devs[0], copy_stream)
        copied[0].record(copy_stream)
        for k in range(k_steps):
            cur, nxt = k % 2, 1 - k % 2
            stream.wait_event(copied[cur])
            if fetched[cur] is not None:  # its outputs of step k-2 are on the host
                stream.wait_event(fetched[cur])
            if k + 1 < k_steps:  # next step's inputs, once its slot's last compute is done
                if freed[nxt] is not None:
                    copy_stream.wait_event(freed[nxt])
                upload(devs[nxt], copy_stream)
                copied[nxt].record(copy_stream)
            compute(cur, with_stats)
            freed[cur] = torch.cuda.Event()
            freed[cur].record(stream)
            d2h_stream.wait_event(freed[cur])
            with torch.cuda.stream(d2h_stream):
                for h, d in zip(host_out[cur], out_list(cur)):
                    h.copy_(d, non_blocking=True)
            fetched[cur] = torch.cuda.Event()
            fetched[cur].record(d2h_stream)
        for e in fetched:
            if e is not None:
                stream.wait_event(e)
        end.record(stream)
        return start, end

    run(1, with_stats=True)
    torch.cuda.synchronize()
    evals = pipe.candidates_per_step() if pipe.exhaustive else int(stats[0].item())
    ev_t = torch.tensor([evals], dtype=torch.int64, device="cuda")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(ev_t, op=dist.ReduceOp.SUM)
    evals = int(ev_t.item())
    run(2)
    torch.cuda.synchronize()
    a, b = run(args.steps)
    torch.cuda.synchronize()
    use_slot(0)
    pipe.settings = settings
    ms = a.elapsed_time(b)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": evals * args.steps / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ms / args.steps,
            "path": "pinned host task sets -> H2D (copy stream) -> gp_sched_ratio(EXHAUSTIVE) + "
                    "gp_allocate x5 + gp_sched_ratio -> D2H counts, verdicts, per-set results "
                    "(second copy stream), every step inside the timed region; two slots of "
                    "inputs and outputs, so step k+1's H2D and step k-1's D2H overlap step k"
                    + ("; the compute replayed as one CUDA graph per slot"
                       if egraphs is not None else "")}


if __name__ == "__main__":
    sys.exit(main())
