#!/usr/bin/env python
"""§8(f) f1: the paper's own experiment on the GPU path (§7.2).

M = 68 SMs (RTX 2080 Ti shape), 50 and 200 tasks, total utilisation
2, 4, ..., 68, 100 task sets per point, prm 50 %, all five variants (1G,
SMS_ACT, SMS_INA, BF_ACT, BF_INA), task sets in curve mode (the §7.1 curves).
Reports per U point: schedulability rate (Figs 5, 7), mean number of
partitions of the solutions, scheduled workload between its bounds
(Figs 6, 8; f2) and EDF tests per set (the analysis-time analogue, Fig. 9),
plus the GPU time of the whole sweep.

  python scripts/f1_sweep.py [--reps 100] [--out profiles/r01/f1_sweep.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gp_workloads as W  # noqa: E402
from paper_2105_10312_b200 import gpart as G  # noqa: E402


def run(key, reps):
    wl = W.WORKLOADS[key]
    gen = wl["gen"](R=reps)
    n, M = wl["n"], wl["M"]
    ts = G.TaskSets(34 * reps, n, M, 34)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    G.gp_generate(gen, W.SEED, 0, reps, ts)
    outs = {}
    stats = torch.zeros(4, dtype=torch.int64, device="cuda")
    for v in W.VARIANT_NAMES:
        outs[v] = G.gp_allocate(ts, v, G.AllocOut(ts.n_sets, n).want_efficiency(), stats=stats)
    counts = torch.zeros((1, 34, len(W.VARIANT_NAMES), 3), dtype=torch.int64, device="cuda")
    verdicts = torch.stack([outs[v].ok for v in W.VARIANT_NAMES])
    G.gp_sched_ratio(ts, G.GP_FROM_VERDICTS, counts, verdicts=verdicts, slot0=0,
                     n_slots=len(W.VARIANT_NAMES))
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    c = counts.cpu().numpy()[0]
    valid = ts.valid.cpu().numpy().reshape(34, reps)
    res = {"workload": wl["name"], "n": n, "M": M, "reps": reps, "gpu_ms": ms,
           "edf_tests": int(stats[0].item()), "U": [2 * (b + 1) for b in range(34)],
           "valid_rate": valid.mean(1).tolist(), "variants": {}}
    for vi, v in enumerate(W.VARIANT_NAMES):
        h = outs[v].to_host()
        ok = h["ok"].reshape(34, reps).astype(bool)
        k = h["k"].reshape(34, reps)
        eff = h["efficiency"].reshape(34, reps, 4).astype(np.float64)
        tests = h["n_tests"].reshape(34, reps)
        rate = (c[:, vi, 0] / np.maximum(c[:, vi, 1], 1)).tolist()
        mean_k = [float(k[b][ok[b]].mean()) if ok[b].any() else None for b in range(34)]
        # scheduled workload / bounds in utilisation units (divide the H-scaled sums by H)
        ach = [float((eff[b, ok[b], 2] / eff[b, ok[b], 3]).mean()) if ok[b].any() else None
               for b in range(34)]
        lo = [float((eff[b, :, 0] / eff[b, :, 3]).mean()) for b in range(34)]
        up = [float((eff[b, :, 1] / eff[b, :, 3]).mean()) for b in range(34)]
        res["variants"][v] = {"sched_rate": rate, "mean_partitions": mean_k,
                              "workload_achieved": ach, "workload_lower": lo, "workload_upper": up,
                              "edf_tests_per_set": tests.mean(1).tolist()}
    return res


def claims(r50, r200):
    """The paper's qualitative claims."""
    out = {}
    U = r50["U"]
    heur = ("SMS_ACT", "SMS_INA", "BF_ACT", "BF_INA")
    v50 = r50["variants"]
    out["heuristics_100pct_below_U"] = {
        v: max([u for u, x in zip(U, v50[v]["sched_rate"]) if x == 1.0] or [0]) for v in heur}
    out["1G_last_U_at_100pct"] = max([u for u, x in zip(U, v50["1G"]["sched_rate"]) if x == 1.0]
                                     or [0])
    out["dominance_heuristics_ge_1G_every_U"] = {
        v: all(a >= b for a, b in zip(v50[v]["sched_rate"], v50["1G"]["sched_rate"])) for v in heur}
    ks = [x for x in v50["SMS_ACT"]["mean_partitions"] if x is not None]
    out["SMS_ACT_mean_partitions_n50"] = float(np.mean(ks)) if ks else None
    tests = {v: float(np.mean(v50[v]["edf_tests_per_set"])) for v in heur}
    out["edf_tests_per_set_n50"] = tests
    out["ACT_cheaper_than_INA"] = {f"{a}<{b}": tests[a] < tests[b]
                                   for a, b in (("SMS_ACT", "SMS_INA"), ("BF_ACT", "BF_INA"))}
    if r200:
        v200 = r200["variants"]
        spread = [max(v200[v]["sched_rate"][b] for v in heur) - min(v200[v]["sched_rate"][b]
                                                                    for v in heur)
                  for b in range(34)]
        out["n200_max_spread_between_heuristics"] = float(max(spread))
        spread50 = [max(v50[v]["sched_rate"][b] for v in heur) - min(v50[v]["sched_rate"][b]
                                                                     for v in heur)
                    for b in range(34)]
        out["n50_max_spread_between_heuristics"] = float(max(spread50))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "f1_sweep.json"))
    ap.add_argument("--skip200", action="store_true")
    a = ap.parse_args()
    t0 = time.time()
    r50 = run("f1_50", a.reps)
    r200 = None if a.skip200 else run("f1_200", a.reps)
    res = {"f1_50": r50, "f1_200": r200, "claims": claims(r50, r200),
           "wall_s": time.time() - t0, "device": torch.cuda.get_device_name()}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(res, fh, indent=1)
    for r in (r50, r200):
        if not r:
            continue
        print(f"== {r['workload']}: {r['reps']} sets/point, GPU {r['gpu_ms']:.1f} ms, "
              f"{r['edf_tests']} EDF tests")
        print("U    " + " ".join(f"{v:>8s}" for v in W.VARIANT_NAMES))
        for b, u in enumerate(r["U"]):
            print(f"{u:3d}  " + " ".join(f"{r['variants'][v]['sched_rate'][b]:8.2f}"
                                          for v in W.VARIANT_NAMES))
    print(json.dumps(res["claims"], indent=1))


if __name__ == "__main__":
    main()
