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


def run(key, reps, flags=0, sizes=None):
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
    ev = []
    for v in W.VARIANT_NAMES:
        ev.append(torch.cuda.Event(enable_timing=True))
        ev[-1].record(st)
        outs[v] = G.gp_allocate(ts, v, G.AllocOut(ts.n_sets, n).want_efficiency(), stats=stats,
                                flags=flags, sizes=sizes)
    ev.append(torch.cuda.Event(enable_timing=True))
    ev[-1].record(st)
    counts = torch.zeros((1, 34, len(W.VARIANT_NAMES), 3), dtype=torch.int64, device="cuda")
    verdicts = torch.stack([outs[v].ok for v in W.VARIANT_NAMES])
    G.gp_sched_ratio(ts, G.GP_FROM_VERDICTS, counts, verdicts=verdicts, slot0=0,
                     n_slots=len(W.VARIANT_NAMES))
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    variant_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(W.VARIANT_NAMES))]
    c = counts.cpu().numpy()[0]
    valid = ts.valid.cpu().numpy().reshape(34, reps)
    res = {"workload": wl["name"], "n": n, "M": M, "reps": reps, "gpu_ms": ms, "flags": flags,
           "sizes": sizes,
           "edf_tests": int(stats[0].item()), "U": [2 * (b + 1) for b in range(34)],
           "valid_rate": valid.mean(1).tolist(), "variants": {}}
    res["variant_gpu_ms"] = dict(zip(W.VARIANT_NAMES, variant_ms))
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
    """SPEC acceptance 3-7 (the paper's qualitative claims P:975, P:1014, P:1053,
    P:1121-1125), evaluated on this sweep; each entry holds the measured
    quantity and whether the criterion holds."""
    heur = ("SMS_ACT", "SMS_INA", "BF_ACT", "BF_INA")
    U = r50["U"]
    v50 = r50["variants"]
    out = {}
    # 3. every variant (1G included) schedules 100 % for U <= 30
    last100 = {v: max([u for u, x in zip(U, v50[v]["sched_rate"]) if x == 1.0] or [0])
               for v in W.VARIANT_NAMES}
    out["3_plateau_U_le_30"] = {"last_U_at_100pct": last100, "holds": all(
        all(x == 1.0 for u, x in zip(U, v50[v]["sched_rate"]) if u <= 30) for v in W.VARIANT_NAMES)}
    # 4. 1G <= 0.1 by U = 45, heuristics >= 1G everywhere, >= 0.3 better somewhere in [36, 50]
    g = v50["1G"]["sched_rate"]
    dom = all(all(a >= b for a, b in zip(v50[v]["sched_rate"], g)) for v in heur)
    gap = max(v50[v]["sched_rate"][i] - g[i] for v in heur for i, u in enumerate(U) if 36 <= u <= 50)
    g45 = [x for u, x in zip(U, g) if 44 <= u <= 46]
    out["4_1G_collapse_dominance"] = {"1G_rate_U44_46": g45, "max_gain_U36_50": gap,
                                      "dominance": dom,
                                      "holds": dom and max(g45) <= 0.1 and gap >= 0.3}
    # 5. at U where all SMS_ACT runs succeed: achieved within 10 % of the lower bound and
    #    mean partition count 25 +- 5
    sa = v50["SMS_ACT"]
    idx = [i for i in range(len(U)) if sa["sched_rate"][i] == 1.0]
    eff = [sa["workload_achieved"][i] / sa["workload_lower"][i] for i in idx]
    kk = [sa["mean_partitions"][i] for i in idx]
    out["5_pairing_efficiency"] = {
        "U_all_succeed": [U[i] for i in idx], "mean_achieved_over_lower": float(np.mean(eff)),
        "mean_partitions": float(np.mean(kk)),
        "holds": float(np.mean(eff)) <= 1.10 and abs(float(np.mean(kk)) - 25) <= 5}
    # 6. n = 200: heuristics within 0.15 of each other at every U, all dominate 1G
    if r200:
        v200 = r200["variants"]
        spread = [max(v200[v]["sched_rate"][b] for v in heur) -
                  min(v200[v]["sched_rate"][b] for v in heur) for b in range(len(U))]
        dom200 = all(all(a >= b for a, b in zip(v200[v]["sched_rate"], v200["1G"]["sched_rate"]))
                     for v in heur)
        out["6_n200_convergence"] = {"max_spread": float(max(spread)), "dominance": dom200,
                                     "holds": max(spread) <= 0.15 and dom200}
    # 7. analysis cost over the high-load region (U >= 36): ACT < INA and BF < SMS.
    #    Measured as EDF tests per set (the work unit; GPU time is per variant, whole sweep)
    hi = [i for i, u in enumerate(U) if u >= 36]
    t = {v: float(np.mean([v50[v]["edf_tests_per_set"][i] for i in hi])) for v in heur}
    order = {"SMS_ACT<SMS_INA": t["SMS_ACT"] < t["SMS_INA"], "BF_ACT<BF_INA": t["BF_ACT"] < t["BF_INA"],
             "BF_ACT<SMS_ACT": t["BF_ACT"] < t["SMS_ACT"], "BF_INA<SMS_INA": t["BF_INA"] < t["SMS_INA"]}
    out["7_analysis_cost_order"] = {"edf_tests_per_set_U_ge_36": t, "order": order,
                                    "gpu_ms_whole_sweep": r50["variant_gpu_ms"],
                                    "holds": all(order.values())}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "f1_sweep.json"))
    ap.add_argument("--skip200", action="store_true")
    ap.add_argument("--f4", action="store_true", help="also run the f4 variants (n = 50)")
    ap.add_argument("--readings", default="A-1,A-1b",
                    help="A-1: b = beta*a (P:950 as written); A-1b: b = beta*a/M")
    a = ap.parse_args()
    t0 = time.time()
    res = {"device": torch.cuda.get_device_name()}
    for reading in a.readings.split(","):
        pre = {"A-1": "f1", "A-1b": "f1b"}[reading]
        r50 = run(pre + "_50", a.reps)
        r200 = None if a.skip200 else run(pre + "_200", a.reps)
        res[reading] = {"n50": r50, "n200": r200, "claims": claims(r50, r200)}
        for r in (r50, r200):
            if not r:
                continue
            print(f"== {reading} {r['workload']}: {r['reps']} sets/point, GPU {r['gpu_ms']:.1f} ms, "
                  f"{r['edf_tests']} EDF tests")
            print("U    " + " ".join(f"{v:>8s}" for v in W.VARIANT_NAMES))
            for b, u in enumerate(r["U"]):
                print(f"{u:3d}  " + " ".join(f"{r['variants'][v]['sched_rate'][b]:8.2f}"
                                              for v in W.VARIANT_NAMES))
        print(reading, json.dumps(res[reading]["claims"], indent=1))
    if a.f4:
        # f4 variants at paper scale (reading A-1): binary merge, increasing order,
        # MIG-style slices (1/7, 2/7, 3/7, 4/7, 7/7 of the 68 SMs)
        mig = sorted({max(1, (68 * g) // 7) for g in (1, 2, 3, 4, 7)})
        f4 = {}
        for name, fl, sz in (("binary", G.GP_AL_BINARY_MERGE, None),
                             ("increasing", G.GP_AL_INCREASING, None),
                             ("mig_slices", 0, mig), ("mig_slices_binary", G.GP_AL_BINARY_MERGE, mig)):
            r = run("f1_50", a.reps, fl, sz)
            f4[name] = {"gpu_ms": r["gpu_ms"], "edf_tests": r["edf_tests"],
                        "variant_gpu_ms": r["variant_gpu_ms"], "sizes": sz,
                        "sched_rate": {v: r["variants"][v]["sched_rate"] for v in W.VARIANT_NAMES},
                        "mean_tests_per_set": {v: float(np.mean(r["variants"][v]["edf_tests_per_set"]))
                                               for v in W.VARIANT_NAMES}}
            print(f"f4 {name}: GPU {r['gpu_ms']:.1f} ms, {r['edf_tests']} EDF tests")
        res["f4_n50"] = f4
    res["wall_s"] = time.time() - t0
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
