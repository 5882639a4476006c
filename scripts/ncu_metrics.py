#!/usr/bin/env python
"""Fold an ncu --set full report into profiles/rNN/ncu_metrics.json (the
entry bench.py's roofline.traffic / ncu_issue fields read).

  python scripts/ncu_metrics.py REPORT KEY [--out profiles/r01/ncu_metrics.json]
      [--candidates N] [--note TEXT]

KEY is the bench workload name (e.g. c3_exhaustive_20sm).  All launches in the
report are combined: durations summed, issue/pipe percentages time-weighted,
dram bytes (dram__bytes_read.sum + dram__bytes_write.sum) summed per step.
"""
import argparse
import csv
import io
import json
import subprocess


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    global UNITS
    UNITS = dict(zip(hdr, units))
    return [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


UNITS = {}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3,
         "usecond": 1e-3, "msecond": 1, "ms": 1, "s": 1e3, "second": 1e3, "nsecond": 1e-6}


def f(r, k):
    """Value in bytes (memory metrics) or ms (durations), per the ncu unit row."""
    try:
        v = float(r[k].replace(",", ""))
    except (KeyError, ValueError, AttributeError):
        return None
    if v != v:  # NaN: metric not collected for this launch
        return None
    return v * SCALE.get(UNITS.get(k, ""), 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("key")
    ap.add_argument("--out", default="profiles/r01/ncu_metrics.json")
    ap.add_argument("--candidates", type=float, default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    rs = raw(a.report)
    per = []
    for r in rs:
        dur_ms = f(r, "gpu__time_duration.sum")
        per.append({
            "kernel": r.get("Kernel Name", "?").split("(")[0],
            "duration_ms": dur_ms,
            "inst_issued_pct": f(r, "sm__inst_issued.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": f(r, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": f(r, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "warp_inst_executed": f(r, "smsp__inst_executed.sum"),
            "active_threads_per_inst": f(r, "smsp__thread_inst_executed_per_inst_executed.ratio"),
            "dram_bytes": (None if f(r, "dram__bytes_read.sum") is None
                       else f(r, "dram__bytes_read.sum") + (f(r, "dram__bytes_write.sum") or 0)),
        })
    T = sum(p["duration_ms"] or 0 for p in per)

    def tw(k):  # time-weighted over the launches that have the metric
        have = [p for p in per if p[k] is not None and p["duration_ms"]]
        t = sum(p["duration_ms"] for p in have)
        return sum(p[k] * p["duration_ms"] for p in have) / t if t else None
    ent = {
        "kernel": " + ".join(p["kernel"] for p in per),
        "dram_bytes": sum(p["dram_bytes"] for p in per if p["dram_bytes"] is not None),
        "duration_ms": T,
        "inst_issued_pct": tw("inst_issued_pct"),
        "alu_pipe_pct": tw("alu_pipe_pct"),
        "fma_pipe_pct": tw("fma_pipe_pct"),
        "warp_inst_executed": sum(p["warp_inst_executed"] or 0 for p in per),
        "launches_missing_metrics": sum(1 for p in per if p["inst_issued_pct"] is None),
        "active_threads_per_inst": tw("active_threads_per_inst"),
        "per_kernel": per,
        "note": a.note,
    }
    if a.candidates:
        ent["candidates"] = a.candidates
        ent["warp_inst_per_candidate"] = ent["warp_inst_executed"] / a.candidates
    try:
        m = json.load(open(a.out))
    except (OSError, ValueError):
        m = {}
    if a.key in m:
        m[a.key + "_prev"] = m[a.key]
    m[a.key] = ent
    json.dump(m, open(a.out, "w"), indent=1)
    print(json.dumps(ent, indent=1)[:1500])


if __name__ == "__main__":
    main()
