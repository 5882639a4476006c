#!/usr/bin/env python
"""Summarise an ncu report (--set full) or a launch-list CSV into profiles/.

  python scripts/ncu_summary.py report.ncu-rep [--top 25] > profiles/rNN/xxx.txt
  python scripts/ncu_summary.py --launches launches.csv > profiles/rNN/launches.txt

For a report: per kernel launch the speed-of-light, issue, occupancy,
divergence, DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and the
hottest source lines (needs -lineinfo + --import-source on).
"""
import argparse
import collections
import csv
import json
import subprocess
import sys

DETAILS = ["Duration", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
           "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "No Eligible",
           "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
           "Avg. Not Predicated Off Threads Per Warp", "Branch Efficiency",
           "Executed Instructions", "Registers Per Thread", "Theoretical Occupancy",
           "Achieved Occupancy", "Achieved Active Warps Per SM", "Grid Size", "Block Size",
           "Dynamic Shared Memory Per Block", "L1/TEX Hit Rate", "L2 Hit Rate"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_issued.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__thread_inst_executed_per_inst_executed.ratio", "gpu__time_duration.sum",
       "launch__registers_per_thread", "smsp__inst_executed.sum"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def details(rep):
    rows = list(csv.reader(ncu("-i", rep, "--page", "details", "--csv").splitlines()))
    h = rows[0]
    out = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        key = (d.get("ID"), d.get("Kernel Name", "")[:60])
        if d.get("Metric Name") in DETAILS:
            out.setdefault(key, {})[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}".strip()
    return out


def raw(rep):
    rows = list(csv.reader(ncu("-i", rep, "--page", "raw", "--csv").splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        e = {k: d.get(k) for k in RAW if k in d} | {"Kernel Name": d.get("Kernel Name", "")[:60],
                                                   "ID": d.get("ID")}
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):  # -> bytes
            u = units[h.index(k)] if k in h else "byte"
            sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            try:
                e[k] = str(float(e[k].replace(",", "")) * sc)
            except (KeyError, AttributeError, ValueError):
                pass
        res.append(e)
    return res


def stalls(rep):
    rows = list(csv.reader(ncu("-i", rep, "--page", "raw", "--csv").splitlines()))
    h = rows[0]
    res = []
    for r in rows[2:]:
        items = [(n.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "") or 0))
                 for n, v in zip(h, r)
                 if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
        tot = sum(v for _, v in items) or 1
        res.append(", ".join(f"{n} {100 * v / tot:.1f}%" for n, v in sorted(items, key=lambda t: -t[1])[:8]))
    return res


def source_top(rep, top, launch=None):
    args = ["-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if launch is not None:
        args += ["--launch-skip", str(launch), "--launch-count", "1"]
    rows = list(csv.reader(ncu(*args).splitlines()))
    cur, agg = None, {}
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if not r or r[0] in ("Function Name", "Line No") or len(r) < 8 or r[0] == "":
            continue
        try:
            ie = int(r[7]) if r[7] not in ("-", "") else 0
            samp = int(r[4]) if r[4] not in ("-", "") else 0
        except ValueError:
            continue
        k = (cur, int(r[0]))
        a = agg.get(k, (0, 0, r[1][:80]))
        agg[k] = (a[0] + ie, a[1] + samp, a[2])
    tot = sum(v[0] for v in agg.values()) or 1
    tots = sum(v[1] for v in agg.values()) or 1
    lines = [f"  {'file':18s}{'line':>5s} {'inst%':>7s} {'stall%':>7s}  source"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        lines.append(f"  {k[0]:18s}{k[1]:5d} {100 * v[0] / tot:6.2f}% {100 * v[1] / tots:6.2f}%  {v[2]}")
    return "\n".join(lines)


def launches(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            h, start = r, i
            break
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    order = []
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
        order.append(name)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'mean_us':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:60]:60s} {len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {100 * sum(v) / tot:6.2f}%")
    print(f"(gpu__time_duration.sum, ncu --clock-control none: cold-cache and serialised; compare shares)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("--launches")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--json", action="store_true")
    a = ap.parse_args()
    if a.launches:
        return launches(a.launches)
    det = details(a.report)
    rw = raw(a.report)
    st = stalls(a.report)
    if a.json:
        print(json.dumps({"raw": rw}, indent=1))
        return
    for idx, (key, d) in enumerate(det.items()):
        print(f"== launch {key[0]}: {key[1]}")
        for m in DETAILS:
            if m in d:
                print(f"  {m:42s} {d[m]}")
        if idx < len(rw):
            r = rw[idx]
            try:
                tr = float(r["dram__bytes_read.sum"].replace(",", "")) + float(
                    r["dram__bytes_write.sum"].replace(",", ""))
                print(f"  {'DRAM traffic (read+write)':42s} {tr:.0f} bytes")
            except (KeyError, AttributeError, ValueError):
                pass
            for k in RAW[2:7]:
                if r.get(k):
                    print(f"  {k:42s} {r[k]}")
        if idx < len(st):
            print(f"  stall mix: {st[idx]}")
        print(source_top(a.report, a.top, launch=idx))
        print()


if __name__ == "__main__":
    sys.exit(main())
