#!/usr/bin/env python
"""Per-variant heuristic work counters (GP_AL_STATS_EXT) and kernel times on one config.
  python scripts/alloc_stats.py [c4|c5|c3|c2] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gp_workloads as W  # noqa: E402
from paper_2105_10312_b200 import gpart as G  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
gen = W.WORKLOADS[key]["gen"](R=reps)
ng = gen["n_prm"] * gen["n_bins"]
ts = G.TaskSets(ng * reps, gen["n_tasks"], gen["M"], ng)
G.gp_generate(gen, W.SEED, 0, reps, ts)
names = ["tests_counted", "tasks", "deadlines", "sets", "tests_run", "selections", "scanned",
         "partner_searches"]
for v in W.VARIANT_NAMES:
    st = torch.zeros(8, dtype=torch.int64, device="cuda")
    out = G.gp_allocate(ts, v, stats=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    G.gp_allocate(ts, v, out)
    e1.record()
    torch.cuda.synchronize()
    s = st.cpu().tolist()
    S = s[3]
    print(f"{v:8s} {e0.elapsed_time(e1):8.3f} ms  " + "  ".join(f"{n}/set {x / S:8.2f}" for n, x in zip(names, s) if n != "sets"))
