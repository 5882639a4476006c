"""Time GP_EXHAUSTIVE on C3 with each evaluator (events) -- a dev helper."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import gp_workloads as W
from paper_2105_10312_b200 import gpart as G

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
wl = W.WORKLOADS[cfg]
gen = wl["gen"](R=reps)
ts = G.TaskSets(10 * reps, wl["n"], wl["M"], 10)
G.gp_generate(gen, W.SEED, 0, reps, ts)
per = torch.empty((ts.n_sets, 4), dtype=torch.int64, device="cuda")
work = torch.zeros(1, dtype=torch.int64, device="cuda")
res = {}
for name, fl in (("bitsliced", 0), ("bitsliced_nohash", 1), ("per_candidate", 2)):
    outs = []
    for rep in range(4):
        st = torch.zeros(4, dtype=torch.int64, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        G.gp_sched_ratio(ts, G.GP_EXHAUSTIVE, None, per_set=per, work_counter=work, stats=st, flags=fl)
        e1.record()
        torch.cuda.synchronize()
        outs.append(e0.elapsed_time(e1))
    res[name] = {"ms": outs, "stats": st.cpu().tolist(), "n_sched": int(per[:, 0].sum().item()),
                 "hash": int(per[:, 3].sum().item()) & ((1 << 64) - 1)}
    print(name, ["%.2f" % x for x in outs], res[name]["stats"], res[name]["n_sched"])
