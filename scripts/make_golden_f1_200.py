#!/usr/bin/env python
"""Golden oracle outputs for the f1 200-task scenario at load (the
paper's Fig. 7 setting): U = 30, 32, ..., 50 (bins 14..24 of 34), the first
REPS sets of each point, all five variants.  Calls only oracle/ (test infrastructure):
the oracle needs minutes per loaded 200-task set, too slow for the GPU test run, so the
GPU test compares against this committed file (regenerate: python scripts/make_golden_f1_200.py).
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gp_workloads as W  # noqa: E402
import oracle  # noqa: E402

REPS = int(os.environ.get("REPS", "2"))
BINS = list(range(14, 25))  # U = 2 (b + 1) = 30 .. 50


def main(out=os.path.join(ROOT, "tests", "golden", "f1_200_load.npz")):
    gen = W.WORKLOADS["f1_200"]["gen"](R=100)
    s = oracle.generate(gen, W.SEED, 0, REPS)  # local set = bin * REPS + rep
    idx = [b * REPS + r for b in BINS for r in range(REPS)]
    sub = s.subset(idx)
    res = {"idx": np.array(idx, np.int32), "reps": np.int32(REPS), "bins": np.array(BINS)}
    for f in ("T", "D", "B", "cn", "cc", "fn", "fc", "type", "valid"):
        res[f"set_{f}"] = getattr(sub, f)
    for v in W.VARIANT_NAMES:
        t = time.time()
        r = oracle.allocate(sub, v)
        for k, a in r.items():
            res[f"{v}_{k}"] = a
        print(f"{v}: {time.time() - t:.1f} s, ok {int(r['ok'].sum())}/{sub.n_sets}", flush=True)
    np.savez_compressed(out, **res)
    print("wrote", out)


if __name__ == "__main__":
    main()
