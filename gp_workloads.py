"""gp_workloads -- the neutral input module shared by the oracle and the CUDA path.

Holds the workload *recipes* (SURVEY.md §8(d) configs C1-C5 as plain dicts)
and seeded numpy generators of small random task sets for tests.  It holds
none of the method's arithmetic: no WCET, no demand test, no heuristic, no
task-set generator step.  Both ``oracle`` and ``paper_2105_10312_b200`` accept
these plain dicts / arrays; neither imports the other.

Parameter encodings (all integers):
  * prm_q = floor(prm * 2^32): a task is memory-intensive iff its Philox word
    w0 < prm_q (reading A-15), so 2^31 is prm = 50 %.
  * period_menu in paper time units (reading A-11); ticks = units*Q.
  * beta = beta_*_num / beta_den  (0.02 compute, 0.1 memory).
  * k    = k*_num / k_den         (1.2 compute, 2.3 memory).
"""
from __future__ import annotations

import numpy as np

SEED = 0x2105_10312
MENU = (50, 100, 200, 400, 500, 1000, 2000, 4000)  # reading A-11
Q = 1000                                            # ticks per paper time unit (C.1.1)

PRM_Q = {0.0: 0, 0.25: 1 << 30, 0.5: 1 << 31, 0.75: 3 << 30, 1.0: 1 << 32}

VARIANT_NAMES = ("1G", "SMS_ACT", "SMS_INA", "BF_ACT", "BF_INA")


def _same_den(kc, km):
    assert kc[1] == km[1], "k_C and k_M must share a denominator"
    return kc[1]


def gen_params(M, n_tasks, sets_per_group, n_bins=10, prm=(0.5,), kc=(12, 10), km=(23, 10),
               max_attempts=1000, curve_gran=0, b_per_sm=False):
    """Generator parameters in the integer encoding both sides accept."""
    return dict(
        M=M, n_tasks=n_tasks, n_bins=n_bins, n_prm=len(prm), sets_per_group=sets_per_group,
        prm_q=[PRM_Q[p] for p in prm], ticks_per_unit=Q, period_menu=list(MENU),
        b_max=4 * M,                       # reading A-13: B ~ U{1..4M}
        # b = beta * a (reading A-1); b_per_sm: b = beta * a / M (reading A-1b, f1 only)
        beta_c_num=2, beta_m_num=10, beta_den=100 * (M if b_per_sm else 1),
        kc_num=kc[0], km_num=km[0], k_den=_same_den(kc, km),
        max_attempts=max_attempts,
        curve_gran=curve_gran,  # > 0: §7.1 curve C = k(a/|P| + b) in the W form (f1, reading A-1)
    )


# (k_C, k_M) coefficient settings of C5, tenths: {1.0,1.2,1.5,2.0} x {1.0,1.5,2.3,3.0}
C5_SETTINGS = [(kc, km) for kc in (10, 12, 15, 20) for km in (10, 15, 23, 30)]


def _c1_sets():
    """C1: the paper's worked example scaled to exhaustive: M=4, three
    tasks of B=5 blocks, T=20, D=7, C^M=1, C^C=2 (BASELINE.json configs[0]),
    Q=1 (paper units).  All 8 type vectors; vector 0 = CCC (reading A-29)."""
    S, n = 8, 3
    types = np.array([[(v >> (n - 1 - i)) & 1 for i in range(n)] for v in range(S)], np.uint8)
    full = lambda x: np.full((S, n), x, np.int32)  # noqa: E731
    return dict(M=4, n_groups=1, T=full(20), D=full(7), B=full(5), cn=full(1), cc=full(2),
                fn=full(0), fc=full(0), type=types, valid=np.ones(S, np.uint8),
                group=np.zeros(S, np.int32))


WORKLOADS = {
    "c1": dict(name="c1_worked_example", M=4, n=3, sets=_c1_sets, exhaustive=True,
               variants=VARIANT_NAMES),
    "c2": dict(name="c2_embedded_8sm", M=8, n=6, exhaustive=True, variants=VARIANT_NAMES,
               gen=lambda R=10000: gen_params(8, 6, R)),
    "c3": dict(name="c3_exhaustive_20sm", M=20, n=6, exhaustive=True, variants=VARIANT_NAMES,
               gen=lambda R=1000: gen_params(20, 6, R)),
    "c4": dict(name="c4_b200_148sm", M=148, n=32, exhaustive=False, variants=VARIANT_NAMES,
               gen=lambda R=20000: gen_params(148, 32, R, prm=(0.0, 0.25, 0.5, 0.75, 1.0))),
    "c5": dict(name="c5_coeff_sweep_68sm", M=68, n=16, exhaustive=False, variants=VARIANT_NAMES,
               gen=lambda R=10000, kc=12, km=23: gen_params(68, 16, R, kc=(kc, 10), km=(km, 10))),
    # §8(f) f1: the paper's own experiment (§7.2; Figs 5 and 7): RTX 2080 Ti shape
    # (M = 68), 50 or 200 tasks, total utilisation 2, 4, ..., 68 (34 bins of U/M = bin/34),
    # 100 task sets per point, prm 50 %, the §7.1 curves in curve mode (10-tick granules).
    "f1_50": dict(name="f1_paper_68sm_50tasks", M=68, n=50, exhaustive=False,
                  variants=VARIANT_NAMES,
                  gen=lambda R=100: gen_params(68, 50, R, n_bins=34, curve_gran=10)),
    "f1_200": dict(name="f1_paper_68sm_200tasks", M=68, n=200, exhaustive=False,
                   variants=VARIANT_NAMES,
                   gen=lambda R=100: gen_params(68, 200, R, n_bins=34, curve_gran=10)),
    # the same sweep under reading A-1b: the non-parallel part b measured in all-SM time
    # (b = beta * a / M), the reading under which P:975's 1G plateau (U < 35) is reachable
    "f1b_50": dict(name="f1b_paper_68sm_50tasks_b_per_sm", M=68, n=50, exhaustive=False,
                   variants=VARIANT_NAMES,
                   gen=lambda R=100: gen_params(68, 50, R, n_bins=34, curve_gran=10,
                                                b_per_sm=True)),
    "f1b_200": dict(name="f1b_paper_68sm_200tasks_b_per_sm", M=68, n=200, exhaustive=False,
                    variants=VARIANT_NAMES,
                    gen=lambda R=100: gen_params(68, 200, R, n_bins=34, curve_gran=10,
                                                 b_per_sm=True)),
}


# --------------------------------------------------------------------------
# Seeded random inputs for tests (no method arithmetic)
# --------------------------------------------------------------------------

def random_edf_instance(rng: np.random.Generator, max_tasks=6, max_h=10_000):
    """Random (C, D, T) lists with D <= T, small hyperperiod."""
    periods = [p for p in (2, 3, 4, 5, 6, 8, 10, 12, 15, 16, 20, 24, 25, 30, 40, 50, 60)]
    while True:
        n = int(rng.integers(1, max_tasks + 1))
        T = [int(rng.choice(periods)) for _ in range(n)]
        H = int(np.lcm.reduce(np.array(T, dtype=np.int64)))
        if H <= max_h:
            break
    D = [int(rng.integers(1, t + 1)) for t in T]
    C = [int(rng.integers(0, max(1, d) + 1)) for d in D]
    return C, D, T


def random_sets(rng: np.random.Generator, n_sets, n_tasks, M, periods=(20, 40, 50, 100, 200),
                b_max=None, cost_max=8, n_groups=1):
    """Random task-set batch (dict of arrays, fields [n_sets][n_tasks]) obeying
    the model invariants of §8(c) C.1.2 (0<D<=T, 1<=cn<=cc, 0<=fn<=fc, B>=1)."""
    b_max = b_max or 2 * M
    shp = (n_sets, n_tasks)
    T = rng.choice(np.array(periods, np.int32), size=shp).astype(np.int32)
    D = np.maximum(1, (T * rng.integers(50, 101, size=shp)) // 100).astype(np.int32)
    B = rng.integers(1, b_max + 1, size=shp).astype(np.int32)
    cn = rng.integers(1, cost_max + 1, size=shp).astype(np.int32)
    cc = (cn + rng.integers(0, cost_max + 1, size=shp)).astype(np.int32)
    fn = rng.integers(0, cost_max + 1, size=shp).astype(np.int32)
    fc = (fn + rng.integers(0, cost_max + 1, size=shp)).astype(np.int32)
    typ = rng.integers(0, 2, size=shp).astype(np.uint8)
    return dict(M=M, n_groups=n_groups, T=T, D=D, B=B, cn=cn, cc=cc, fn=fn, fc=fc, type=typ,
                valid=np.ones(n_sets, np.uint8),
                group=rng.integers(0, n_groups, size=n_sets).astype(np.int32))
