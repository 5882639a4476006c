"""Pins of the oracle's per-partition schedulability test (A4).

The policy is preemptive EDF with the processor-demand criterion (paper leaves
it open; reading A-6).  Pins: SPEC worked
values, the textbook reductions (single task, implicit deadlines = Liu &
Layland), a brute-force EDF simulation over one hyperperiod,
witness validity recomputed from the dbf definition, resource monotonicity.
"""
import json
import os
from fractions import Fraction

import numpy as np

import gp_workloads as W
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_spec_edf_examples():
    with open(os.path.join(GOLD, "spec_examples.json")) as f:
        ex = json.load(f)["edf_demand_test"]
    for e in ex:
        C = [t[0] for t in e["tasks_CDT"]]
        D = [t[1] for t in e["tasks_CDT"]]
        T = [t[2] for t in e["tasks_CDT"]]
        ok, wit, _ = oracle.edf_pdc(C, D, T)
        assert ok == e["schedulable"], e["S"]
        if not ok:
            assert wit == e["witness"]
            # demand at the witness (13 > 12), recomputed by hand-listing jobs
            jobs = sum(C[i] for i in range(len(C)) for q in range(100) if D[i] + q * T[i] <= wit)
            assert jobs == e["demand_at_witness"]
        if C:
            assert oracle.simulate_edf(C, D, T, oracle.hyperperiod(T)) == e["schedulable"]


def test_single_task_iff_c_le_d():
    """Textbook: one task is EDF-schedulable iff C <= D."""
    for T in (5, 7, 20):
        for D in range(1, T + 1):
            for Cv in range(0, T + 2):
                ok, _, _ = oracle.edf_pdc([Cv], [D], [T])
                assert ok == (Cv <= D)


def test_implicit_deadlines_liu_layland():
    """D_i = T_i: EDF schedulable iff sum C_i/T_i <= 1 (Liu & Layland 1973)."""
    rng = np.random.default_rng(3)
    for _ in range(800):
        n = int(rng.integers(1, 6))
        T = [int(rng.choice([2, 3, 4, 5, 6, 8, 10, 12, 15, 20])) for _ in range(n)]
        C = [int(rng.integers(0, t + 1)) for t in T]
        ok, _, _ = oracle.edf_pdc(C, T, T)
        assert ok == (sum(Fraction(c, t) for c, t in zip(C, T)) <= 1)


def test_pdc_equals_simulation():
    """SPEC acceptance 1: agreement with a unit-tick EDF simulation
    over one hyperperiod on 1,000 random instances (<= 6 tasks, H <= 10^4)."""
    rng = np.random.default_rng(4)
    mism = 0
    for _ in range(1000):
        C, D, T = W.random_edf_instance(rng)
        ok, _, _ = oracle.edf_pdc(C, D, T)
        sim = oracle.simulate_edf(C, D, T, oracle.hyperperiod(T))
        mism += ok != sim
    assert mism == 0


def _dbf(C, D, T, t):
    # job-by-job demand: every job with release r = q*T and deadline r+D <= t
    tot = 0
    for c, d, p in zip(C, D, T):
        q = 0
        while q * p + d <= t:
            tot += c
            q += 1
    return tot


def test_witness_is_min_violating_deadline():
    """the witness is an absolute deadline whose demand exceeds it, and
    no earlier deadline violates."""
    rng = np.random.default_rng(5)
    seen = 0
    for _ in range(600):
        C, D, T = W.random_edf_instance(rng, max_tasks=5, max_h=2000)
        ok, wit, _ = oracle.edf_pdc(C, D, T)
        if ok:
            continue
        seen += 1
        assert any((wit - d) % p == 0 and wit >= d for d, p in zip(D, T))
        assert _dbf(C, D, T, wit) > wit
        H = oracle.hyperperiod(T)
        earlier = sorted({d + q * p for d, p in zip(D, T) for q in range(H // p + 1)
                          if d + q * p < wit})
        assert all(_dbf(C, D, T, t) <= t for t in earlier)
    assert seen > 50


def test_resource_monotonicity():
    """a block that passes at m passes at every m' > m with the
    (smaller) WCETs resolved at m' -- follows from P:445."""
    rng = np.random.default_rng(6)
    for _ in range(300):
        n = int(rng.integers(1, 5))
        T = [int(rng.choice([20, 40, 50, 100])) for _ in range(n)]
        D = [int(rng.integers(t // 2, t + 1)) for t in T]
        B = [int(rng.integers(1, 30)) for _ in range(n)]
        c = [int(rng.integers(1, 6)) for _ in range(n)]
        f = [int(rng.integers(0, 4)) for _ in range(n)]
        verdicts = []
        for m in range(1, 16):
            Cm = [oracle.wcet(B[i], c[i], f[i], m) for i in range(n)]
            verdicts.append(oracle.edf_pdc(Cm, D, T)[0])
        first = verdicts.index(True) if True in verdicts else len(verdicts)
        assert all(verdicts[first:])


def test_empty_block_schedulable():
    assert oracle.edf_pdc([], [], [])[0]
