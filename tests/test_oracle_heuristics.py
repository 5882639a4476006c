"""Pins of the oracle's heuristics (A5: Alg. 1-3, Lemmas 1-3, Defs 3-5, 1G).

SPEC's partitioner examples transcribed to the integer W form with
B = 1 (so W(m) = c + f for every m), hand-traced n_tests, the C1 worked
example, and certificate properties (Lemma 3, task conservation, Def. 3).
Tie-breaking beyond these is "parity unpinned" against the paper.
"""
import numpy as np
import pytest

import gp_workloads as W
import oracle

VARIANTS = ("SMS_ACT", "SMS_INA", "BF_ACT", "BF_INA")


def make_sets(M, tasks, n_copies=1):
    """tasks: list of dicts with T, D, B, cn, cc, fn, fc, type."""
    n = len(tasks)
    d = {k: np.array([[t[k] for t in tasks]] * n_copies, np.int32)
         for k in ("T", "D", "B", "cn", "cc", "fn", "fc")}
    d["type"] = np.array([[t["type"] for t in tasks]] * n_copies, np.uint8)
    d.update(M=M, n_groups=1, valid=np.ones(n_copies, np.uint8), group=np.zeros(n_copies, np.int32))
    return oracle.Sets.from_dict(d)


def task(c, f, T, D, typ, B=1, cc=None, fc=None):
    return dict(T=T, D=D, B=B, cn=c, fn=f, cc=cc if cc is not None else c,
                fc=fc if fc is not None else f, type=typ)


# SPEC try_merge example S:254 (ticks x10): compute a=100,b=2 + memory a=100,b=10
MERGEABLE = [task(100, 2, 1000, 750, 0), task(100, 10, 1000, 750, 1)]
# a=400 pair, demand 848 > 750
UNMERGEABLE = [task(400, 8, 1000, 750, 0), task(400, 40, 1000, 750, 1)]


@pytest.mark.parametrize("v,tests", [("SMS_INA", 1), ("BF_INA", 1), ("SMS_ACT", 2), ("BF_ACT", 2)])
def test_spec_partition_and_allocate_mergeable(v, tests):
    """M=1, the mergeable pair -> success, one partition of size 1.
    n_tests: INA = 1 (one merge test); ACT = 1 prefill test + 1."""
    r = oracle.allocate(make_sets(1, MERGEABLE), v)
    assert r["ok"][0] == 1 and r["k"][0] == 1 and r["pi"][0] == 1
    assert list(r["block_of_task"][0]) == [0, 0] and r["block_size"][0][0] == 1
    assert r["n_tests"][0] == tests


@pytest.mark.parametrize("v", VARIANTS)
def test_spec_partition_and_allocate_unmergeable(v):
    """M=1, the unmergeable pair -> fail after exactly one EDF test
    (demand 848 > 750 at the only deadline); Def. 3 forbids m=2."""
    r = oracle.allocate(make_sets(1, UNMERGEABLE), v)
    assert r["ok"][0] == 0 and r["n_tests"][0] == 1
    assert r["k"][0] == 2 and r["pi"][0] == 2


@pytest.mark.parametrize("v", VARIANTS)
def test_spec_no_merge_needed(v):
    """M=2, two tasks of different types needing 1 SM each -> success
    without any merge (Lemma 3), and no ACT prefill (reading A-24)."""
    r = oracle.allocate(make_sets(2, UNMERGEABLE), v)
    assert r["ok"][0] == 1 and r["k"][0] == 2 and r["pi"][0] == 2 and r["n_tests"][0] == 0


def test_lemma1_reject():
    """S:139 (Lemma 1): two tasks with C^n(1)=50, T=10 on M=8: 10 > 8."""
    s = make_sets(8, [task(50, 0, 10, 10, 0), task(50, 0, 10, 10, 1)])
    for v in VARIANTS:
        r = oracle.allocate(s, v)
        assert r["ok"][0] == 0 and r["k"][0] == 0 and r["n_tests"][0] == 0


def test_lemma1_boundary_equality_passes():
    """sum = M exactly is not rejected (strict >, reading A-16)."""
    s = make_sets(1, [task(10, 0, 10, 10, 0)])
    r = oracle.allocate(s, "SMS_INA")
    assert r["ok"][0] == 1 and r["pi"][0] == 1


@pytest.mark.parametrize("M,size", [(68, 4), (4, 4), (3, None)])
def test_lemma2_min_sms(M, size):
    """S:159 (Lemma 2): a=100, b=2, D=27 -> 4 SMs (100/4 + 2 = 27);
    with M=3 there is no feasible size -> fail before merging."""
    s = make_sets(M, [task(1, 2, 1000, 27, 0, B=100)])
    r = oracle.allocate(s, "BF_INA")
    if size is None:
        assert r["ok"][0] == 0 and r["k"][0] == 0
    else:
        assert r["ok"][0] == 1 and r["pi"][0] == size and r["block_size"][0][0] == size


def test_one_g_examples():
    """one task fitting at m=M succeeds; 2 memory + 2 compute with
    infeasible conflict WCETs at m=M fails; 1G always runs exactly one test."""
    r = oracle.allocate(make_sets(4, [task(1, 2, 1000, 27, 0, B=100)]), "1G")
    assert r["ok"][0] == 1 and r["pi"][0] == 4 and r["k"][0] == 1 and r["n_tests"][0] == 1
    four = [task(10, 0, 100, 75, t, cc=40, fc=0) for t in (0, 0, 1, 1)]
    r = oracle.allocate(make_sets(1, four), "1G")
    assert r["ok"][0] == 0 and r["n_tests"][0] == 1
    # without conflicts (one task of each type per partition) the heuristic succeeds
    r = oracle.allocate(make_sets(2, four), "SMS_INA")
    assert r["ok"][0] == 1 and r["k"][0] == 2


def test_c1_heuristics():
    """C1: Lemma 1 passes (15 <= 80), all m_i = 1 (5 <= 7),
    Pi = 3 <= 4: success with 3 singleton partitions and 0 tests; 1G fails
    (3 * ceil(5/4) * 2 = 12 > 7 for CCC) after one test."""
    s = oracle.Sets.from_dict(W._c1_sets())
    for v in VARIANTS:
        r = oracle.allocate(s, v)
        assert (r["ok"] == 1).all() and (r["k"] == 3).all() and (r["pi"] == 3).all()
        assert (r["n_tests"] == 0).all()
        assert (r["block_of_task"] == [0, 1, 2]).all()
    r = oracle.allocate(s, "1G")
    assert (r["ok"] == 0).all() and (r["n_tests"] == 1).all()


def test_sms_prefers_smallest_merge():
    """Def. 4: among valid merges with the head partition P, >> keeps
    the one with the smallest merged size.  P = task 0 (largest U); partner 1
    needs 2 SMs merged, partner 2 merges at 1 SM -> SMS merges {0,2}."""
    # B=2 so W(1) = 2c + f, W(2) = c + f.
    t0 = task(30, 0, 100, 75, 0, B=2)          # alone m=1: 60 <= 75
    t1 = task(30, 0, 100, 75, 0, B=2)          # same type as t0 -> conflict when merged
    t2 = task(5, 0, 100, 75, 1, B=2)           # other type, small
    for t in (t0, t1):
        t["cc"], t["fc"] = 40, 0
    s = make_sets(2, [t0, t1, t2])
    r = oracle.allocate(s, "SMS_INA")
    assert r["ok"][0] == 1
    assert list(r["block_of_task"][0]) == [0, 1, 0] and r["pi"][0] == 2


@pytest.fixture(scope="module")
def c4_small():
    gen = W.WORKLOADS["c4"]["gen"](R=20000)
    return oracle.generate(gen, W.SEED, 0, 2)  # 2 reps x 50 groups = 100 sets


@pytest.mark.parametrize("v", ("1G",) + VARIANTS)
def test_certificates_on_generated_sets(c4_small, v):
    """Lemma 3 certificate, task conservation, 1G Pi = M,
    determinism under any thread count, Lemma 1 soundness."""
    s = c4_small
    r = oracle.allocate(s, v, threads=1)
    r8 = oracle.allocate(s, v, threads=8)
    for key in r:
        assert (r[key] == r8[key]).all()
    n = s.n_tasks
    for g in range(s.n_sets):
        if not r["ok"][g]:
            continue
        bot = [int(x) for x in r["block_of_task"][g]]
        k = int(r["k"][g])
        assert sorted(set(bot)) == list(range(k))
        assert all(bot.index(j) < bot.index(j + 1) for j in range(k - 1))  # canonical
        sizes = [int(x) for x in r["block_size"][g][:k]]
        assert sum(sizes) == r["pi"][g] <= s.M
        if v == "1G":
            assert k == 1 and sizes == [s.M]
        types = [int(x) for x in s.type[g]]
        for j in range(k):
            mem = [i for i in range(n) if bot[i] == j]
            C = []
            for i in mem:
                conflict = any(types[o] == types[i] for o in mem if o != i)
                c, f = (s.cc[g, i], s.fc[g, i]) if conflict else (s.cn[g, i], s.fn[g, i])
                C.append(oracle.wcet(int(s.B[g, i]), int(c), int(f), sizes[j]))
            assert oracle.edf_pdc(C, [int(s.D[g, i]) for i in mem], [int(s.T[g, i]) for i in mem])[0]
        if v != "1G":
            H = oracle.hyperperiod([int(x) for x in s.T[g]])
            lhs = sum(oracle.wcet(int(s.B[g, i]), int(s.cn[g, i]), int(s.fn[g, i]), 1)
                      * (H // int(s.T[g, i])) for i in range(n))
            assert lhs <= s.M * H


def test_heuristics_find_solutions_on_c4(c4_small):
    """Sanity: at low utilisation bins the heuristics schedule most sets and
    succeed at least as often as 1G overall (qualitative)."""
    s = c4_small
    one_g = oracle.allocate(s, "1G")["ok"].mean()
    for v in VARIANTS:
        assert oracle.allocate(s, v)["ok"].mean() >= one_g


# ---------------------------------------------------------------- f2 efficiency
def _eff_sets(types, cn=10, cc=23, B=2, T=100):
    n = len(types)
    return make_sets(8, [dict(T=T, D=T, B=B, cn=cn, cc=cc, fn=0, fc=0, type=t) for t in types])


def test_efficiency_spec_examples():
    """SPEC S:420-422 in the work form (work = c * B per period):
    one memory + one compute per partition -> achieved = lower;
    one partition holding >= 2 of each type (1G) -> achieved = upper;
    one conflicting memory task among conflict-free ones -> lower + its (cc-cn)B."""
    s = _eff_sets([0, 1, 0, 1])
    e = oracle.efficiency(s, np.array([[0, 0, 1, 1]], np.int8))[0]
    assert e[3] == 100 and e[0] == 4 * 10 * 2 and e[1] == 4 * 23 * 2
    assert e[2] == e[0]
    e = oracle.efficiency(s, np.array([[0, 0, 0, 0]], np.int8))[0]
    assert e[2] == e[1]
    # tasks 1 and 3 (memory) share partition 1 with nobody else of their type? no:
    # labels [0, 1, 2, 1]: tasks 1,3 memory together -> both conflict; 0 and 2 alone
    e = oracle.efficiency(s, np.array([[0, 1, 2, 1]], np.int8))[0]
    assert e[2] == 2 * 10 * 2 + 2 * 23 * 2
    # rejected (no allocation): achieved 0, bounds still reported
    e = oracle.efficiency(s, np.array([[-1, -1, -1, -1]], np.int8))[0]
    assert e[2] == 0 and e[0] == 80


def test_efficiency_bounds_on_heuristic_solutions(c4_small):
    s = c4_small
    for v in ("1G",) + VARIANTS:
        r = oracle.allocate(s, v)
        e = oracle.efficiency(s, r["block_of_task"])
        assert (e[:, 0] <= e[:, 1]).all()
        has = r["k"] > 0
        assert ((e[has, 0] <= e[has, 2]) & (e[has, 2] <= e[has, 1])).all()
        assert (e[~has, 2] == 0).all()
        if v == "1G":  # 1G always schedules the worst load
            mixed = [(s.type[g].sum() >= 2) and ((1 - s.type[g]).sum() >= 2) for g in range(s.n_sets)]
            assert all(e[g, 2] == e[g, 1] for g in range(s.n_sets) if mixed[g])
