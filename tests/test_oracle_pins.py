"""Pins of the oracle functions round 1 left unpinned.

* ``gpref_wcet_batch`` (A3 on candidates): hand-computed WCETs / conflict flags for
  labelled candidates, including a NON-canonical label order (the size of task i's
  block is block_size[label], not block_size[rank of the label]) and set indexing.
* Curve-mode ``gpref_task_fields`` (f1, reading A-1 / B-8): hand values of
  B = ceil(a/g), cn = g, cc = ceil(k g), fn = ceil(beta a), fc = ceil(k fn), and the
  W form's distance to the paper's rational curve k(a/|P| + b) for every m.
* Algorithm 1's forbidden-list semantics: a 4-task hand trace
  where INA builds a partition holding a task pair that ACT's prefill forbade
  (through a merge of a larger partition) and ACT therefore fails; SPEC's
  select_partitions and fill_forbidden_list examples.

Every expected value below is written out by hand in the test (derivation in
the docstring); none is computed by re-typing the oracle's formula.
"""
from fractions import Fraction

import numpy as np
import pytest

import gp_workloads as W
import oracle
from test_oracle_heuristics import MERGEABLE, UNMERGEABLE, make_sets, task


# ---------------------------------------------------------------- wcet_batch
def _wb_sets():
    """Two sets of 4 tasks (T = D = 100; only B, c, f and types matter here).
    set 0 types C M C M; set 1 identical except task 1 is compute (C C C M)."""
    base = [dict(B=5, cn=2, cc=3, fn=1, fc=4), dict(B=7, cn=1, cc=5, fn=0, fc=2),
            dict(B=4, cn=3, cc=6, fn=2, fc=3), dict(B=9, cn=2, cc=4, fn=1, fc=1)]
    rows = []
    for types in ((0, 1, 0, 1), (0, 0, 0, 1)):
        rows.append([dict(T=100, D=100, type=t, **b) for b, t in zip(base, types)])
    d = {k: np.array([[t[k] for t in r] for r in rows], np.int32)
         for k in ("T", "D", "B", "cn", "cc", "fn", "fc")}
    d["type"] = np.array([[t["type"] for t in r] for r in rows], np.uint8)
    d.update(M=8, n_groups=1, valid=np.ones(2, np.uint8), group=np.zeros(2, np.int32))
    return oracle.Sets.from_dict(d)


def test_wcet_batch_hand_values():
    """C.1.3 / C.1.5 on four candidates.
    A (set 0), labels [2,0,2,1], sizes by label [3,4,2]:
      tau0 label 2 (size 2) with tau2 (same type) -> conflict: ceil(5/2)*3+4 = 13
      tau1 label 0 (size 3) alone                 -> ceil(7/3)*1+0 = 3
      tau2 label 2 (size 2) conflict              -> ceil(4/2)*6+3 = 15
      tau3 label 1 (size 4) alone                 -> ceil(9/4)*2+1 = 7
    B (set 0), labels [1,1,0,0], sizes [5,1]: {0,1} at 1 (C+M, no conflict): 5*2+1 = 11,
      7*1+0 = 7; {2,3} at 5 (C+M): ceil(4/5)*3+2 = 5, ceil(9/5)*2+1 = 5.
    C (set 0), one block of 8 (C,M,C,M: everyone has a same-type partner):
      ceil(5/8)*3+4 = 7, 1*5+2 = 7, 1*6+3 = 9, ceil(9/8)*4+1 = 9.
    D (set 1 -- tau1 compute), labels [1,1,0,0], sizes [5,1]: {0,1} both compute ->
      conflict: 5*3+4 = 19, 7*5+2 = 37; {2,3} (C+M) as in B: 5, 5."""
    s = _wb_sets()
    soc = [0, 0, 0, 1]
    bot = [[2, 0, 2, 1], [1, 1, 0, 0], [0, 0, 0, 0], [1, 1, 0, 0]]
    bs = [[3, 4, 2, 0], [5, 1, 0, 0], [8, 0, 0, 0], [5, 1, 0, 0]]
    w, cf = oracle.wcet_batch(s, soc, bot, bs)
    assert w.tolist() == [[13, 3, 15, 7], [11, 7, 5, 5], [7, 7, 9, 9], [19, 37, 5, 5]]
    assert cf.tolist() == [[1, 0, 1, 0], [0, 0, 0, 0], [1, 1, 1, 1], [1, 1, 0, 0]]


@pytest.mark.parametrize("soc,bot,bs", [
    ([0], [[0, 0, 1, 1]], [[3, 0, 0, 0]]),    # label 1 used, its size 0 (m = 0)
    ([0], [[0, 4, 0, 0]], [[3, 3, 3, 3]]),    # label 4 >= n (task outside)
    ([0], [[0, -1, 0, 0]], [[3, 3, 3, 3]]),   # negative label
    ([2], [[0, 0, 0, 0]], [[3, 0, 0, 0]]),    # set index out of range
])
def test_wcet_batch_rejects_malformed(soc, bot, bs):
    with pytest.raises(oracle.OracleError):
        oracle.wcet_batch(_wb_sets(), soc, bot, bs)


# --------------------------------------------------------- curve-mode fields
def _curve_gen():
    return W.gen_params(68, 50, 1, n_bins=34, curve_gran=10)


@pytest.mark.parametrize("typ,fn,cc,fc", [(0, 1000, 12, 1200), (1, 5000, 23, 11500)])
def test_curve_fields_round_numbers(typ, fn, cc, fc):
    """u = 1/2 (2^19 in Q20), T = 100 units (menu[1]) = 100,000 ticks:
    a = T u = 50,000 >= Q (no bump), D = 75,000, B = 50,000/10 = 5,000 granules,
    cn = g = 10; compute: fn = 0.02 a = 1,000, cc = 1.2*10 = 12, fc = 1.2*1,000 = 1,200;
    memory: fn = 0.1 a = 5,000, cc = 2.3*10 = 23, fc = 2.3*5,000 = 11,500."""
    f = oracle.task_fields(_curve_gen(), 1 << 19, 1, 1, typ)
    assert (f["T"], f["D"], f["a"], f["B"], f["cn"]) == (100_000, 75_000, 50_000, 5_000, 10)
    assert (f["fn"], f["cc"], f["fc"]) == (fn, cc, fc)
    assert f["feasible"] == 1  # W(68) = ceil(5000/68)*10 + fn = 740 + fn <= 75,000


@pytest.mark.parametrize("typ,fn,fc", [(0, 247, 297), (1, 1235, 2841)])
def test_curve_fields_rounding(typ, fn, fc):
    """a = 12,345 ticks (u = 129,447 / 2^20, T = 100,000: floor(12,944,700,000 / 2^20)
    = 12,345): B = ceil(12,345/10) = 1,235 (floor would give 1,234);
    compute fn = ceil(246.9) = 247, fc = ceil(1.2*247 = 296.4) = 297;
    memory fn = ceil(1,234.5) = 1,235, fc = ceil(2.3*1,235 = 2,840.5) = 2,841."""
    f = oracle.task_fields(_curve_gen(), 129_447, 1, 1, typ)
    assert f["a"] == 12_345 and f["B"] == 1_235 and f["cn"] == 10
    assert f["fn"] == fn and f["fc"] == fc


def test_curve_period_bump():
    """Reading A-10 in curve mode (bump while a < Q): u = 2^10 / 2^20 from
    T = 50 units: a = 48, 97, 195, 390, 488, 976 ticks at 50..1000 units, then
    1,953 >= 1,000 at 2,000 units -> T = 2,000,000 ticks, D = 1,500,000, B = 196."""
    f = oracle.task_fields(_curve_gen(), 1 << 10, 0, 1, 0)
    assert f["T"] == 2_000_000 and f["D"] == 1_500_000 and f["a"] == 1_953
    assert f["B"] == 196


def test_curve_w_form_is_within_granule_of_paper_curve():
    """Reading B-8: the W form W^x(m) = ceil(B/m) c^x + f^x of curve
    mode is never below the paper's curve C^x(m) = k^x (a/m + b), b = beta a
    (k = 1 without conflict), and exceeds it by less than k (g + 1) + 1
    ticks, for every m = 1..68 and many a (exact rationals)."""
    gen = _curve_gen()
    rng = np.random.default_rng(7)
    g = 10
    for typ, beta, k in ((0, Fraction(2, 100), Fraction(12, 10)),
                         (1, Fraction(10, 100), Fraction(23, 10))):
        for u in rng.integers(1 << 8, 1 << 21, size=60):
            f = oracle.task_fields(gen, int(u), int(rng.integers(0, 8)), 1, typ)
            a, B = f["a"], f["B"]
            for m in range(1, 69):
                for kx, c, fl in ((Fraction(1), f["cn"], f["fn"]), (k, f["cc"], f["fc"])):
                    w = oracle.wcet(B, c, fl, m)
                    curve = kx * (Fraction(a, m) + beta * a)
                    assert 0 <= w - curve < kx * (g + 1) + 1, (typ, a, m, w, curve)


# ------------------------------------------------ forbidden lists, ACT vs INA
# T = D = 100 for all tasks and f = 0, so a partition is schedulable at m iff
# sum_i W_i(m) <= 100 (one deadline, t = 100).  B = 3 for all: W(1) = 3c, W(2) = 2c,
# W(m >= 3) = c.   (B, cn, cc, type):
P975 = [task(40, 0, 100, 100, 0, B=3, cc=40), task(40, 0, 100, 100, 1, B=3, cc=80),
        task(20, 0, 100, 100, 0, B=3, cc=60), task(5, 0, 100, 100, 0, B=3, cc=15)]


def test_act_prefill_hand_trace():
    """fill_forbidden_list on P975.  Lemma 2 sizes: tau0 3*40 = 120 > 100,
    2*40 = 80 -> 2; tau1 -> 2; tau2 60 -> 1; tau3 15 -> 1.  Pairs in id order
    (Algorithm 2 tries m = max(|P1|,|P2|) .. |P1|+|P2|-1):
      (0,1) C+M no conflict: m=2 80+80 = 160 fail, m=3 40+40 = 80 ok   (2 tests)
      (0,2) C+C conflict, m=2 only: 2*40 + 2*60 = 200 fail             (1) forbidden
      (0,3) C+C, m=2: 80 + 2*15 = 110 fail                               (1) forbidden
      (1,2) M+C, m=2: 80 + 2*20 = 120 fail                               (1) forbidden
      (1,3) M+C, m=2: 80 + 2*5 = 90 ok                                   (1)
      (2,3) C+C, m=1 only: 3*60 + 3*15 = 225 fail                        (1) forbidden
    -> forbidden {(0,2),(0,3),(1,2),(2,3)}, 7 tests."""
    forb, nt = oracle.fill_forbidden_list(make_sets(4, P975))
    exp = np.zeros((4, 4), np.uint8)
    for i, j in ((0, 2), (0, 3), (1, 2), (2, 3)):
        exp[i, j] = exp[j, i] = 1
    assert (forb == exp).all() and nt == 7


@pytest.mark.parametrize("v,ok,bot,bs,tests", [
    # BF_INA: head {0} (U*H 80, id 0); elig by U*H: {1} 80, {2} 60, {3} 15.
    #  {0}+{1}: m=2 fail, m=3 ok (2 tests) -> {0,1}@3, Pi = 5.  head {0,1}; elig {2},{3}.
    #  {0,1}+{2} m=3: tau0,tau2 conflict: 40 + 40 + 60 = 140 fail (test 3, snapshot);
    #  {0,1}+{3} m=3: 40 + 40 + 15 = 95 ok (test 4) -> {0,1,3}@3, Pi = 4 <= M: success.
    #  {0,1,3} holds the pair (0,3) that fails as singletons: P:975's "partitions
    #  including forbidden pairs through valid merging of larger partitions".
    ("BF_INA", 1, [0, 0, 1, 0], [3, 1, 0, 0], 4),
    # SMS_INA: head {0} tries every partner: {1} 2 tests (ok @3), {2} 1 (fail), {3} 1
    #  (fail) -> commit {0,1}@3 (tests 4); head {0,1} (snapshots ({0},{2}), ({0},{3})
    #  do not match it): {2} fail (5), {3} ok @3 (6) -> {0,1,3}@3, success.
    ("SMS_INA", 1, [0, 0, 1, 0], [3, 1, 0, 0], 6),
    # ACT (both orders): prefill 7 tests; head {0}: forbidden partners {2},{3} -> elig
    #  {1}: 2 tests -> {0,1}@3 (9 tests), Pi = 5.  head {0,1}: {2} holds a task forbidden
    #  with 0 and 1, {3} one forbidden with 0 -> empty; head {2}: {0,1} (2-0), {3} (2-3)
    #  -> empty; head {3}: {0,1} (3-0), {2} -> empty: fail with {0,1}@3, {2}@1, {3}@1.
    ("BF_ACT", 0, [0, 0, 1, 2], [3, 1, 1, 0], 9),
    ("SMS_ACT", 0, [0, 0, 1, 2], [3, 1, 1, 0], 9),
])
def test_ina_builds_forbidden_pair_act_refuses(v, ok, bot, bs, tests):
    """P:975 (and P:785 vs Alg. 3 line 7, reading A-23), hand-traced on P975."""
    r = oracle.allocate(make_sets(4, P975), v)
    assert r["ok"][0] == ok and r["n_tests"][0] == tests
    assert r["block_of_task"][0].tolist() == bot and r["block_size"][0].tolist() == bs
    assert r["pi"][0] == sum(bs) and r["k"][0] == max(bot) + 1


def test_select_act_excludes_partner_through_task_pair_ina_only_snapshot():
    """Alg. 3 line 7 under the two readings (A-23): state par_list = {0,1}@3, {2}@1,
    {3}@1 (U*H 80, 60, 15).  ACT with forbidden task pair (0,3): P = {0,1} has elig
    {2} only, since {3} holds a task forbidden with task 0 of P.  INA with
    the snapshot ({0},{3}): the snapshot names the old singleton {0}, not {0,1},
    so {3} stays eligible: elig {2}, {3}."""
    s = make_sets(4, P975)
    parts = [([0, 1], 3), ([2], 1), ([3], 1)]
    forb = np.zeros((4, 4), np.uint8)
    forb[0, 3] = forb[3, 0] = 1
    assert oracle.select_partitions(s, parts, forb=forb) == ([0, 1], [[2]])
    assert oracle.select_partitions(s, parts, snapshots=[([0], [3])]) == ([0, 1], [[2], [3]])
    # an exact snapshot of (P, P') excludes P' in both modes
    assert oracle.select_partitions(s, parts, snapshots=[([0, 1], [2])]) == ([0, 1], [[3]])


def test_spec_select_partitions_examples():
    """SPEC S:284-286 (Algorithm 3).
    S:284: two mergeable singletons, empty forbidden list -> (first, [second]); the
      first in par_list order is tau1 (U*H = W = 110 > 102 of tau0, A-17).
    S:285: two partitions whose only tasks form a forbidden pair (ACT) -> none.
    S:286: three partitions A, B, C with (A, B) forbidden -> (A, [C]); A = tau0
      (U*H 300), B = tau1 (200), C = tau2 (100), INA snapshot and ACT pair alike."""
    s = make_sets(1, MERGEABLE)
    assert oracle.select_partitions(s, [([0], 1), ([1], 1)]) == ([1], [[0]])
    s = make_sets(1, UNMERGEABLE)
    forb, _ = oracle.fill_forbidden_list(s)
    assert oracle.select_partitions(s, [([0], 1), ([1], 1)], forb=forb) == (None, [])
    three = make_sets(3, [task(300, 0, 1000, 1000, 0), task(200, 0, 1000, 1000, 1),
                          task(100, 0, 1000, 1000, 0)])
    parts = [([0], 1), ([1], 1), ([2], 1)]
    assert oracle.select_partitions(three, parts, snapshots=[([0], [1])]) == ([0], [[2]])
    f = np.zeros((3, 3), np.uint8)
    f[0, 1] = f[1, 0] = 1
    assert oracle.select_partitions(three, parts, forb=f) == ([0], [[2]])
    # BF sorts elig by partner U*H descending (A-21): P = tau0, elig tau1 (200), tau2 (100)
    assert oracle.select_partitions(three, parts, best_fit=True) == ([0], [[1], [2]])


def test_spec_fill_forbidden_list_examples():
    """SPEC S:294-296 (§5.3): the failing pair of try_merge example 2 is
    recorded (one test: demand 848 > 750 at m = 1, Def. 3 forbids m = 2); the
    succeeding pair of example 1 is not (one test, 212 <= 750); a singleton task set
    gives an empty list and no test."""
    forb, nt = oracle.fill_forbidden_list(make_sets(1, UNMERGEABLE))
    assert forb.tolist() == [[0, 1], [1, 0]] and nt == 1
    forb, nt = oracle.fill_forbidden_list(make_sets(1, MERGEABLE))
    assert forb.tolist() == [[0, 0], [0, 0]] and nt == 1
    forb, nt = oracle.fill_forbidden_list(make_sets(1, [MERGEABLE[0]]))
    assert forb.tolist() == [[0]] and nt == 0


# ------------------------------------------------------------ generator wiring
@pytest.mark.parametrize("key,group,rep", [("c3", 0, 0), ("c3", 7, 123), ("c4", 37, 5),
                                            ("c5", 9, 9999)])
def test_generate_wiring_from_c_1_10(key, group, rep):
    """gpref_generate's assembly, restated from SURVEY §8(c) C.1.10 with pinned parts
    only (Philox by its KAT vectors, uunisort by its invariants, task_fields by the
    §7.1 pins above): g = group * R + rep; counter (g lo, g hi, attempt, j), key =
    seed (lo, hi); w0 < prm_q -> memory; period index floor(w1 * n_periods / 2^32);
    B = 1 + floor(w2 * b_max / 2^32); point p_j = floor(w3 (U_q + 1) / 2^32) for
    j < n - 1; U_q = floor((bin + 1) M 2^20 / n_bins); the first attempt whose tasks
    are all feasible alone is kept."""
    gen = W.WORKLOADS[key]["gen"](R=10000)
    n, M, nb = gen["n_tasks"], gen["M"], gen["n_bins"]
    prm_idx, b = divmod(group, nb)
    g = group * gen["sets_per_group"] + rep
    Uq = ((b + 1) * M << 20) // nb
    key_w = [W.SEED & 0xFFFFFFFF, W.SEED >> 32]
    for attempt in range(gen["max_attempts"]):
        words = [oracle.philox4x32_10([g & 0xFFFFFFFF, g >> 32, attempt, j], key_w)
                 for j in range(n)]
        types = [int(w[0] < gen["prm_q"][prm_idx]) for w in words]
        pidx = [(w[1] * len(gen["period_menu"])) >> 32 for w in words]
        Bs = [1 + ((w[2] * gen["b_max"]) >> 32) for w in words]
        pts = [(w[3] * (Uq + 1)) >> 32 for w in words[:n - 1]]
        u = oracle.uunisort(n, Uq, pts)
        fields = [oracle.task_fields(gen, int(u[i]), pidx[i], Bs[i], types[i]) for i in range(n)]
        if all(f["feasible"] for f in fields):
            break
    s = oracle.generate(gen, W.SEED, rep, 1)
    row = group  # one repetition per group: local set index = group
    assert s.valid[row] == 1 and s.group[row] == group
    assert s.type[row].tolist() == types
    for name in ("T", "D", "B", "cn", "cc", "fn", "fc"):
        assert getattr(s, name)[row].tolist() == [f[name] for f in fields], name
