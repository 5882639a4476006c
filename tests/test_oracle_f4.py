"""Pins of the oracle's f4 variants: the binary-search merge
(P:704-706), the increasing-utilisation par_list and admissible
partition sizes (MIG-style slices).

Hand-traced examples in the integer W form with T = D (implicit deadlines, so
a partition is schedulable iff its utilisation is <= 1, Liu & Layland), the
special case "only size M is admissible" that reduces every heuristic to the
1G test, the binary/linear equivalence that resource monotonicity implies,
and solution certificates under random masks.
"""
import numpy as np
import pytest

import gp_workloads as W
import oracle

HEUR = ("SMS_ACT", "SMS_INA", "BF_ACT", "BF_INA")
BIN, INC = oracle.AL_BINARY_MERGE, oracle.AL_INCREASING


def make_sets(M, tasks):
    n = len(tasks)
    d = {k: np.array([[t[k] for t in tasks]], np.int32) for k in ("T", "D", "B", "cn", "cc", "fn", "fc")}
    d["type"] = np.array([[t["type"] for t in tasks]], np.uint8)
    d.update(M=M, n_groups=1, valid=np.ones(1, np.uint8), group=np.zeros(1, np.int32))
    return oracle.Sets.from_dict(d)


def task(c, T, typ, B=1, f=0):
    return dict(T=T, D=T, B=B, cn=c, cc=c, fn=f, fc=f, type=typ)


# ---------------------------------------------------------------- increasing order
# Three compute tasks, B = 1 (W = c for every m), T = D = 10, M = 2: each alone
# needs 1 SM (Lemma 2), Pi = 3 > 2, so exactly one merge at m = 1 (Def. 3:
# m < 1 + 1).  U*H = c (H = 10): 6, 4, 3.  A pair is schedulable iff c_i + c_j
# <= 10: all three pairs are (10, 9, 7), so ACT forbids nothing.
ORDER = [task(6, 10, 0), task(4, 10, 0), task(3, 10, 0)]


@pytest.mark.parametrize("v,flags,labels,tests", [
    # decreasing (A-17): P = t0; SMS picks the smaller merged U: {0,2} (9 < 10)
    ("SMS_INA", 0, [0, 1, 0], 2), ("SMS_ACT", 0, [0, 1, 0], 5),
    # decreasing, BF: partners by U desc -> t1 first, {0,1} succeeds
    ("BF_INA", 0, [0, 0, 1], 1), ("BF_ACT", 0, [0, 0, 1], 4),
    # increasing: P = t2; SMS picks {1,2} (7 < 9)
    ("SMS_INA", INC, [0, 1, 1], 2), ("SMS_ACT", INC, [0, 1, 1], 5),
    # increasing, BF: partners still by U desc (best fit, A-21) -> t0 first, {0,2}
    ("BF_INA", INC, [0, 1, 0], 1), ("BF_ACT", INC, [0, 1, 0], 4),
])
def test_increasing_order_hand_trace(v, flags, labels, tests):
    r = oracle.allocate(make_sets(2, ORDER), v, flags=flags)
    assert r["ok"][0] == 1 and r["k"][0] == 2 and r["pi"][0] == 2
    assert list(r["block_of_task"][0]) == labels
    assert list(r["block_size"][0][:2]) == [1, 1]
    assert r["n_tests"][0] == tests  # ACT adds the 3 pair tests of the prefill


# ---------------------------------------------------------------- binary merge
# t0 (memory) B=310, t1 (compute) B=610, c = 1, T = D = H = 100, M = 10:
# alone ceil(310/m) <= 100 iff m >= 4, ceil(610/m) <= 100 iff m >= 7, Pi = 11.
# merged (no conflict: different types): ceil(310/m) + ceil(610/m) <= 100
#   m = 9: 35 + 68 = 103 (no);  m = 10: 31 + 61 = 92 (yes).
# Candidate sizes L = [7, 8, 9, 10].  Linear: 4 tests.  Binary: mid = 2 (9) no ->
# lo = 3; mid = 3 (10) yes -> hi = 3; 2 tests.  Lemma 1: (310 + 610)/100 <= 10.
PAIR = [task(1, 100, 1, B=310), task(1, 100, 0, B=610)]


@pytest.mark.parametrize("v,flags,tests", [
    ("SMS_INA", 0, 4), ("SMS_INA", BIN, 2), ("BF_INA", 0, 4), ("BF_INA", BIN, 2),
    ("SMS_ACT", 0, 8), ("SMS_ACT", BIN, 4), ("BF_ACT", 0, 8), ("BF_ACT", BIN, 4),
])
def test_binary_merge_hand_trace(v, flags, tests):
    r = oracle.allocate(make_sets(10, PAIR), v, flags=flags)
    assert r["ok"][0] == 1 and r["k"][0] == 1 and r["pi"][0] == 10
    assert list(r["block_size"][0][:1]) == [10]
    assert r["n_tests"][0] == tests


@pytest.mark.parametrize("flags,tests", [(0, 2), (BIN, 2)])
def test_admissible_sizes_hand_trace(flags, tests):
    """Sizes {2, 4, 8, 10}: t0 -> 4 (min admissible >= 4), t1 -> 8; Pi = 12 > 10;
    merge candidates: admissible sizes in [8, 11] within 1..M = [8, 10];
    m = 8: 39 + 77 = 116 (no), m = 10 (yes).  Binary: mid = 1 (10) yes, mid = 0
    (8) no -> 10, also 2 tests."""
    s = make_sets(10, PAIR)
    r = oracle.allocate(s, "SMS_INA", flags=flags, sizes=[2, 4, 8, 10])
    assert r["ok"][0] == 1 and list(r["block_size"][0][:1]) == [10]
    assert r["n_tests"][0] == tests
    # without the merge (M = 12): the Lemma 2 sizes are the admissible ones
    s12 = make_sets(12, PAIR)
    r = oracle.allocate(s12, "BF_INA", sizes=[2, 4, 8, 10])
    assert r["ok"][0] == 1 and list(r["block_size"][0][:2]) == [4, 8] and r["n_tests"][0] == 0
    # 1G with a mask: the largest admissible size (10), schedulable (92 <= 100)
    r = oracle.allocate(s12, "1G", sizes=[2, 4, 8, 10])
    assert r["ok"][0] == 1 and list(r["block_size"][0][:1]) == [10]
    # only {2}: nothing fits alone -> Lemma 2 rejects
    r = oracle.allocate(s, "SMS_ACT", sizes=[2])
    assert r["ok"][0] == 0 and r["k"][0] == 0


def test_empty_mask_is_an_error():
    with pytest.raises(oracle.OracleError):
        oracle.allocate(make_sets(10, PAIR), "SMS_INA", sizes=[])


# ---------------------------------------------------------------- properties
@pytest.fixture(scope="module")
def c4_small():
    return oracle.generate(W.WORKLOADS["c4"]["gen"](R=20000), W.SEED, 0, 2)


@pytest.fixture(scope="module")
def c5_small():
    return oracle.generate(W.WORKLOADS["c5"]["gen"](R=10000), W.SEED, 0, 4)


@pytest.mark.parametrize("v", HEUR)
def test_binary_equals_linear_except_tests(c4_small, c5_small, v):
    """Resource monotonicity (W_i non-increasing in m) makes the minimal
    schedulable m unique, so the binary search finds the linear scan's m and
    every verdict and partition is identical; it never needs more tests."""
    for s in (c4_small, c5_small):
        for flags in (0, INC):
            a = oracle.allocate(s, v, flags=flags)
            b = oracle.allocate(s, v, flags=flags | BIN)
            for key in ("ok", "block_of_task", "block_size", "pi", "k"):
                assert (a[key] == b[key]).all(), key
            assert (b["n_tests"] <= a["n_tests"]).all()
            assert b["n_tests"].sum() < a["n_tests"].sum()


@pytest.mark.parametrize("v", HEUR)
def test_only_size_M_reduces_to_1G(c4_small, c5_small, v):
    """With M the only admissible size every partition has M SMs, merges can
    only produce M (Def. 3: M <= m < 2M), and a subset of a partition
    schedulable at M is schedulable at M (fewer conflicts, never larger
    WCETs; the demand test is monotone), so the greedy succeeds iff all tasks
    fit one partition of M SMs: the heuristic's verdict is the 1G verdict
     -- except for sets Lemma 1 rejects first (a necessary test)."""
    for s in (c4_small, c5_small):
        g = oracle.allocate(s, "1G")
        r = oracle.allocate(s, v, sizes=[s.M])
        assert (r["ok"] <= g["ok"]).all()
        lemma1 = r["k"] == 0
        assert (r["ok"][~lemma1] == g["ok"][~lemma1]).all()
        assert g["ok"][~lemma1].sum() > 0 and (~g["ok"].astype(bool)).sum() > 0
        ok = r["ok"].astype(bool)
        assert (r["k"][ok] == 1).all() and (r["pi"][ok] == s.M).all()


@pytest.mark.parametrize("v", HEUR)
@pytest.mark.parametrize("flags", [0, INC, BIN | INC])
def test_certificates_with_masks(c4_small, v, flags):
    """Every reported size is admissible, Pi <= M on success, every partition
    passes the (separately pinned) EDF demand test at its size, and tasks are
    conserved; the verdict never beats the unmasked run by more than the
    admissible sizes allow -- checked here only as validity."""
    s = c4_small
    rng = np.random.default_rng(7)
    sizes = sorted(set([s.M] + [int(x) for x in rng.choice(np.arange(1, s.M), 20, replace=False)]))
    r = oracle.allocate(s, v, flags=flags, sizes=sizes)
    n = s.n_tasks
    assert r["ok"].sum() > 0
    for g in range(s.n_sets):
        if r["k"][g] == 0:
            continue
        k = int(r["k"][g])
        bot = [int(x) for x in r["block_of_task"][g]]
        assert sorted(set(bot)) == list(range(k))
        szs = [int(x) for x in r["block_size"][g][:k]]
        assert all(z in sizes for z in szs)
        if not r["ok"][g]:
            continue
        assert sum(szs) == r["pi"][g] <= s.M
        types = [int(x) for x in s.type[g]]
        for j in range(k):
            mem = [i for i in range(n) if bot[i] == j]
            C = []
            for i in mem:
                conflict = any(types[o] == types[i] for o in mem if o != i)
                c, f = (s.cc[g, i], s.fc[g, i]) if conflict else (s.cn[g, i], s.fn[g, i])
                C.append(oracle.wcet(int(s.B[g, i]), int(c), int(f), szs[j]))
            assert oracle.edf_pdc(C, [int(s.D[g, i]) for i in mem], [int(s.T[g, i]) for i in mem])[0]


# ---------------------------------------------------------------- masks on the exhaustive path
# Reading B-9: with admissible sizes A a candidate (pi, s)
# is deployable only if every s_j is in A; an inadmissible one counts as
# unschedulable, and the rank space (C.1.6) is unchanged.  Pinned by
# composition with separately pinned pieces: the unmasked verdict bits
# (test_oracle_exhaustive.py) and the enumeration (test_oracle_enum.py).
MASK64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def c2_masked_sample():
    gen = W.WORKLOADS["c2"]["gen"](R=10000)
    s = oracle.generate(gen, W.SEED, 0, 3)  # 3 reps x 10 bins
    per, bits = oracle.exhaustive(s, bits=True)
    bot, bs = oracle.enumerate_candidates(s.M, s.n_tasks)
    return s, per, bits, bs


@pytest.mark.parametrize("sizes", [[1, 2, 4, 8], [3, 5, 6], [2, 4, 6, 8], [7]])
def test_exhaustive_mask_is_unmasked_bits_filtered(c2_masked_sample, sizes):
    s, per, bits, bs = c2_masked_sample
    per_m, bits_m = oracle.exhaustive(s, bits=True, sizes=sizes)
    adm = np.zeros(s.M + 1, bool)
    adm[sizes] = True
    deploy = np.all(adm[bs.astype(np.int64)] | (bs == 0), axis=1)  # every used size admissible
    n_c = len(bs)
    for g in range(s.n_sets):
        v = np.array([(int(bits[g, r // 32]) >> (r % 32)) & 1 for r in range(n_c)], bool)
        ranks = np.nonzero(v & deploy)[0]
        vm = np.array([(int(bits_m[g, r // 32]) >> (r % 32)) & 1 for r in range(n_c)], bool)
        assert (vm == (v & deploy)).all()
        assert per_m[g, 0] == len(ranks)
        assert per_m[g, 2] == (ranks[0] if len(ranks) else -1)
        assert per_m[g, 1] == (int(bs[ranks].sum(axis=1).min()) if len(ranks) else 0)
        h = sum(oracle.splitmix64(int(r)) for r in ranks) & MASK64
        assert int(np.int64(per_m[g, 3]).view(np.uint64)) == h
    assert per_m[:, 0].sum() < per[:, 0].sum()


def test_exhaustive_mask_every_size_is_unmasked(c2_masked_sample):
    s, per, _, _ = c2_masked_sample
    assert (oracle.exhaustive(s, sizes=list(range(1, s.M + 1))) == per).all()


def test_exhaustive_only_M_is_1G(c2_masked_sample):
    """Only size M admissible: the one deployable candidate is all tasks in one
    partition of M SMs (rank N(M,n) of k = 1 is s = M, rank M - 1), so the set is
    schedulable iff 1G schedules it, at pi* = M."""
    s, _, _, _ = c2_masked_sample
    per = oracle.exhaustive(s, sizes=[s.M])
    g1 = oracle.allocate(s, "1G")["ok"]
    assert (per[:, 0] == g1).all()
    assert (per[g1 == 1, 1] == s.M).all() and (per[g1 == 1, 2] == s.M - 1).all()
    assert 0 < g1.sum() < s.n_sets
