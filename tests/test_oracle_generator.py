"""Pins of the oracle's task-set generator (A1, §7.1, §8(c) C.1.10)."""
from fractions import Fraction

import numpy as np
import pytest
from scipy import stats

import gp_workloads as W
import oracle


def test_uunisort_sum_exact_and_nonnegative():
    rng = np.random.default_rng(8)
    for _ in range(500):
        n = int(rng.integers(1, 33))
        Uq = int(rng.integers(0, 1 << 30))
        pts = rng.integers(0, Uq + 1, size=max(n - 1, 0))
        u = oracle.uunisort(n, Uq, pts)
        assert int(u.sum()) == Uq and (u >= 0).all()
        assert sorted(np.cumsum(u)[:-1].tolist()) == sorted(pts.tolist())


def test_uunisort_has_uunifast_law():
    """UUniFast (Bini & Buttazzo) draws uniformly on the simplex; one
    coordinate of a uniform point on the n-simplex is U * Beta(1, n-1).  Sorted
    uniform spacings (reading A-12) must show that law (KS test)."""
    rng = np.random.default_rng(9)
    n, Uq = 5, 1 << 28
    first, last = [], []
    for _ in range(4000):
        u = oracle.uunisort(n, Uq, rng.integers(0, Uq + 1, size=n - 1))
        first.append(u[0] / Uq)
        last.append(u[-1] / Uq)
    assert stats.kstest(first, stats.beta(1, n - 1).cdf).pvalue > 0.01
    assert stats.kstest(last, stats.beta(1, n - 1).cdf).pvalue > 0.01


def test_section_7_1_constants():
    """u = 0.4, T = 100: compute -> curve_n
    (40, 0.8), curve_c (48, 0.96); memory -> (40, 4), (92, 9.2); D = 75.
    In ticks (Q = 1000) with B = 1 (c = a); u is 0.4 rounded down in Q20."""
    gen = W.gen_params(68, 16, 1)
    u = (2 * 2**20) // 5
    c = oracle.task_fields(gen, u, 1, 1, 0)          # menu[1] = 100
    assert c["T"] == 100_000 and c["D"] == 75_000
    assert abs(c["a"] - 40_000) <= 1 and c["cn"] == c["a"]
    assert c["fn"] == 800 and c["fc"] == 960
    assert abs(c["cc"] - 48_000) <= 2
    m = oracle.task_fields(gen, u, 1, 1, 1)
    assert m["fn"] == 4000 and m["fc"] == 9200
    assert abs(m["cc"] - 92_000) <= 3


def test_reasonable_time_bump():
    """P:942-944 / reading A-10: the period is raised (up to 4000) until the
    baseline execution time reaches max(Q, B)."""
    gen = W.gen_params(8, 6, 1)
    tiny = 2**20 // 2000  # u ~ 0.0005: at T = 50 units a = 25 ticks < Q
    f = oracle.task_fields(gen, tiny, 0, 1, 0)
    assert f["a"] >= 1000 or f["T"] == 4000 * 1000
    assert f["T"] > 50_000
    f0 = oracle.task_fields(gen, 0, 0, 1, 0)      # u = 0: bumped to the end of the menu
    assert f0["T"] == 4_000_000 and f0["cn"] == 1 and f0["fn"] == 0


@pytest.fixture(scope="module")
def c4_sets():
    gen = W.WORKLOADS["c4"]["gen"](R=20000)
    return gen, oracle.generate(gen, W.SEED, 0, 40)  # 40 x 50 groups = 2000 sets


def test_generated_invariants(c4_sets):
    gen, s = c4_sets
    Q, M = gen["ticks_per_unit"], gen["M"]
    menu = {p * Q for p in gen["period_menu"]}
    assert set(np.unique(s.T).tolist()) <= menu
    assert (s.D * 4 == s.T * 3).all()
    assert (s.B >= 1).all() and (s.B <= 4 * M).all()                # A-13
    assert (s.cn >= 1).all() and (s.cc >= s.cn).all() and (s.fc >= s.fn).all()
    for g in range(s.n_sets):
        if s.valid[g]:
            for i in range(s.n_tasks):  # feasible alone on M SMs (A-9)
                assert oracle.wcet(int(s.B[g, i]), int(s.cn[g, i]), int(s.fn[g, i]), M) <= s.D[g, i]
    assert s.valid.mean() > 0.5
    assert (s.group == np.repeat(np.arange(50), 40)).all()


def test_total_utilisation(c4_sets):
    """sum u_i = U_q exactly (UUniFast); a_i = floor(u_i T_i / 2^20)
    gives U - sum(1/T_i) < sum(a_i/T_i) <= U in utilisation units."""
    gen, s = c4_sets
    M, n_bins = gen["M"], gen["n_bins"]
    for g in range(0, s.n_sets, 7):
        b = int(s.group[g]) % n_bins
        U = Fraction((b + 1) * M * 2**20 // n_bins, 2**20)
        # a is not stored; recover a lower/upper envelope from f = ceil(beta*a)
        beta = [Fraction(10 if t else 2, 100) for t in s.type[g]]
        lo = sum(Fraction(int(f) - 1, 1) / bt / int(T) for f, bt, T in zip(s.fn[g], beta, s.T[g])
                 if f > 0)
        hi = sum(Fraction(int(f), 1) / bt / int(T) for f, bt, T in zip(s.fn[g], beta, s.T[g]))
        assert lo <= U
        assert hi >= U - sum(Fraction(1, int(T)) for T in s.T[g]) - Fraction(1, 10**9)


def test_prm_type_frequency(c4_sets):
    """P:955-957 with prm in {0, .25, .5, .75, 1}: prm 0 -> all compute,
    prm 1 -> all memory, others match prm (chi-square at 1 %).  The
    frequency is a property of the draw; whole-vector discards (A-9) bias the
    accepted sets at high load (memory tasks carry b = 0.1a), so the
    chi-square uses the lowest utilisation bins, where discards are rare."""
    gen, s = c4_sets
    for p_idx, prm in enumerate((0.0, 0.25, 0.5, 0.75, 1.0)):
        rows = ((s.group // gen["n_bins"]) == p_idx) & ((s.group % gen["n_bins"]) < 3)
        t = s.type[rows].ravel()
        if prm in (0.0, 1.0):
            assert (t == int(prm)).all()
        else:
            k = int(t.sum())
            chi = stats.chisquare([k, len(t) - k], [prm * len(t), (1 - prm) * len(t)])
            assert chi.pvalue > 0.01


def test_shard_invariance_and_determinism():
    """Counter-based: sets [0,10) in one call == [0,4) + [4,10) per group."""
    gen = W.WORKLOADS["c2"]["gen"](R=10000)
    a = oracle.generate(gen, W.SEED, 0, 10)
    b1 = oracle.generate(gen, W.SEED, 0, 4)
    b2 = oracle.generate(gen, W.SEED, 4, 6)
    for f in ("T", "D", "B", "cn", "cc", "fn", "fc", "type"):
        x = getattr(a, f).reshape(10, 10, -1)
        y = np.concatenate([getattr(b1, f).reshape(10, 4, -1), getattr(b2, f).reshape(10, 6, -1)], 1)
        assert (x == y).all(), f
    assert (oracle.generate(gen, W.SEED, 0, 10).T == a.T).all()
    assert not (oracle.generate(gen, W.SEED + 1, 0, 10).T == a.T).all()


def test_coefficients_do_not_change_base_sets():
    """C5 reuses the task sets across (k_C, k_M) settings: only cc/fc move."""
    g1 = W.WORKLOADS["c5"]["gen"](R=100, kc=10, km=10)
    g2 = W.WORKLOADS["c5"]["gen"](R=100, kc=20, km=30)
    a, b = oracle.generate(g1, W.SEED, 0, 3), oracle.generate(g2, W.SEED, 0, 3)
    for f in ("T", "D", "B", "cn", "fn", "type", "valid"):
        assert (getattr(a, f) == getattr(b, f)).all()
    assert (a.cc == a.cn).all() and (b.cc >= 2 * b.cn).all()


def test_sched_ratio_by_hand():
    """C.1.11 on a hand example: 3 sets, 2 groups, set 1 invalid."""
    d = W.random_sets(np.random.default_rng(0), 3, 2, 4, n_groups=2)
    d["group"] = np.array([0, 1, 1], np.int32)
    d["valid"] = np.array([1, 0, 1], np.uint8)
    s = oracle.Sets.from_dict(d)
    counts = np.zeros((1, 2, 2, 3), np.int64)
    oracle.sched_ratio(s, np.array([[1, 1, 0], [0, 1, 1]], np.uint8), 0, 2, 0, counts)
    assert counts[0, 0].tolist() == [[1, 1, 0], [0, 1, 0]]
    assert counts[0, 1].tolist() == [[0, 2, 1], [1, 2, 1]]
