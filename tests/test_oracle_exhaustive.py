"""Pins of the oracle's exhaustive verdicts (A2-A4 fused, §8(c) C.1.8) and the
cross-step invariants of SURVEY §8(c) C.3."""
import functools
import itertools
import json
import os

import numpy as np
import pytest

import gp_workloads as W
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
MASK64 = 2**64 - 1


def _sizes(M, k):
    if k == 0:
        yield ()
        return
    for v in range(1, M - (k - 1) + 1):
        for rest in _sizes(M - v, k - 1):
            yield (v,) + rest


@functools.lru_cache(maxsize=None)
def brute_candidates(M, n):
    """Independent construction: surjections relabelled to canonical RGS,
    crossed with every size vector (sum <= M), sorted into rank order."""
    out = set()
    for k in range(1, min(M, n) + 1):
        for f in itertools.product(range(k), repeat=n):
            if len(set(f)) != k:
                continue
            relabel, rgs = {}, []
            for x in f:
                relabel.setdefault(x, len(relabel))
                rgs.append(relabel[x])
            for s in _sizes(M, k):
                out.add((k, tuple(rgs), s))
    return sorted(out)


def test_c1_table_golden_and_hand_rule():
    """BASELINE configs[0] (worked example scaled to exhaustive).  Hand rule
    (single deadline t = 7 <= H = 20): a block passes iff sum of
    ceil(5/s) * c^x <= 7, with c^x = 2 when another task of the same type
    shares the block, else 1."""
    with open(os.path.join(GOLD, "c1_exhaustive_table.json")) as f:
        table = json.load(f)
    sets = oracle.Sets.from_dict(W._c1_sets())
    per, bits = oracle.exhaustive(sets, bits=True)
    cands = brute_candidates(4, 3)
    assert len(cands) == table["n_candidates"] == 26
    g1 = oracle.allocate(sets, "1G")
    for v, row in enumerate(table["rows"]):
        types = [0 if ch == "C" else 1 for ch in row["types"]]
        assert list(sets.type[v]) == types
        ok_ranks = []
        for r, (k, rgs, s) in enumerate(cands):
            good = True
            for j in range(k):
                members = [i for i in range(3) if rgs[i] == j]
                load = 0
                for i in members:
                    conflict = any(types[o] == types[i] for o in members if o != i)
                    load += -(-5 // s[j]) * (2 if conflict else 1)
                good &= load <= 7
            if good:
                ok_ranks.append(r)
        assert len(ok_ranks) == row["schedulable"] == per[v, 0]
        assert min(sum(cands[r][2]) for r in ok_ranks) == row["pi_star"] == per[v, 1]
        assert ok_ranks[0] == row["first_rank"] == per[v, 2]
        h = sum(oracle.splitmix64(r) for r in ok_ranks) & MASK64
        assert np.int64(per[v, 3]).view(np.uint64) == h
        got_bits = [r for r in range(26) if (int(bits[v, r // 32]) >> (r % 32)) & 1]
        assert got_bits == ok_ranks
        assert bool(g1["ok"][v]) == row["one_g"]
    # label-expanded space for CCC: 18 of 37 schedulable
    types = [0, 0, 0]
    n_ok = n_all = 0
    for k in range(1, 4):
        for f in itertools.product(range(k), repeat=3):
            if len(set(f)) != k:
                continue
            for s in itertools.product(range(1, 5), repeat=k):
                if sum(s) != 4:
                    continue
                n_all += 1
                good = True
                for j in range(k):
                    mem = [i for i in range(3) if f[i] == j]
                    C = [oracle.wcet(5, 2 if len(mem) > 1 else 1, 0, s[j]) for _ in mem]
                    good &= oracle.edf_pdc(C, [7] * len(mem), [20] * len(mem))[0]
                n_ok += good
    assert (n_ok, n_all) == (18, 37)


@pytest.fixture(scope="module")
def c2_sample():
    gen = W.WORKLOADS["c2"]["gen"](R=10000)
    s = oracle.generate(gen, W.SEED, 0, 6)  # 6 reps x 10 bins = 60 sets
    per, bits = oracle.exhaustive(s, bits=True)
    return gen, s, per, bits


def _rank_index(M, n):
    return {c: r for r, c in enumerate(brute_candidates(M, n))}


def test_bits_consistent_with_per_set(c2_sample):
    gen, s, per, bits = c2_sample
    cands = brute_candidates(8, 6)
    for g in range(s.n_sets):
        ranks = [r for r in range(len(cands)) if (int(bits[g, r // 32]) >> (r % 32)) & 1]
        assert per[g, 0] == len(ranks)
        assert per[g, 2] == (ranks[0] if ranks else -1)
        assert per[g, 1] == (min(sum(cands[r][2]) for r in ranks) if ranks else 0)
        h = sum(oracle.splitmix64(r) for r in ranks) & MASK64
        assert int(np.int64(per[g, 3]).view(np.uint64)) == h


def test_cross_step_invariants(c2_sample):
    """SURVEY §8(c) C.3 cross-step invariants on generated C2 sets."""
    gen, s, per, bits = c2_sample
    M, n = 8, 6
    idx = _rank_index(M, n)
    cands = brute_candidates(M, n)
    g1 = oracle.allocate(s, "1G")
    heur = {v: oracle.allocate(s, v) for v in ("SMS_ACT", "SMS_INA", "BF_ACT", "BF_INA")}
    for g in range(s.n_sets):
        bit = lambda r: (int(bits[g, r // 32]) >> (r % 32)) & 1  # noqa: E731
        # the (k=1, s=M) candidate, rank M-1, is the 1G baseline
        assert bit(M - 1) == g1["ok"][g]
        # Lemma 2 sizes, scanned independently
        m_i = []
        for i in range(n):
            ms = [m for m in range(1, M + 1)
                  if oracle.wcet(int(s.B[g, i]), int(s.cn[g, i]), int(s.fn[g, i]), m) <= s.D[g, i]]
            m_i.append(ms[0] if ms else M + 1)
        for r in range(len(cands)):
            if bit(r):
                k, rgs, sz = cands[r]
                for j in range(k):
                    assert sz[j] >= max(m_i[i] for i in range(n) if rgs[i] == j)
        for v, res in heur.items():
            if res["k"][g] == 0:  # rejected by Lemma 1 / Lemma 2 before merging
                assert per[g, 0] == 0
            if res["ok"][g]:
                k = int(res["k"][g])
                key = (k, tuple(int(x) for x in res["block_of_task"][g]),
                       tuple(int(x) for x in res["block_size"][g][:k]))
                assert bit(idx[key]), v  # heuristic solution is a schedulable candidate
                assert res["pi"][g] >= per[g, 1]  # Pi_heur >= Pi*
                assert res["pi"][g] <= M
    # exists(M) => exists(M+1): more SMs never hurt
    s9 = oracle.Sets.from_dict({**s.to_dict(), "M": M + 1})
    per9 = oracle.exhaustive(s9)
    assert all(per9[g, 0] > 0 for g in range(s.n_sets) if per[g, 0] > 0)


def test_m1_is_uniprocessor_edf():
    """M = 1: the only candidate is all tasks on one SM; its verdict is
    uniprocessor EDF with conflict-resolved costs, checked by simulation."""
    rng = np.random.default_rng(7)
    d = W.random_sets(rng, 40, 4, 1, periods=(4, 6, 8, 12, 24), cost_max=2)
    s = oracle.Sets.from_dict(d)
    per = oracle.exhaustive(s)
    for g in range(s.n_sets):
        types = [int(x) for x in s.type[g]]
        C = []
        for i in range(4):
            conflict = any(types[o] == types[i] for o in range(4) if o != i)
            c, f = (s.cc[g, i], s.fc[g, i]) if conflict else (s.cn[g, i], s.fn[g, i])
            C.append(oracle.wcet(int(s.B[g, i]), int(c), int(f), 1))
        T = [int(x) for x in s.T[g]]
        D = [int(x) for x in s.D[g]]
        assert per[g, 0] == int(oracle.simulate_edf(C, D, T, oracle.hyperperiod(T)))


def test_rank_window_matches_full(c2_sample):
    gen, s, per, bits = c2_sample
    sub = s.subset(slice(0, 5))
    full = oracle.exhaustive(sub)
    lo, hi = 3000, 7000
    part, pbits = oracle.exhaustive(sub, lo, hi, bits=True)
    for g in range(sub.n_sets):
        ranks = [r for r in range(lo, hi) if (int(bits[g, r // 32]) >> (r % 32)) & 1]
        assert part[g, 0] == len(ranks)
        got = [lo + o for o in range(hi - lo) if (int(pbits[g, o // 32]) >> (o % 32)) & 1]
        assert got == ranks
    assert full[:, 0].sum() == per[:5, 0].sum()
