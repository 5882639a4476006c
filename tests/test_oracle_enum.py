"""Pins of the oracle's candidate space (A2, §8(c) C.1.6).

Closed form: N_c(M,n) = sum_k S(n,k) C(M,k), with S computed here by the
explicit inclusion-exclusion formula (not the recurrence the oracle uses).
Brute force: every (task partition, SM sizes) configuration of tiny GPUs is
built independently with itertools and must appear exactly once, in the
stated rank order; unrank(r) must agree with the enumeration.
"""
import itertools
from math import comb, factorial

import pytest

import oracle


def stirling2_closed(n, k):
    return sum((-1) ** j * comb(k, j) * (k - j) ** n for j in range(k + 1)) // factorial(k)


def n_c(M, n):
    return sum(stirling2_closed(n, k) * comb(M, k) for k in range(1, min(M, n) + 1))


def test_count_configs():
    """26 / 11,334 / 694,755 for C1 / C2 / C3."""
    assert oracle.count_candidates(4, 3) == 26 == n_c(4, 3)
    assert oracle.count_candidates(8, 6) == 11334 == n_c(8, 6)
    assert oracle.count_candidates(20, 6) == 694755 == n_c(20, 6)


@pytest.mark.parametrize("M,n", [(1, 1), (3, 5), (7, 7), (16, 9), (68, 10), (148, 12)])
def test_count_closed_form(M, n):
    assert oracle.count_candidates(M, n) == n_c(M, n)


def test_count_overflow_refused():
    """C4/C5 shapes exceed 2^63 candidates: exhaustive mode is refused."""
    with pytest.raises(OverflowError):
        oracle.count_candidates(148, 32)
    with pytest.raises(OverflowError):
        oracle.count_candidates(68, 16)


def brute_candidates(M, n):
    """Every set partition of the n tasks (as canonical RGS: blocks numbered by
    first appearance) with every size vector, built from surjections."""
    out = set()
    for k in range(1, min(M, n) + 1):
        for f in itertools.product(range(k), repeat=n):
            if len(set(f)) != k:
                continue
            relabel, rgs = {}, []
            for x in f:
                relabel.setdefault(x, len(relabel))
                rgs.append(relabel[x])
            for s in itertools.product(range(1, M + 1), repeat=k):
                if sum(s) <= M:
                    out.add((k, tuple(rgs), tuple(s)))
    return sorted(out)  # k, then RGS lexicographic, then s lexicographic


@pytest.mark.parametrize("M,n", [(1, 1), (1, 3), (2, 2), (3, 3), (4, 3), (5, 4), (6, 4), (8, 3), (4, 5)])
def test_enumeration_matches_brute_force(M, n):
    want = brute_candidates(M, n)
    bot, bs = oracle.enumerate_candidates(M, n)
    got = []
    for r in range(len(bot)):
        k = int(bot[r].max()) + 1
        got.append((k, tuple(int(x) for x in bot[r]), tuple(int(x) for x in bs[r][:k])))
        assert all(int(x) == 0 for x in bs[r][k:])
    assert got == want
    assert len(got) == oracle.count_candidates(M, n)


@pytest.mark.parametrize("M,n", [(4, 3), (6, 4), (8, 5), (5, 6)])
def test_unrank_matches_enumeration(M, n):
    bot, bs = oracle.enumerate_candidates(M, n)
    for r in range(len(bot)):
        b2, s2 = oracle.unrank(M, n, r)
        assert (b2 == bot[r]).all() and (s2 == bs[r]).all()


def test_unrank_deep_ranks_c3():
    """Far ranks of C3 agree with a windowed enumeration."""
    total = oracle.count_candidates(20, 6)
    for first in (0, 5000, 123456, total - 40):
        bot, bs = oracle.enumerate_candidates(20, 6, first, 40)
        for r in range(40):
            b2, s2 = oracle.unrank(20, 6, first + r)
            assert (b2 == bot[r]).all() and (s2 == bs[r]).all()


def test_label_expanded_count_is_derived_figure():
    """Reading A-28: the label-expanded space (ordered compositions of exactly
    M x surjective task->part maps) has sum_k k! S(n,k) C(M-1,k-1) elements:
    37 for (4,3) and 16,954,119 for (20,6)."""
    def expanded(M, n):
        return sum(factorial(k) * stirling2_closed(n, k) * comb(M - 1, k - 1)
                   for k in range(1, min(M, n) + 1))
    assert expanded(4, 3) == 37 and expanded(20, 6) == 16954119
    brute = 0
    for k in range(1, 4):
        surj = sum(1 for f in itertools.product(range(k), repeat=3) if len(set(f)) == k)
        comps = sum(1 for s in itertools.product(range(1, 5), repeat=k) if sum(s) == 4)
        brute += surj * comps
    assert brute == 37
