"""CPU checks of the closed forms the bit-sliced evaluator's main pass relies on
("Full corner" / "Tables"), against brute force over the candidate space of
C.1.6: an allocation with k blocks has the size vectors s (s_j >= 1, sum(s) <= M) in
lexicographic order, i.e. the prefix-sum k-subsets c of {1..M} in lexicographic order.

- the lex rank of a k-subset, rank(c) = C(M, k) - 1 - sum_j C(M - c_j, k - j);
- a corner {s : s_j >= lo_j + 1} holds C(M - sum(lo), k) candidates, its smallest sum(s) is
  sum(lo) + k and its lexicographically first element is the apex lo + 1;
- the full corner table built as k suffix scans, one chain per (allocation, dimension),
  walking each chain downwards and summing in place (k_fct_pass), equals the domination sum
  over the corner at every candidate;
- the three-part corner table (k_corner_table) equals the domination sum in the last three
  parts with the outer parts fixed.

These restate the kernels' arithmetic in Python and pin it to enumeration; the GPU parity
tests then compare the kernels with the oracle on the same sets."""
import itertools
from math import comb

import pytest


def candidates(M, k):
    """Size vectors of one allocation with k blocks, in rank order (brute force)."""
    return [tuple(b - a for a, b in zip((0,) + c[:-1], c))
            for c in itertools.combinations(range(1, M + 1), k)]


def lex_rank(c, M):
    k = len(c)
    return comb(M, k) - 1 - sum(comb(M - cj, k - j) for j, cj in enumerate(c))


def prefix(s):
    return tuple(itertools.accumulate(s))


def h(r):  # any fixed per-rank value stands in for splitmix64
    return (r * 0x9E3779B97F4A7C15 + 12345) % (1 << 64)


@pytest.mark.parametrize("M,k", [(1, 1), (5, 1), (5, 2), (6, 3), (8, 4), (9, 5), (7, 7), (10, 3)])
def test_lex_rank_formula(M, k):
    for r, s in enumerate(candidates(M, k)):
        assert lex_rank(prefix(s), M) == r


@pytest.mark.parametrize("M,k", [(5, 2), (6, 3), (8, 4), (9, 3), (7, 5)])
def test_corner_closed_forms(M, k):
    cands = candidates(M, k)
    for lo in itertools.product(range(M), repeat=k):
        corner = [(r, s) for r, s in enumerate(cands) if all(sj >= l + 1 for sj, l in zip(s, lo))]
        L = M - sum(lo)
        n = comb(L, k) if L >= k else 0
        assert len(corner) == n
        if n:
            apex = tuple(l + 1 for l in lo)
            assert corner[0][1] == apex  # lexicographically first = the apex
            assert corner[0][0] == lex_rank(prefix(apex), M)
            assert min(sum(s) for _, s in corner) == sum(lo) + k


def full_corner_table(M, k):
    """k_fct_pass: level 0 = h(rank); pass j scans part i = k - j along every chain (the
    candidates differing in part i only), downwards, summing in place."""
    F = [h(r) for r in range(comb(M, k))]
    for j in range(1, k + 1):
        i = k - j
        for d in itertools.combinations(range(1, M), k - 1):  # the chain's other parts
            dtot = d[-1] if d else 0
            acc = 0
            for t in range(M - dtot, 0, -1):
                c = list(d[:i]) + [(d[i - 1] if i > 0 else 0) + t] + [x + t for x in d[i:]]
                r = lex_rank(c, M)
                acc = (acc + F[r]) % (1 << 64)
                F[r] = acc
    return F


@pytest.mark.parametrize("M,k", [(4, 1), (5, 2), (6, 3), (7, 4), (6, 6)])
def test_full_corner_table(M, k):
    cands = candidates(M, k)
    F = full_corner_table(M, k)
    for r, s in enumerate(cands):
        ref = sum(h(r2) for r2, s2 in enumerate(cands)
                  if all(a >= b for a, b in zip(s2, s))) % (1 << 64)
        assert F[r] == ref


@pytest.mark.parametrize("M,k", [(6, 3), (7, 4), (8, 5)])
def test_three_part_corner_table(M, k):
    """k_corner_table: within a block (outer parts s_0..s_{k-4} fixed), the sum over the
    candidates dominating r in the last three parts."""
    cands = candidates(M, k)
    for r, s in enumerate(cands):
        ref = sum(h(r2) for r2, s2 in enumerate(cands)
                  if s2[:k - 3] == s[:k - 3] and all(a >= b for a, b in zip(s2[k - 3:], s[k - 3:])))
        # the same sum restated as the kernel builds it: sweeps v >= s_{k-3}, runs with
        # s_{k-2} >= y + 1, each run's top range of last parts >= z + 1
        q = sum(s[:k - 3])
        x, y, z = s[k - 3] - 1, s[k - 2] - 1, s[k - 1] - 1
        got = 0
        for v in range(x + 1, M - q + 1):
            for s2 in range(y + 1, M - q - v + 1):
                for s3 in range(z + 1, M - q - v - s2 + 1):
                    got += h(lex_rank(prefix(s[:k - 3] + (v, s2, s3)), M))
        assert got % (1 << 64) == ref % (1 << 64)
