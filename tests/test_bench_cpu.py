"""bench.py's host-side helpers, checked on CPU against independent counts: the
candidate count per set (C.1.6) against the oracle's enumeration count, the
allocations-per-k (Stirling numbers of the second kind) against a brute-force count of
restricted growth strings, the roofline denominator, and the default sizes of the
workloads the bench times."""
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import gp_workloads as W  # noqa: E402
import oracle  # noqa: E402


def rgs_count(n, k):
    """Restricted growth strings of length n with exactly k labels, by brute force."""
    c = 0
    for s in itertools.product(range(n), repeat=n):
        if s[0] != 0:
            continue
        mx, ok = 0, True
        for x in s[1:]:
            if x > mx + 1:
                ok = False
                break
            mx = max(mx, x)
        c += ok and mx + 1 == k
    return c


def test_stirling_numbers_match_rgs_counts():
    for n in range(1, 7):
        for k in range(1, n + 1):
            assert bench.stirling2(n, k) == rgs_count(n, k), (n, k)


def test_candidate_counts_match_the_oracle():
    for M, n in [(4, 3), (8, 6), (20, 6), (5, 4), (12, 4), (32, 3)]:
        assert bench.n_candidates(M, n) == oracle.count_candidates(M, n), (M, n)
    assert bench.n_candidates(20, 6) == 694755 and bench.n_candidates(8, 6) == 11334


def test_peak_is_the_issue_ceiling():
    peak, src = bench.peak_lane_ops()
    assert "148 SM" in src
    assert 3.0e13 < peak < 4.5e13  # 148 x 4 x 32 lanes x ~2 GHz


def test_default_sizes_are_the_survey_configs():
    sets = {k: W.WORKLOADS[k]["gen"](R=bench.DEFAULT_REPS[k]) for k in ("c2", "c3", "c4", "c5")}
    total = {k: g["n_prm"] * g["n_bins"] * g["sets_per_group"] for k, g in sets.items()}
    assert total == {"c2": 10**5, "c3": 10**5, "c4": 10**6, "c5": 10**5}
    assert (sets["c4"]["M"], sets["c4"]["n_tasks"]) == (148, 32)
    assert (sets["c3"]["M"], sets["c3"]["n_tasks"]) == (20, 6)
