"""Pins of the oracle's model layer (A1 RNG, A3 WCET/conflict) against the paper.

Each test names the passage it checks.  None re-types the oracle's formula:
the expected values come from the paper's worked example, SPEC's worked
values, external known-answer vectors, or an independent form of the model
(the per-SM round-robin form, which the paper's example defines).
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- Philox KAT
def test_philox_known_answers():
    """Random123 KAT vectors (tests/golden/philox_kat.json)."""
    for v in gold("philox_kat.json")["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        assert oracle.philox4x32_10(ctr, key) == [int(x, 16) for x in v["out"]]


def test_splitmix64_reference_stream():
    """SplitMix64 from state 0 emits e220a8397b1dcdaf, 6e789e6aa1b965f4,
    06c45d188009454f (Steele et al. OOPSLA'14 reference stream); our
    splitmix64(x) is the output for state x, so x = i * gamma."""
    gamma = 0x9E3779B97F4A7C15
    exp = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    for i, e in enumerate(exp):
        assert oracle.splitmix64((i * gamma) % 2**64) == e


# ------------------------------------------------------- worked example P:4-25
def test_worked_example_per_sm():
    """P:4-25 + figure: 5 blocks; on p1 alone with a memory co-runner
    (cost 1) WCET = 5; split over p1 (memory co-runner, cost 1) and p2
    (compute co-runner, cost 2): 3 and 2 blocks, WCET(tau,p2) = 4, task WCET 4,
    both within D = 7."""
    g = gold("worked_example.json")
    B, D = g["blocks"], g["deadline"]
    per, w = oracle.wcet_per_sm(B, g["all_on_p1"]["cost_per_sm"])
    assert w == g["all_on_p1"]["task_wcet"] == 5
    sp = g["split_p1_p2"]
    per, w = oracle.wcet_per_sm(B, sp["cost_per_sm"])
    assert per == sp["wcet_per_sm"] == [3, 4]
    assert per[1] == sp["wcet_tau_p2"] == 4
    assert w == sp["task_wcet"] == 4
    assert w <= D and 5 <= D


def test_round_robin_blocks_per_sm():
    """P:257-258 round-robin dealing: blocks per SM differ by at most one,
    the first B mod m SMs get the extra block, and they sum to B (figure
    P:82-88 / P:110-113: 3 on p1, 2 on p2)."""
    for B in range(0, 40):
        for m in range(1, 12):
            per, w = oracle.wcet_per_sm(B, [1] * m)  # cost 1 -> per-SM block counts
            assert sum(per) == B
            assert max(per) - min(per) <= 1
            assert per == sorted(per, reverse=True)


@pytest.mark.parametrize("B,c,f", [(5, 1, 0), (5, 2, 0), (17, 3, 4), (100, 1, 2), (1, 9, 9)])
def test_block_form_equals_per_sm_form_with_uniform_cost(B, c, f):
    """§8(c) C.1.3 vs C.1.4: with the same cost on every SM the per-SM
    maximum equals the wave form ceil(B/m)*c + f (tail effect)."""
    for m in range(1, 30):
        _, w = oracle.wcet_per_sm(B, [c] * m, f)
        assert oracle.wcet(B, c, f, m) == w


def test_spec_curve_examples_in_w_form():
    """SPEC eval_curve examples S:64-66 (a/m + b with m | a)."""
    for e in gold("spec_examples.json")["eval_curve"]:
        assert oracle.wcet(e["B"], e["c"], e["f"], e["m"]) == e["W"], e["S"]


def test_curve_form_when_m_divides_B():
    """§3.3: C(m) = a/m + b exactly when m divides the blocks."""
    for B in (12, 60, 120):
        for m in range(1, B + 1):
            if B % m == 0:
                assert oracle.wcet(B, 1, 7, m) == B // m + 7


def test_wcet_monotone_non_increasing():
    """No timing anomaly (Lemma 2 proof P:592): W(m+1) <= W(m)."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        B, c, f = (int(x) for x in (rng.integers(1, 500), rng.integers(1, 50), rng.integers(0, 50)))
        ws = [oracle.wcet(B, c, f, m) for m in range(1, 160)]
        assert all(a >= b for a, b in zip(ws, ws[1:]))


def test_wcet_in_partition_spec():
    """SPEC wcet_in_partition S:84-86: memory task alone 20, with another
    memory task 46 (conflict), with a compute task only 20."""
    e = gold("spec_examples.json")["wcet_in_partition"]
    types_alone = [1]
    assert not oracle.conflict(types_alone, 0b1, 0)
    assert oracle.wcet(e["B"], e["cn"], e["fn"], e["m"]) == e["alone"]
    # with another memory task: conflict -> C^c
    assert oracle.conflict([1, 1], 0b11, 0)
    assert oracle.wcet(e["B"], e["cc"], e["fc"], e["m"]) == e["with_memory"]
    # with a compute task only: no conflict
    assert not oracle.conflict([1, 0], 0b11, 0)


def test_ten_kernel_conflict_example():
    """9 compute + 1 memory kernel in one partition -> the nine compute
    kernels are in conflict, the memory kernel is not."""
    types = [0] * 9 + [1]
    mask = (1 << 10) - 1
    flags = [oracle.conflict(types, mask, i) for i in range(10)]
    assert sum(flags) == 9 and flags[9] is False


def test_conflict_symmetry_and_membership():
    """S:98-101 symmetry; conflict only counts tasks inside the block."""
    rng = np.random.default_rng(2)
    for _ in range(300):
        n = int(rng.integers(1, 12))
        types = [int(x) for x in rng.integers(0, 2, n)]
        mask = int(rng.integers(0, 1 << n))
        for i, j in itertools.combinations(range(n), 2):
            if (mask >> i) & 1 and (mask >> j) & 1 and types[i] == types[j]:
                assert oracle.conflict(types, mask, i) and oracle.conflict(types, mask, j)
        for i in range(n):
            others = [j for j in range(n) if j != i and (mask >> j) & 1]
            assert oracle.conflict(types, mask, i) == any(types[j] == types[i] for j in others)


def test_hyperperiod_spec():
    """SPEC hyperperiod S:94-96."""
    for e in gold("spec_examples.json")["hyperperiod"]:
        assert oracle.hyperperiod(e["T"]) == e["H"]


def test_hyperperiod_overflow_is_loud():
    """LCM overflow is an explicit error, never a silent wrap."""
    primes = [1000003, 1000033, 1000037, 1000039]
    with pytest.raises(oracle.OracleError):
        oracle.hyperperiod(primes)
