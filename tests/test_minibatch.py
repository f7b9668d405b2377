"""Experience hand-off: length-balanced DP mini-batches.

balance_minibatch is the reference's LPT packing (workflow.hpp:63-66,
workflow.cpp:160-182). Golden cases are the reference's own unit tests
(test_workflow.cpp:54-104); random cases are diffed call for call against
the reference library built from its sources (oracle/_ref).
"""
import random

import pytest

from paper_2409_13221_b200._lib import FpError


def test_known_optimum(sched):  # test_workflow.cpp:54-59
    assert sched.balance_minibatch([8, 7, 2, 1], 2) == [[0, 3], [1, 2]]


def test_equal_lengths_split_perfectly(sched):  # test_workflow.cpp:61-64
    groups = sched.balance_minibatch([5] * 12, 4)
    assert [len(g) for g in groups] == [3, 3, 3, 3]


def test_lpt_bound_and_round_robin(sched):  # test_workflow.cpp:66-97 (same checks, own RNG)
    rng = random.Random(31)
    for _ in range(50):
        n, dp = 4 + rng.randrange(60), 2 + rng.randrange(3)
        if n < dp:
            continue
        lengths = [1 + rng.randrange(1000) for _ in range(n)]
        groups = sched.balance_minibatch(lengths, dp)
        assert sorted(i for g in groups for i in g) == list(range(n))
        load = [sum(lengths[i] for i in g) for g in groups]
        assert max(load) <= sum(lengths) // dp + max(lengths)
        rr = [sum(lengths[i] for i in range(n) if i % dp == g) for g in range(dp)]
        assert max(load) <= max(rr)


def test_argument_checks(sched):  # test_workflow.cpp:99-102
    with pytest.raises(FpError) as e:
        sched.balance_minibatch([1, 2], 0)
    assert e.value.status == 2
    with pytest.raises(FpError):
        sched.balance_minibatch([1], 2)


def test_matches_reference_library(sched, ref_sched):
    rng = random.Random(7)
    for _ in range(200):
        dp = 1 + rng.randrange(16)
        n = dp + rng.randrange(300)
        # many ties: lengths from a small range exercise the tie rules
        hi = rng.choice([3, 50, 4096])
        lengths = [1 + rng.randrange(hi) for _ in range(n)]
        assert sched.balance_minibatch(lengths, dp) == ref_sched.balance_minibatch(lengths, dp)
