"""K8 on the B200: pairwise_sorting_accuracy (priority.cpp:165-189) by exact
integer counting, bit-exact against the reference's O(N^2) double sums."""
import numpy as np
import pytest

import kxf
import oracle_ffi as O
from helpers import bits
from paper_2508_06948_b200.sched import sorting_accuracy

pytestmark = pytest.mark.gpu


def test_matches_reference_fixture(gpu_lib):
    d = kxf.read("accuracy.kxf")
    off = d["offsets"]
    for t in range(len(off) - 1):
        sl = slice(off[t], off[t + 1])
        for scope, key in (("cross_agent", "acc_cross"), ("all", "acc_all")):
            acc, _, _ = sorting_accuracy(d["agent"][sl], d["remaining"][sl], d["present"][sl], scope)
            exp = d[key][t]
            if np.isnan(exp):
                assert acc is None
            else:
                assert bits(acc) == bits(exp)


@pytest.mark.parametrize("n,agents,ties", [(2, 1, False), (1000, 5, True), (20000, 37, False),
                                           (30000, 3, True)])
def test_matches_oracle_random(gpu_lib, n, agents, ties):
    rng = np.random.default_rng(n)
    agent = rng.integers(0, agents, n)
    rem = np.floor(rng.uniform(0, 50, n)) if ties else rng.uniform(0, 50, n)
    present = (rng.uniform(size=n) < 0.95).astype(np.uint8)
    for scope in ("cross_agent", "all"):
        acc, pairs, _ = sorting_accuracy(agent, rem, present, scope)
        eacc, epairs = O.pairwise_accuracy(agent, rem, present, scope == "all")
        assert pairs == epairs
        assert (acc is None and eacc is None) or bits(acc) == bits(eacc)


def test_large_schedule_is_fast_and_sane(gpu_lib):
    # 4M requests: the reference's O(N^2) walk would take hours.
    rng = np.random.default_rng(1)
    n = 4_000_000
    agent = rng.integers(0, 10, n)
    rem = np.sort(rng.uniform(0, 10, n))  # perfectly ordered schedule
    acc, pairs, correct = sorting_accuracy(agent, rem, None, "cross_agent")
    assert pairs > 0 and acc == 1.0
