"""K9 on the B200: profiler ingestion (EmpiricalDistribution::add with the
sliding window and doubling-checkpoint W1 convergence, record_remaining /
record_execution) against the reference fixture and the oracle."""
import numpy as np
import pytest

import kxf
import oracle_ffi as O
import paper_2508_06948_b200 as kx
from helpers import bits

pytestmark = pytest.mark.gpu


def _check(p, ex, rm, A):
    for kind, dists in ((0, ex), (1, rm)):
        for a in range(A):
            s, tot, cv, last = p.read(kind, a)
            es, etot, ecv, elast = dists[a].read()
            assert np.array_equal(bits(s), bits(es)), (kind, a)
            assert tot == etot and cv == bool(ecv) and bits(last) == bits(elast), (kind, a)


def test_profiler_matches_reference_fixture(gpu_lib):
    d = kxf.read("profiler.kxf")
    A = int(d["n_agents"][0])
    p = kx.Profiler(A, capacity=8192)
    off, agent, es, ee = d["off"], d["agent"], d["exec_start"], d["exec_end"]
    # execution samples in record order, then the workflows (two batches)
    p.record_execution(agent, ee - es)
    h = len(off) // 2
    n1 = p.record_remaining(off[:h + 1], agent[:off[h]], es[:off[h]], ee[:off[h]])
    n2 = p.record_remaining(off[h:] - off[h], agent[off[h]:], es[off[h]:], ee[off[h]:])
    assert np.array_equal(np.concatenate([n1, n2]), d["newly"])
    for kind, pre in ((0, "exec"), (1, "rem")):
        for a in range(A):
            s, tot, cv, last = p.read(kind, a)
            q = f"{pre}{a}."
            assert np.array_equal(bits(s), bits(d[q + "samples"])), q
            assert tot == int(d[q + "total"][0]) and cv == bool(d[q + "converged"][0]), q
            assert bits(last) == bits(d[q + "last"][0]), q


@pytest.mark.parametrize("capacity", [600, 20000])  # shared-memory and global-memory windows
def test_profiler_matches_oracle_random(gpu_lib, capacity):
    rng = np.random.default_rng(capacity)
    A = 7
    exec_cfg, rem_cfg = (3, 0.2, 0), (4, 0.3, 37)
    p = kx.Profiler(A, exec_cfg=exec_cfg, remaining_cfg=rem_cfg, capacity=capacity)
    ex = [O.Dist(*exec_cfg) for _ in range(A)]
    rm = [O.Dist(*rem_cfg) for _ in range(A)]
    for batch in range(4):
        W = int(rng.integers(20, 120))
        nrec = rng.integers(0, 5, W)  # empty workflows included
        off = np.concatenate([[0], np.cumsum(nrec)]).astype(np.int64)
        n = int(off[-1])
        agent = rng.integers(0, A, n).astype(np.int32)
        es = np.round(rng.uniform(0, 10, n), 1)  # coarse: equal samples and ties
        ee = es + np.round(rng.uniform(0, 3, n) * (1 + agent), 1)
        p.record_execution(agent, ee - es)
        got = p.record_remaining(off, agent, es, ee)
        # oracle, with the same state carried between batches
        newly = np.zeros(W, np.uint8)
        for r in range(n):
            ex[agent[r]].add(ee[r] - es[r])
        for w in range(W):
            b, e = off[w], off[w + 1]
            if b == e:
                continue
            fin = ee[b]
            for r in range(b, e):
                fin = ee[r] if fin < ee[r] else fin
            for r in range(b, e):
                if rm[agent[r]].add(fin - es[r]) == 1:
                    newly[w] = 1
        assert np.array_equal(got, newly), batch
        _check(p, ex, rm, A)


def test_profiler_errors(gpu_lib):
    p = kx.Profiler(2, remaining_cfg=(16, 0.05, 8), capacity=64)
    with pytest.raises(kx.KxError):  # negative sample: nothing applied
        p.record_remaining([0, 2], [0, 1], [5.0, 1.0], [1.0, 2.0])
    assert p.read(1, 0)[1] == 0
    with pytest.raises(kx.KxError):  # unbounded execution kind beyond capacity
        p.record_execution(np.zeros(100, np.int32), np.ones(100))
    with pytest.raises(kx.KxError):
        kx.Profiler(2, remaining_cfg=(16, 0.05, 4096), capacity=100)  # window does not fit
