"""K2/K3/K4 on the B200 against the reference's own order (golden fixtures)
and the oracle restatement. Integer/index output: bit-exact."""
import numpy as np
import pytest

import oracle_ffi as O
import paper_2508_06948_b200 as kx
from helpers import POLICIES, bits, order_fixture, random_queue

pytestmark = pytest.mark.gpu

ORDER = ["order_unit.kxf", "order_ties.kxf", "order_colocated_s1.kxf", "order_colocated_s2.kxf"]


def make_sched(n_pools, cap, n_agents=4096):
    inst = [kx.InstanceProfile(id=p, pool=p) for p in range(n_pools)]
    return kx.DeviceScheduler(inst, n_pools=n_pools, queue_capacity=max(cap, 1), max_agents=n_agents)


def load(s, q: O.QueueArrays, t: O.TableArrays, policy):
    s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
    if t.rem is not None:
        s.set_remaining_table(t.view.rem_base, t.rem, t.rem_present)
    s.set_scheduler(policy)
    s.upload(q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid)


@pytest.mark.parametrize("name", ORDER)
@pytest.mark.parametrize("policy", POLICIES)
def test_order_matches_reference_fixture(gpu_lib, name, policy):
    d, q, t, n_pools = order_fixture(name)
    s = make_sched(n_pools, len(q.agent))
    load(s, q, t, policy)
    s.order()
    perm, offs = s.fetch_order()
    assert np.array_equal(offs, d[f"{policy}.pool_offsets"])
    assert np.array_equal(perm, d[f"{policy}.perm"])
    k = s.score()
    for j in range(3):
        assert np.array_equal(bits(k[j]), bits(d[f"{policy}.k{j}"]))


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("n,pools,grain", [(1, 1, 0.0), (1000, 1, 0.0), (65536, 3, 0.5),
                                           (300_001, 8, 0.0), (200_000, 2, 0.25)])
def test_order_matches_oracle_random(gpu_lib, policy, n, pools, grain):
    rng = np.random.default_rng(n + pools)
    q, t = random_queue(rng, n, n_agents=37, n_pools=pools, tie_grain=grain)
    s = make_sched(pools, n)
    load(s, q, t, policy)
    s.order()
    perm, offs = s.fetch_order()
    ref_perm, ref_offs = O.sort(policy, q, t, pools)
    assert np.array_equal(offs, ref_offs)
    assert np.array_equal(perm, ref_perm)


@pytest.mark.parametrize("policy", POLICIES)
def test_order_many_agents(gpu_lib, policy):
    # more agents than key generation's shared-memory table (2048): the
    # global-table variant of k_keygen
    rng = np.random.default_rng(3000)
    q, t = random_queue(rng, 50_000, n_agents=3000, n_pools=4, tie_grain=0.25)
    s = make_sched(4, 50_000)
    load(s, q, t, policy)
    s.order()
    perm, offs = s.fetch_order()
    ref_perm, ref_offs = O.sort(policy, q, t, 4)
    assert np.array_equal(offs, ref_offs)
    assert np.array_equal(perm, ref_perm)


@pytest.mark.parametrize("n", [40, 1500, 40_000])
def test_degenerate_all_equal_keys(gpu_lib, n):
    # every request shares agent, app_start and queue_enter: one tie run of
    # length n resolved by (msg, uid, index) — exercises the warp, CTA-smem
    # and global merge paths of the tie-fix.
    rng = np.random.default_rng(n)
    q = O.QueueArrays(np.zeros(n, np.int32), np.ones(n), np.full(n, 3.0), np.full(n, 3.0),
                      rng.integers(0, 7, n).astype(np.uint64), rng.permutation(n).astype(np.uint64) + 5)
    t = O.TableArrays(np.zeros(1, np.int32), [1.0], [2], [1.0])
    for policy in POLICIES:
        s = make_sched(1, n)
        load(s, q, t, policy)
        s.order()
        perm, _ = s.fetch_order()
        assert np.array_equal(perm, O.sort(policy, q, t, 1)[0])


@pytest.mark.parametrize("seed", [0, 1])
def test_tie_runs_across_chunk_boundaries(gpu_lib, seed):
    # runs of 1-20 equal primary times (the thread fixer takes <= 16, the CTA
    # fixer longer ones), ~31K requests: runs straddle the tie-fix kernel's
    # 4096-key chunks (a run belongs to the chunk of its first key); few
    # queue_enter values and msg keys, so the exact tuple reaches msg and uid
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 21, 3000)
    n = int(lens.sum())
    app = np.repeat(np.arange(len(lens), dtype=np.float64) * 0.5, lens)
    qe = rng.integers(0, 4, n).astype(np.float64) + 2000.0
    msg = rng.integers(0, 3, n).astype(np.uint64)
    uid = rng.permutation(n).astype(np.uint64)
    sh = rng.permutation(n)
    q = O.QueueArrays(np.zeros(n, np.int32), np.ones(n), app[sh], qe[sh], msg[sh], uid[sh])
    t = O.TableArrays(np.zeros(1, np.int32), [1.0], [2], [1.0])
    for policy in POLICIES:
        s = make_sched(1, n)
        load(s, q, t, policy)
        s.order()
        perm, _ = s.fetch_order()
        assert np.array_equal(perm, O.sort(policy, q, t, 1)[0]), policy


def test_negative_zero_equals_zero(gpu_lib):
    n = 64
    app = np.where(np.arange(n) % 2 == 0, -0.0, 0.0)
    q = O.QueueArrays(np.zeros(n, np.int32), np.ones(n), app, app.copy(),
                      np.arange(n)[::-1].astype(np.uint64), np.arange(n).astype(np.uint64))
    t = O.TableArrays(np.zeros(1, np.int32), [0.0], [1], [1.0])
    s = make_sched(1, n)
    load(s, q, t, "fcfs")
    s.order()
    assert np.array_equal(s.fetch_order()[0], O.sort("fcfs", q, t, 1)[0])


def test_empty_queue(gpu_lib):
    s = make_sched(2, 16)
    s.set_agent_tables([0, 1])
    s.upload(np.zeros(0, np.int32), np.zeros(0), np.zeros(0), np.zeros(0), np.zeros(0), np.zeros(0))
    s.order()
    perm, offs = s.fetch_order()
    assert len(perm) == 0 and np.array_equal(offs, [0, 0, 0])


def test_invalid_inputs_raise_invalid_argument(gpu_lib):
    s = make_sched(1, 16)
    s.set_agent_tables([0])
    with pytest.raises(kx.KxError) as e:
        s.upload([5], [1], [0.0], [0.0], [0], [1])  # agent outside the table
    assert e.value.code == 1
    with pytest.raises(kx.KxError) as e:
        s.upload([0], [1], [np.nan], [0.0], [0], [1])
    assert e.value.code == 1
    with pytest.raises(kx.KxError) as e:
        s.upload(np.zeros(17, np.int32), np.ones(17), np.zeros(17), np.zeros(17), np.zeros(17), np.arange(17))
    assert e.value.code == 1


def test_order_reused_across_table_versions(gpu_lib):
    # Rebuilt priority tables take effect on the next order (scheduler.hpp:29-30).
    rng = np.random.default_rng(5)
    q, t = random_queue(rng, 5000, n_agents=9, n_pools=1)
    s = make_sched(1, 5000)
    load(s, q, t, "kairos")
    for _ in range(3):
        t.pk[:] = np.round(rng.uniform(0, 3, len(t.pk)), 1)
        s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
        s.order()
        assert np.array_equal(s.fetch_order()[0], O.sort("kairos", q, t, 1)[0])


@pytest.mark.parametrize("policy", POLICIES)
def test_enqueue_appends_like_readyqueue(gpu_lib, policy):
    # ReadyQueue::enqueue (priority.hpp:72) in chunks == one upload of the
    # concatenation; exact-tuple ties keep queue (push_back) order
    rng = np.random.default_rng(72)
    n, pools = 90_001, 3
    q, t = random_queue(rng, n, n_agents=37, n_pools=pools, tie_grain=0.5)
    s = make_sched(pools, n)
    cols = [q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid]
    cuts = [0, 1, 40_000, 40_000, 77_777, n]
    s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
    if t.rem is not None:
        s.set_remaining_table(t.view.rem_base, t.rem, t.rem_present)
    s.set_scheduler(policy)
    s.upload(*[c[:cuts[1]] for c in cols])
    for a, b in zip(cuts[1:], cuts[2:]):
        s.enqueue(*[c[a:b] for c in cols])
    assert s.size() == n
    s.order()
    perm, offs = s.fetch_order()
    ref_perm, ref_offs = O.sort(policy, q, t, pools)
    assert np.array_equal(offs, ref_offs)
    assert np.array_equal(perm, ref_perm)


def test_enqueue_beyond_capacity_fails(gpu_lib):
    rng = np.random.default_rng(73)
    q, t = random_queue(rng, 100, n_agents=5, n_pools=1)
    s = make_sched(1, 100)
    s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
    s.upload(q.agent[:60], q.prompt[:60], q.app_start[:60], q.queue_enter[:60], q.msg_key[:60], q.uid[:60])
    with pytest.raises(Exception):
        s.enqueue(q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid)
