"""Per-handle re-entrancy (the reference runs one Simulator per
thread, harness.cpp:189-206): four host threads each drive their own
kx_sched handle through upload / tick / fetch / pop rounds concurrently
(ctypes releases the GIL during every library call), and every thread's
decisions and order equal the oracle's for its own inputs."""
import threading

import numpy as np
import pytest

import oracle_ffi as O
import paper_2508_06948_b200 as kx
from helpers import bits, random_queue

pytestmark = pytest.mark.gpu


def one_handle(seed, out):
    try:
        rng = np.random.default_rng(seed)
        n_pools, per_pool, n = 2, 6 + seed % 3, 6000 + 500 * seed
        inst = [kx.InstanceProfile(id=500 - 3 * i, pool=i // per_pool, capacity_tokens=3000.0, max_batch=8)
                for i in range(n_pools * per_pool)]
        s = kx.DeviceScheduler(inst, n_pools=n_pools, queue_capacity=n, max_agents=32)
        q, t = random_queue(rng, n, n_agents=16, n_pools=n_pools, tie_grain=0.1)
        s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
        s.set_scheduler(["kairos", "fcfs", "topo_depth", "kairos"][seed % 4])
        s.upload(q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid)
        got = []
        for r in range(3):
            s.tick(1.0 + r)
            rows, cand = s.fetch_dispatch()
            perm, offs = s.fetch_order()
            got.append((rows, cand, perm, offs))
            s.remove_admitted()
        out[seed] = (inst, q, t, got)
    except Exception as e:  # surfaced by the main thread
        out[seed] = e


def test_four_threads_four_handles(gpu_lib):
    out = {}
    th = [threading.Thread(target=one_handle, args=(sd, out)) for sd in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for seed in range(4):
        assert not isinstance(out[seed], Exception), out[seed]
        inst, q, t, got = out[seed]
        policy = ["kairos", "fcfs", "topo_depth", "kairos"][seed % 4]
        n_pools = 2
        pools = []
        for p in range(n_pools):
            sub = [i for i in inst if i.pool == p]
            pools.append(O.PoolState([i.id for i in sub], [i.capacity_tokens for i in sub],
                                     [i.decode_rate for i in sub], [i.max_batch for i in sub]))
        alive = np.arange(len(q.uid))
        for r, (rows, cand, perm, offs) in enumerate(got):
            sub = O.QueueArrays(q.agent[alive], q.prompt[alive], q.app_start[alive], q.queue_enter[alive],
                                q.msg_key[alive], q.uid[alive])
            ref_perm, ref_offs = O.sort(policy, sub, t, n_pools)
            assert np.array_equal(perm, ref_perm) and np.array_equal(offs, ref_offs), (seed, r)
            gone = []
            for p, ps in enumerate(pools):
                exp, ecand, st = ps.dispatch_round(sub, t, ref_perm[ref_offs[p]:ref_offs[p + 1]], 1.0 + r, p)
                assert st == 0
                assert np.array_equal(rows[p]["uid"], exp["uid"]) and np.array_equal(rows[p]["target"], exp["target"])
                assert np.array_equal(bits(rows[p]["predicted_peak"]), bits(exp["predicted_peak"]))
                assert np.array_equal(bits(cand[p][:, :len(ps.id)]), bits(ecand))
                gone.append(exp["queue_index"][exp["admitted"] == 1])
            alive = np.delete(alive, np.concatenate(gone))
