"""K5w on the B200: round_robin / static_threshold dispatch rounds with
device-resident waiting lists (engine.cpp:259-296). Decisions, admissions
out of the waiting lists, the lists themselves and rr_next_ against the
reference fixtures (oracle/gen_golden.cpp) and against the oracle on random
multi-pool cases with every scheduler policy's try_admit comparator."""
import numpy as np
import pytest

import kxf
import oracle_ffi as O
import paper_2508_06948_b200 as kx
from helpers import POLICIES, bits, dispatch_rounds, random_queue

pytestmark = pytest.mark.gpu


def _q(rd, pre):
    return [rd[pre + f] for f in ("agent", "prompt", "app_start", "queue_enter", "msg_key", "uid")]


@pytest.mark.parametrize("name", ["dispatch_rr.kxf", "dispatch_static.kxf"])
def test_waiting_rounds_match_reference_fixture(gpu_lib, name):
    d = kxf.read(name)
    ids = d["inst_id"]
    policy = {1: "round_robin", 2: "static_threshold"}[int(d["policy"][0])]
    inst = [kx.InstanceProfile(id=int(ids[i]), pool=0, capacity_tokens=float(d["inst_cap"][i]),
                               decode_rate=float(d["inst_k"][i]), max_batch=int(d["inst_max_batch"][i]))
            for i in range(len(ids))]
    s = kx.DeviceScheduler(inst, n_pools=1, dispatcher=kx.DispatcherConfig(policy=policy),
                           queue_capacity=4096, max_agents=16)
    depth = d["agent_depth"]
    s.set_agent_tables(np.zeros(len(depth), np.int32), topo_depth=depth)
    s.set_scheduler("topo_depth")
    for r, rd in dispatch_rounds(d):
        if r == 0:
            s.set_waiting(rd["w.inst"], *_q(rd, "w."))
        for i in range(len(ids)):  # lists carried on the device equal the reference's
            assert np.array_equal(s.waiting_uids(i), rd["w.uid"][rd["w.inst"] == i]), (r, i)
        s.upload(*_q(rd, "q."))
        _, _, waiting, _ = s.get_live()
        s.set_live(rd["live_kv"], rd["running"], waiting)
        s.tick(float(rd["now"][0]))
        rows = s.fetch_dispatch()[0][0]
        adm = s.fetch_admissions()[0]
        assert np.array_equal(rows["uid"], rd["dec_uid"]), r
        assert np.array_equal(rows["target"], rd["dec_target"]), r
        assert np.array_equal(rows["admitted"], rd["dec_admitted"]), r
        assert np.all(rows["predicted_peak"] == 0.0)
        assert np.array_equal(adm["uid"], rd["adm_uid"]), r
        assert np.array_equal(adm["instance"], rd["adm_inst"]), r
        live, running, waiting, _ = s.get_live()
        assert np.array_equal(bits(live), bits(rd["end_live_kv"]))
        assert np.array_equal(running, rd["end_running"])
        for i in range(len(ids)):
            assert np.array_equal(s.waiting_uids(i), rd["end_w.uid"][rd["end_w.inst"] == i]), (r, i)
        # popped heads leave the ready queue
        s.remove_admitted()
        assert s.size() == len(rd["q.uid"]) - int(rows["admitted"].sum())


@pytest.mark.parametrize("dpolicy", ["round_robin", "static_threshold"])
@pytest.mark.parametrize("policy", POLICIES)
def test_waiting_multi_pool_matches_oracle(gpu_lib, dpolicy, policy):
    rng = np.random.default_rng(7 + POLICIES.index(policy) + (dpolicy == "round_robin") * 10)
    n_pools, per_pool, n, rounds = 3, 5, 900, 4
    inst = []
    for p in range(n_pools):
        for j in range(per_pool):
            inst.append(kx.InstanceProfile(id=500 - (p * per_pool + j) * 3, pool=p,
                                           capacity_tokens=1500.0 * (0.6 if j % 3 == 2 else 1.0),
                                           decode_rate=50.0, max_batch=3))
    s = kx.DeviceScheduler(inst, n_pools=n_pools, dispatcher=kx.DispatcherConfig(policy=dpolicy),
                           queue_capacity=n, max_agents=64)
    q, t = random_queue(rng, n, n_agents=12, n_pools=n_pools, tie_grain=0.5, msg_space=40)
    q.prompt[:] = rng.integers(1, 700, n)
    s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
    s.set_remaining_table(int(t.view.rem_base), t.rem, t.rem_present)
    s.set_scheduler(policy)
    pools = []
    for p in range(n_pools):
        sub = [i for i in inst if i.pool == p]
        pools.append(O.PoolState([i.id for i in sub], [i.capacity_tokens for i in sub],
                                 [i.decode_rate for i in sub], [i.max_batch for i in sub]))
    # initial waiting lists: a few queued requests already sit on instances
    pre = rng.choice(n, size=60, replace=False)
    alive = np.ones(n, bool)
    alive[pre] = False
    pos = rng.integers(0, n_pools * per_pool, len(pre)).astype(np.int32)
    pos = np.array([i for i in pos])
    # keep each entry in its agent's pool
    pos = np.array([int(t.pool[q.agent[j]]) * per_pool + int(rng.integers(per_pool)) for j in pre], np.int32)
    s.set_waiting(pos, q.agent[pre], q.prompt[pre], q.app_start[pre], q.queue_enter[pre], q.msg_key[pre], q.uid[pre])
    for p, ps in enumerate(pools):
        m = (pos // per_pool) == p
        sel = pre[m]
        ps.set_waiting(O.QueueArrays(q.agent[sel], q.prompt[sel], q.app_start[sel], q.queue_enter[sel],
                                     q.msg_key[sel], q.uid[sel]), pos[m] % per_pool)
    now = 3.0
    for r in range(rounds):
        idx = np.nonzero(alive)[0]
        sub = O.QueueArrays(q.agent[idx], q.prompt[idx], q.app_start[idx], q.queue_enter[idx], q.msg_key[idx],
                            q.uid[idx])
        s.upload(sub.agent, sub.prompt, sub.app_start, sub.queue_enter, sub.msg_key, sub.uid)
        _, _, waiting, _ = s.get_live()
        s.set_live(np.concatenate([ps.live_kv for ps in pools]), np.concatenate([ps.running for ps in pools]),
                   waiting)
        s.tick(now)
        rows = s.fetch_dispatch()[0]
        adm = s.fetch_admissions()
        perm, offs = O.sort(policy, sub, t, n_pools)
        _, _, waiting, _ = s.get_live()
        for p, ps in enumerate(pools):
            exp, eadm, st = ps.dispatch_round_waiting(dpolicy, policy, sub, t, perm[offs[p]:offs[p + 1]], now,
                                                      pool_index=p)
            assert st == 0
            for f in ["uid", "target", "admitted", "queue_index"]:
                assert np.array_equal(rows[p][f], exp[f]), (r, p, f)
            for f in ["uid", "instance", "queue_index"]:
                assert np.array_equal(adm[p][f], eadm[f]), (r, p, f)
            assert np.array_equal(waiting[p * per_pool:(p + 1) * per_pool], ps.waiting)
            for j in range(per_pool):
                assert np.array_equal(s.waiting_uids(p * per_pool + j), ps.waiting_uids(j)), (r, p, j)
            alive[idx[exp["queue_index"][exp["admitted"] == 1]]] = False
        assert np.array_equal(s.rr_next(), [ps.rr_next % per_pool for ps in pools])
        for ps in pools:  # engine side: some requests finish
            ps.running[:] = np.maximum(ps.running - rng.integers(0, 3, per_pool), 0)
            ps.live_kv[:] = np.maximum(ps.live_kv * rng.uniform(0.2, 0.9, per_pool), 0.0)
        now += 0.7


def test_waiting_capacity_is_reported(gpu_lib):
    inst = [kx.InstanceProfile(id=1, pool=0, capacity_tokens=100.0, max_batch=1)]
    s = kx.DeviceScheduler(inst, dispatcher=kx.DispatcherConfig(policy="round_robin"), queue_capacity=4096,
                           max_agents=4)
    s.set_agent_tables(np.zeros(1, np.int32))
    s.set_scheduler("fcfs")
    n = 1100  # > the default 1024 waiting entries per instance
    s.upload(np.zeros(n, np.int32), np.full(n, 500), np.arange(n, dtype=float), np.arange(n, dtype=float),
             np.arange(n, dtype=np.uint64), np.arange(1, n + 1, dtype=np.uint64))
    s.tick(1.0)
    with pytest.raises(kx.KxError):
        s.fetch_dispatch()
