"""K5 on the B200: the reference's dispatch decisions (decision-log rows:
target, predicted_peak bits, candidate_peaks bits), suspension and ledger
state, replayed round by round; plus random multi-pool cases vs the oracle."""
import ctypes

import numpy as np
import pytest

import kxf
import oracle_ffi as O
import paper_2508_06948_b200 as kx
from helpers import bits, dispatch_rounds, ledger_expect, random_queue, round_queue

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["dispatch_small.kxf", "dispatch_preload.kxf", "dispatch_overload.kxf"])
def test_dispatch_matches_reference_fixture(gpu_lib, name):
    d = kxf.read(name)
    ids = d["inst_id"]
    inst = [kx.InstanceProfile(id=int(ids[i]), pool=0, capacity_tokens=float(d["inst_cap"][i]),
                               decode_rate=float(d["inst_k"][i]), max_batch=int(d["inst_max_batch"][i]))
            for i in range(len(ids))]
    s = kx.DeviceScheduler(inst, n_pools=1, queue_capacity=4096, max_agents=16)
    n_agents = len(d["agent_T"])
    s.set_agent_tables(np.zeros(n_agents, np.int32), expected_T=d["agent_T"])
    s.set_scheduler("fcfs")
    for i, uid, P, t0, T in zip(d["pre_inst"], d["pre_uid"], d["pre_P"], d["pre_t0"], d["pre_T"]):
        k = float(d["inst_k"][list(ids).index(int(i))])
        s.commit(int(i), int(uid), P, k, t0, T)
    for r, rd in dispatch_rounds(d):
        q = round_queue(rd)
        s.upload(q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid)
        s.set_live(rd["live_kv"], rd["running"], rd["waiting"])
        s.tick(float(rd["now"][0]))
        rows, cand = s.fetch_dispatch()
        rows, cand = rows[0], cand[0]
        assert len(rows) == len(rd["dec_uid"]), f"round {r}"
        assert np.array_equal(rows["uid"], rd["dec_uid"]), f"round {r}"
        assert np.array_equal(rows["target"], rd["dec_target"])
        assert np.array_equal(rows["admitted"], rd["dec_admitted"])
        assert np.array_equal(bits(rows["predicted_peak"]), bits(rd["dec_peak"]))
        assert np.array_equal(bits(cand[:, :len(ids)].ravel()), bits(rd["dec_cand"]))
        live, running, waiting, susp = s.get_live()
        assert np.array_equal(susp, rd["suspended"])
        for iid in ids:
            got = {k: v for k, v in s.ledger(int(iid))[0].items() if v != 0.0}
            exp = ledger_expect(rd, iid)
            assert got.keys() == exp.keys(), (r, iid)
            assert all(bits(got[k]) == bits(exp[k]) for k in exp)
        for iid, uid, end in zip(rd["fin_inst"], rd["fin_uid"], rd["fin_end"]):
            s.on_request_finished(int(iid), int(uid), float(end))


def build_pools(rng, n_pools, per_pool, cap=3000.0, max_batch=8, uniform=False):
    inst, ids = [], []
    for p in range(n_pools):
        for j in range(per_pool):
            iid = 1000 - (p * per_pool + j) * 7  # ids decreasing: tie-break by id, not index
            k = 50.0 if uniform else 40.0 + 10.0 * (j % 2)
            inst.append(kx.InstanceProfile(id=iid, pool=p, capacity_tokens=cap * (0.8 if j % 3 == 2 else 1.0),
                                           decode_rate=k, max_batch=max_batch))
            ids.append(iid)
    return inst


# Tick modes: "overlap" = top-K order prefix + dispatch on a side stream while
# the full sort runs (the default for <= 32 instances per pool), "serial" =
# order then dispatch, "short1"/"short5" = overlap with prefixes capped at 1
# / 5 heads so every round resumes over the full order (phase 2).
TICK_MODES = {"overlap": {}, "serial": {"KX_NO_OVERLAP": "1"}, "short1": {"KX_TOPK_NEED": "1"},
              "short5": {"KX_TOPK_NEED": "5"}}


def set_mode(monkeypatch, mode):
    for k in ("KX_NO_OVERLAP", "KX_TOPK_NEED"):
        monkeypatch.delenv(k, raising=False)
    for k, v in TICK_MODES[mode].items():
        monkeypatch.setenv(k, v)


MULTI_POOL_CASES = [(1, 4, 500, 4, 0, 8), (8, 32, 20000, 3, 0, 8), (3, 17, 5000, 5, 0, 8),
                    (2, 8, 6000, 3, 1, 8), (2, 8, 6000, 3, 2, 8)]
# pools of more than 32 instances (C3 has 64): the shared-memory ring layout
# (33, 64) and the global-ring layout (256), max_batch 8 and 64
WIDE_POOL_CASES = [(2, 33, 8000, 3, 0, 8), (1, 64, 20000, 3, 0, 8), (1, 64, 30000, 2, 0, 64),
                   (2, 48, 12000, 3, 1, 16), (1, 256, 40000, 2, 0, 8), (1, 256, 40000, 2, 0, 64)]


@pytest.mark.parametrize("mode", list(TICK_MODES))
@pytest.mark.parametrize("n_pools,per_pool,n,rounds,ties,max_batch", MULTI_POOL_CASES + WIDE_POOL_CASES)
def test_dispatch_multi_pool_matches_oracle(gpu_lib, monkeypatch, mode, n_pools, per_pool, n, rounds, ties,
                                            max_batch):
    if per_pool > 32 and mode != "overlap":
        pytest.skip("pools of > 32 instances always dispatch after the full order")
    run_multi_pool(monkeypatch, mode, n_pools, per_pool, n, rounds, ties, max_batch, uniform=False)


# Uniform decode rates: pools of <= 32 instances take the register-resident
# resolver (kx_dispatch.cu, rr), 33-64 the two-warp one (rr2); both also
# decide the round's last head (no instance fits). Spans longer than their 16
# slots (T up to 8 s at 0.5 s slots), overloads and full active tables take
# the exact path: these cases are known to reach it.
EXACT_PATH_CASES = {(3, 17, 5000, 5, 0, 8), (2, 32, 12000, 3, 0, 64), (1, 64, 20000, 3, 0, 8),
                    (2, 48, 12000, 3, 1, 16)}


@pytest.mark.parametrize("mode", ["overlap", "serial", "short1"])
@pytest.mark.parametrize("n_pools,per_pool,n,rounds,ties,max_batch",
                         MULTI_POOL_CASES + [(2, 32, 12000, 3, 0, 64), (4, 16, 8000, 4, 0, 2),
                                             # two resolver warps (33-64 instances)
                                             (2, 33, 8000, 3, 0, 8), (1, 64, 20000, 3, 0, 8),
                                             (1, 64, 30000, 2, 0, 64), (2, 48, 12000, 3, 1, 16)])
def test_dispatch_register_resolver_matches_oracle(gpu_lib, monkeypatch, mode, n_pools, per_pool, n, rounds, ties,
                                                   max_batch):
    cnt = (ctypes.c_uint64 * 2)()
    gpu_lib.kx_debug_dispatch_counts(cnt, 1)
    run_multi_pool(monkeypatch, mode, n_pools, per_pool, n, rounds, ties, max_batch, uniform=True)
    gpu_lib.kx_debug_dispatch_counts(cnt, 1)
    assert cnt[0] > 0, "the register resolver took no decision"
    if (n_pools, per_pool, n, rounds, ties, max_batch) in EXACT_PATH_CASES:
        assert cnt[1] > 0, "no head took the exact path (long spans / overloads are expected)"


def run_multi_pool(monkeypatch, mode, n_pools, per_pool, n, rounds, ties, max_batch, uniform):
    set_mode(monkeypatch, mode)
    rng = np.random.default_rng(n_pools * 100 + per_pool + max_batch + (7 if uniform else 0))
    inst = build_pools(rng, n_pools, per_pool, max_batch=max_batch, uniform=uniform)
    s = kx.DeviceScheduler(inst, n_pools=n_pools, queue_capacity=n, max_agents=64)
    q, t = random_queue(rng, n, n_agents=30, n_pools=n_pools)
    # prompts up to 400 against capacities 2400-3000: some heads overload
    # their target (suspension + retry, engine.cpp:254-258)
    q.prompt[:] = rng.integers(1, 400, n)
    q.view.prompt = q.prompt.ctypes.data
    if ties:  # > kTopKMax equal compact keys per pool: a prefix cut below them (1)
        t.pk[:] = 1.0  # or none at all (2, the whole pool waits for the full order)
        q.app_start[:] = np.where(rng.random(n) < 0.9, 0.25, q.app_start)
        if ties == 2:
            q.app_start[:] = np.maximum(q.app_start, 0.25)
    s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
    s.set_scheduler("kairos")
    pools = []
    for p in range(n_pools):
        sub = [i for i in inst if i.pool == p]
        pools.append(O.PoolState([i.id for i in sub], [i.capacity_tokens for i in sub],
                                 [i.decode_rate for i in sub], [i.max_batch for i in sub]))
    # preload ledgers identically on both sides
    for p, ps in enumerate(pools):
        for j in range(3 * len(ps.id)):
            i = int(rng.integers(len(ps.id)))
            P, t0, T = float(rng.integers(20, 500)), float(rng.uniform(0, 1)), float(rng.uniform(0.5, 6))
            fits, _, _ = ps.ledgers[i].try_place(P, ps.k[i], t0, T)
            if fits:
                ps.ledgers[i].commit(9_000_000 + p * 1000 + j, P, ps.k[i], t0, T)
                s.commit(int(ps.id[i]), 9_000_000 + p * 1000 + j, P, float(ps.k[i]), t0, T)
    now = 1.0
    alive = np.ones(n, bool)
    for r in range(rounds):
        idx = np.nonzero(alive)[0]
        sub = O.QueueArrays(q.agent[idx], q.prompt[idx], q.app_start[idx], q.queue_enter[idx],
                            q.msg_key[idx], q.uid[idx])
        s.upload(sub.agent, sub.prompt, sub.app_start, sub.queue_enter, sub.msg_key, sub.uid)
        live = np.concatenate([ps.live_kv for ps in pools])
        running = np.concatenate([ps.running for ps in pools])
        s.set_live(live, running, np.zeros_like(running))
        s.tick(now)
        rows, cand = s.fetch_dispatch()
        perm, offs = O.sort("kairos", sub, t, n_pools)
        for p, ps in enumerate(pools):
            exp, ecand, st = ps.dispatch_round(sub, t, perm[offs[p]:offs[p + 1]], now, pool_index=p)
            assert st == 0
            got = rows[p]
            assert len(got) == len(exp)
            for f in ["uid", "target", "admitted", "queue_index"]:
                assert np.array_equal(got[f], exp[f]), f
            assert np.array_equal(bits(got["predicted_peak"]), bits(exp["predicted_peak"]))
            assert np.array_equal(bits(cand[p][:, :len(ps.id)]), bits(ecand))
            for j, iid in enumerate(ps.id):
                a = {k: v for k, v in s.ledger(int(iid))[0].items() if v != 0.0}
                b = {k: v for k, v in ps.ledgers[j].slots().items() if v != 0.0}
                assert a.keys() == b.keys() and all(bits(a[k]) == bits(b[k]) for k in a)
            # dispatched requests leave the queue
            gone = exp["queue_index"][exp["admitted"] == 1]
            alive[idx[gone]] = False
        # engine side: some requests finish, tokens grow
        for p, ps in enumerate(pools):
            ps.running[:] = np.maximum(ps.running - rng.integers(0, 3, len(ps.id)), 0)
            ps.live_kv[:] = np.maximum(ps.live_kv * rng.uniform(0.3, 1.1, len(ps.id)), 0.0)
        now += float(rng.uniform(0.3, 1.2))
        # gc happens only at the end of each round on both sides


def test_livelock_is_reported(gpu_lib):
    # cap 1000, prompt 300 > (1 - 0.85) * cap -> the reference spins.
    inst = [kx.InstanceProfile(id=0, capacity_tokens=1000.0, max_batch=8)]
    s = kx.DeviceScheduler(inst, queue_capacity=8, max_agents=2)
    s.set_agent_tables([0], expected_T=[1.0])
    s.set_scheduler("fcfs")
    s.upload([0], [300], [0.0], [0.0], [0], [1])
    s.set_live([800.0], [1], [0])
    s.tick(1.0)
    with pytest.raises(kx.KxError) as e:
        s.fetch_dispatch()
    assert e.value.code == 6


def test_remove_admitted_compacts_queue(gpu_lib):
    rng = np.random.default_rng(3)
    inst = [kx.InstanceProfile(id=i, capacity_tokens=5000.0, max_batch=4) for i in range(3)]
    s = kx.DeviceScheduler(inst, queue_capacity=1000, max_agents=8)
    q, t = random_queue(rng, 1000, n_agents=5, n_pools=1)
    s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
    s.set_scheduler("fcfs")
    s.upload(q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid)
    s.tick(0.5)
    rows, _ = s.fetch_dispatch()
    adm = rows[0]["queue_index"][rows[0]["admitted"] == 1]
    assert len(adm) == 12
    s.remove_admitted()
    assert s.size() == 1000 - 12
    keep = np.setdiff1d(np.arange(1000), adm)
    s.order()
    perm, _ = s.fetch_order()
    sub = O.QueueArrays(q.agent[keep], q.prompt[keep], q.app_start[keep], q.queue_enter[keep],
                        q.msg_key[keep], q.uid[keep])
    assert np.array_equal(perm, O.sort("fcfs", sub, t, 1)[0])


@pytest.mark.parametrize("mode", ["overlap", "short1"])
def test_checkpoint_restore_replays_identically(gpu_lib, monkeypatch, mode):
    set_mode(monkeypatch, mode)
    rng = np.random.default_rng(9)
    inst = build_pools(rng, 2, 6)
    s = kx.DeviceScheduler(inst, n_pools=2, queue_capacity=3000, max_agents=16)
    q, t = random_queue(rng, 3000, n_agents=10, n_pools=2)
    s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
    s.upload(q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid)
    s.checkpoint()
    s.tick(2.0)
    a = s.fetch_dispatch()[0]
    s.restore()
    s.tick(2.0)
    b = s.fetch_dispatch()[0]
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_graph_replay_matches_direct_tick(gpu_lib):
    # kx_graph_*: the captured step (restore + tick) replays the same kernels
    rng = np.random.default_rng(17)
    inst = build_pools(rng, 3, 8)
    s = kx.DeviceScheduler(inst, n_pools=3, queue_capacity=20000, max_agents=32)
    q, t = random_queue(rng, 20000, n_agents=20, n_pools=3)
    s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
    s.set_scheduler("kairos")
    s.upload(q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid)
    s.checkpoint()
    s.restore()
    s.tick(3.0)
    ref_rows, ref_cand = s.fetch_dispatch()
    ref_perm, ref_offs = s.fetch_order()
    s.capture_begin()
    s.restore()
    s.tick(3.0)
    s.capture_end()
    for _ in range(3):
        s.graph_launch()
        s.synchronize()
        rows, cand = s.fetch_dispatch()
        perm, offs = s.fetch_order()
        assert np.array_equal(perm, ref_perm) and np.array_equal(offs, ref_offs)
        for a, b in zip(rows, ref_rows):
            assert np.array_equal(a, b)
        for a, b in zip(cand, ref_cand):
            assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("policy,graph", [("kairos", False), ("oracle", False), ("kairos", True)])
def test_serving_loop_pop_and_enqueue(gpu_lib, policy, graph):
    # ReadyQueue across rounds: the placed prefix is popped (vector::erase,
    # order kept) and new arrivals are pushed back; the device queue (many
    # 8192-element compaction chunks) must order exactly like the same
    # logical queue sorted by the oracle.
    rng = np.random.default_rng(31)
    n0, n_new, pools = 120_000, 3_000, 3
    q, t = random_queue(rng, n0 + 4 * n_new, n_agents=12, n_pools=pools, tie_grain=0.25)
    inst = [kx.InstanceProfile(id=i, pool=i // 3, capacity_tokens=6000.0, max_batch=64)
            for i in range(3 * pools)]
    s = kx.DeviceScheduler(inst, n_pools=pools, queue_capacity=n0 + 4 * n_new, max_agents=16)
    s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
    if t.rem is not None:
        s.set_remaining_table(t.view.rem_base, t.rem, t.rem_present)
    s.set_scheduler(policy)
    cols = [q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid]
    s.upload(*[c[:n0] for c in cols])
    if graph:  # a captured graph pins the queue's addresses: the pop copies back
        s.checkpoint()
        s.capture_begin()
        s.restore()
        s.tick(5.0)
        s.capture_end()
    logical = np.arange(n0)  # indices into q, in queue order
    nxt = n0
    for rnd in range(4):
        s.restore() if rnd else s.checkpoint()
        s.tick(5.0)
        rows, _ = s.fetch_dispatch()
        gone = np.concatenate([r["queue_index"][r["admitted"] == 1] for r in rows])
        assert len(gone) > 0
        s.remove_admitted()
        logical = np.delete(logical, gone)
        s.enqueue(*[c[nxt:nxt + n_new] for c in cols])
        logical = np.concatenate([logical, np.arange(nxt, nxt + n_new)])
        nxt += n_new
        assert s.size() == len(logical)
        s.order()
        perm, offs = s.fetch_order()
        sub = O.QueueArrays(*[c[logical] for c in cols])
        ref_perm, ref_offs = O.sort(policy, sub, t, pools)
        assert np.array_equal(offs, ref_offs) and np.array_equal(perm, ref_perm), f"round {rnd}"


def test_graph_replay_after_pop_needs_recapture(gpu_lib):
    # A captured step carries the queue size of the capture: after a pop the
    # replay is refused; a pop + enqueue of the same count keeps the size and
    # the addresses, so the replay orders the new contents.
    rng = np.random.default_rng(23)
    inst = build_pools(rng, 2, 6)
    n0 = 5000
    q, t = random_queue(rng, n0 + 400, n_agents=10, n_pools=2)
    s = kx.DeviceScheduler(inst, n_pools=2, queue_capacity=n0 + 400, max_agents=16)
    s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
    s.set_scheduler("kairos")
    cols = [q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid]
    s.upload(*[c[:n0] for c in cols])
    s.checkpoint()
    s.capture_begin()
    s.restore()
    s.tick(2.0)
    s.capture_end()
    s.graph_launch()
    rows, _ = s.fetch_dispatch()  # a replay leaves a fetchable round
    gone = np.concatenate([r["queue_index"][r["admitted"] == 1] for r in rows])
    assert len(gone) > 0
    s.remove_admitted()
    with pytest.raises(kx.KxError) as e:
        s.graph_launch()
    assert e.value.code == 2
    s.enqueue(*[c[n0:n0 + len(gone)] for c in cols])
    logical = np.concatenate([np.delete(np.arange(n0), gone), np.arange(n0, n0 + len(gone))])
    s.graph_launch()
    s.synchronize()
    perm, offs = s.fetch_order()
    ref_perm, ref_offs = O.sort("kairos", O.QueueArrays(*[c[logical] for c in cols]), t, 2)
    assert np.array_equal(perm, ref_perm) and np.array_equal(offs, ref_offs)
