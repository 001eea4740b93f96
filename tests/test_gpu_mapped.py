"""KX_MEM_HOST_MAPPED uploads (kx_queue_upload): the key columns are copied,
prompt / kept / msg / uid are read in place from pinned host memory. The tick
must decide and order exactly as after a plain upload, including exact-tuple
ties that reach msg and uid, and enqueue / remove_admitted / graph capture
after a mapped upload must see the same queue."""
import numpy as np
import pytest
import torch

import paper_2508_06948_b200 as kx
from helpers import bits, random_queue

pytestmark = pytest.mark.gpu


def make(n_pools=3, per_pool=8, n=30000, seed=5):
    rng = np.random.default_rng(seed)
    q, t = random_queue(rng, n, n_agents=12, n_pools=n_pools, tie_grain=0.25)
    # equal (app_start, queue_enter) pairs: the tie fix must read msg / uid
    q.queue_enter[::7] = q.app_start[::7]
    inst = [kx.InstanceProfile(id=500 - 3 * i, pool=i // per_pool, capacity_tokens=4000.0, max_batch=16)
            for i in range(n_pools * per_pool)]
    return q, t, inst


def sched(q, t, inst, n_pools):
    s = kx.DeviceScheduler(inst, n_pools=n_pools, queue_capacity=2 * len(q.agent), max_agents=16)
    s.set_agent_tables(t.pool, t.pk, t.depth, t.T)
    s.set_scheduler("kairos")
    return s


def pinned(q):
    return [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in
            (q.agent.astype(np.int32), q.prompt.astype(np.int64), q.app_start, q.queue_enter,
             q.msg_key.view(np.int64), q.uid.view(np.int64))]


def result(s, now):
    s.tick(now)  # the tick's full order stays readable (kx_order would start a new round)
    rows, cand = s.fetch_dispatch()
    perm, offs = s.fetch_order()
    return rows, cand, perm, offs


def same(a, b):
    ra, ca, pa, oa = a
    rb, cb, pb, ob = b
    assert np.array_equal(pa, pb) and np.array_equal(oa, ob)
    for x, y, cx, cy in zip(ra, rb, ca, cb):
        assert len(x) == len(y)
        for f in ("uid", "target", "admitted", "queue_index", "agent"):
            assert np.array_equal(x[f], y[f]), f
        assert np.array_equal(bits(x["predicted_peak"]), bits(y["predicted_peak"]))
        assert np.array_equal(bits(cx), bits(cy))


def test_mapped_upload_ticks_like_a_copy(gpu_lib):
    q, t, inst = make()
    a = sched(q, t, inst, 3)
    a.upload(q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid)
    a.checkpoint()
    ref = result(a, 2.0)
    b = sched(q, t, inst, 3)
    cols = pinned(q)
    b.upload(*cols, mapped=True)
    b.checkpoint()
    same(result(b, 2.0), ref)
    # replayed from the same state: identical again
    b.restore()
    same(result(b, 2.0), ref)


def test_mapped_queue_serving_loop(gpu_lib):
    q, t, inst = make(seed=9)
    n0 = 20000
    arr = slice(n0, len(q.agent))
    a = sched(q, t, inst, 3)
    b = sched(q, t, inst, 3)
    a.upload(q.agent[:n0], q.prompt[:n0], q.app_start[:n0], q.queue_enter[:n0], q.msg_key[:n0], q.uid[:n0])
    cols = pinned(q)
    b.upload(*[c[:n0] for c in cols], mapped=True)
    pos = n0
    for rnd in range(3):
        ra = result(a, 1.0 + rnd)
        rb = result(b, 1.0 + rnd)
        same(rb, ra)
        m = int(sum(int(r["admitted"].sum()) for r in ra[0]))
        a.remove_admitted()
        b.remove_admitted()  # a mapped queue is copied to the device first
        k = min(m, len(q.agent) - pos)
        sl = slice(pos, pos + k)
        a.enqueue(q.agent[sl], q.prompt[sl], q.app_start[sl], q.queue_enter[sl], q.msg_key[sl], q.uid[sl])
        b.enqueue(q.agent[sl], q.prompt[sl], q.app_start[sl], q.queue_enter[sl], q.msg_key[sl], q.uid[sl])
        pos += k
        assert a.size() == b.size()


def test_graph_replay_refused_after_mapped_upload(gpu_lib):
    q, t, inst = make(n=5000)
    b = sched(q, t, inst, 3)
    b.upload(q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid)
    b.capture_begin()
    b.tick(1.0)
    b.capture_end()
    cols = pinned(q)
    b.upload(*cols, mapped=True)
    with pytest.raises(kx.KxError):
        b.graph_launch()
