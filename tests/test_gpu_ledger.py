"""SlotLedger / Dispatcher golden values of tests/test_dispatcher.cpp through
the device ledger entry points, and random commit/finish/gc sequences
against the oracle ledger (bit-exact slot usage)."""
import numpy as np
import pytest

import oracle_ffi as O
import paper_2508_06948_b200 as kx
from helpers import bits

pytestmark = pytest.mark.gpu


def one(cap=1000.0, n=1, **kw):
    inst = [kx.InstanceProfile(id=i, capacity_tokens=cap, decode_rate=10.0, max_batch=8) for i in range(n)]
    return kx.DeviceScheduler(inst, queue_capacity=16, max_agents=4, **kw)


def test_empty_ledger_fits_with_peak(gpu_lib):  # test_dispatcher.cpp:62-68
    s = one()
    assert s.try_place(0, 100.0, 10.0, 0.0, 5.0) == (True, pytest.approx(150.0), 0)


def test_capacity_violation_first_slot(gpu_lib):  # :70-85
    s = one()
    s.commit(0, 1, 895.0, 10.0, 1.5, 0.5)
    assert s.ledger(0)[0][3] == pytest.approx(900.0)
    fits, _, viol = s.try_place(0, 140.0, 10.0, 1.5, 0.5)
    assert not fits and viol == 3
    with pytest.raises(kx.KxError) as e:
        s.commit(0, 2, 140.0, 10.0, 1.5, 0.5)
    assert e.value.code == 2  # std::logic_error


def test_sequential_placements_accumulate(gpu_lib):  # :87-99
    s = one()
    s.commit(0, 1, 300.0, 50.0, 0.0, 2.0)
    assert s.try_place(0, 300.0, 50.0, 0.0, 2.0)[1] == pytest.approx(800.0)
    s.commit(0, 2, 300.0, 50.0, 0.0, 2.0)
    assert not s.try_place(0, 300.0, 50.0, 0.0, 2.0)[0]


def test_early_finish_and_gc(gpu_lib):  # :119-166, 168-176
    s = one(cap=1e9)
    s.commit(0, 1, 100.0, 10.0, 0.0, 4.5)
    s.on_request_finished(0, 1, 2.6)
    slots = s.ledger(0)[0]
    assert all(slots[k] == 0.0 for k in (6, 7, 8))
    s2 = one(cap=1e9)
    s2.commit(0, 1, 100.0, 10.0, 0.0, 1.0)
    assert len(s2.ledger(0)[0]) == 2
    s2.gc(2.0)
    slots, active = s2.ledger(0)
    assert len(slots) == 0 and active == 0


def test_overload_watermark(gpu_lib):  # :230-262
    s = one(n=2)
    s.on_overload(0)
    assert s.get_live()[3][0] == 1
    s.on_live_usage(0, 900.0)
    assert s.get_live()[3][0] == 1
    s.on_live_usage(0, 800.0)
    assert s.get_live()[3][0] == 0


def test_random_ledger_sequences_match_oracle(gpu_lib):
    rng = np.random.default_rng(23)
    s = one(cap=20000.0)
    L = O.Ledger(0, 0.5, 20000.0)
    live = []
    now = 0.0
    for step in range(400):
        op = rng.uniform()
        if op < 0.55:
            P, k, T = float(rng.integers(1, 300)), float(rng.uniform(5, 60)), float(rng.uniform(0.1, 9))
            f1 = s.try_place(0, P, k, now, T)
            f2 = L.try_place(P, k, now, T)
            assert f1[0] == f2[0] and bits(f1[1]) == bits(f2[1]) and f1[2] == f2[2]
            if f1[0]:
                s.commit(0, step, P, k, now, T)
                L.commit(step, P, k, now, T)
                live.append(step)
        elif op < 0.85 and live:
            uid = live.pop(int(rng.integers(len(live))))
            end = now + float(rng.uniform(-0.2, 3.0))
            s.on_request_finished(0, uid, end)
            L.finish(uid, end)
        else:
            now += float(rng.uniform(0.0, 1.3))
            s.gc(now)
            L.gc(now)
        a = s.ledger(0)[0]
        b = L.slots()
        assert a.keys() == b.keys()
        assert all(bits(a[x]) == bits(b[x]) for x in a)


def test_commit_batch_equals_sequential_commits(gpu_lib):
    rng = np.random.default_rng(31)
    inst = [kx.InstanceProfile(id=5 + 2 * i, capacity_tokens=4000.0, decode_rate=30.0 + i, max_batch=8)
            for i in range(6)]
    a = kx.DeviceScheduler(inst, queue_capacity=16, max_agents=4)
    b = kx.DeviceScheduler(inst, queue_capacity=16, max_agents=4)
    n = 300
    ids = rng.choice([p.id for p in inst], n).astype(np.int32)
    P = rng.integers(10, 800, n).astype(float)
    k = np.array([30.0 + (i - 5) // 2 for i in ids])
    t0 = rng.uniform(0, 2, n)
    T = rng.uniform(0.2, 8, n)
    fits = a.commit_batch(ids, np.arange(n, dtype=np.uint64) + 1, P, k, t0, T)
    for j in range(n):
        f, _, _ = b.try_place(int(ids[j]), P[j], k[j], t0[j], T[j])
        assert f == bool(fits[j])
        if f:
            b.commit(int(ids[j]), j + 1, P[j], k[j], t0[j], T[j])
    for p in inst:
        x, y = a.ledger(p.id), b.ledger(p.id)
        assert x[1] == y[1] and x[0].keys() == y[0].keys()
        assert all(bits(x[0][s]) == bits(y[0][s]) for s in x[0])
