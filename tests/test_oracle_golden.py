"""The oracle's C restatement against golden fixtures produced by the
unmodified reference (oracle/gen_golden.cpp). CPU only: this pins the oracle
before it is trusted as the checker of the CUDA kernels."""
import numpy as np
import pytest

import kxf
import oracle_ffi as O
from helpers import POLICIES, bits, dispatch_rounds, ledger_expect, order_fixture, round_queue

ORDER = ["order_unit.kxf", "order_ties.kxf", "order_colocated_s1.kxf", "order_colocated_s2.kxf"]


@pytest.mark.parametrize("name", ORDER)
@pytest.mark.parametrize("policy", POLICIES)
def test_order_matches_reference(name, policy):
    d, q, t, n_pools = order_fixture(name)
    perm, offs = O.sort(policy, q, t, n_pools)
    assert np.array_equal(offs, d[f"{policy}.pool_offsets"])
    assert np.array_equal(perm, d[f"{policy}.perm"])


@pytest.mark.parametrize("name", ORDER)
@pytest.mark.parametrize("policy", POLICIES)
def test_order_keys_bit_exact(name, policy):
    d, q, t, _ = order_fixture(name)
    k = O.order_keys(policy, q, t)
    for j in range(3):
        assert np.array_equal(bits(k[j]), bits(d[f"{policy}.k{j}"]))


def test_unit_cases_from_reference_tests():
    # tests/test_priority.cpp:179-234 within order_unit: Router before Math,
    # uid tie 10 < 11, lexicographic "m-10" < "m-9".
    d, q, t, n_pools = order_fixture("order_unit.kxf")
    perm, _ = O.sort("kairos", q, t, n_pools)
    uids = d["uid"][perm].tolist()
    assert uids.index(10) < uids.index(11)
    assert uids.index(12) < uids.index(13)  # m-10 sorts before m-9


@pytest.mark.parametrize("name", ["dispatch_small.kxf", "dispatch_preload.kxf", "dispatch_overload.kxf"])
def test_dispatch_rounds_match_reference(name):
    d = kxf.read(name)
    ids = d["inst_id"]
    pool = O.PoolState(ids, d["inst_cap"], d["inst_k"], d["inst_max_batch"])
    idx_of = {int(x): i for i, x in enumerate(ids)}
    for i, uid, P, t0, T in zip(d["pre_inst"], d["pre_uid"], d["pre_P"], d["pre_t0"], d["pre_T"]):
        j = idx_of[int(i)]
        assert pool.ledgers[j].commit(int(uid), P, float(d["inst_k"][j]), t0, T) == 0
    n_agents = len(d["agent_T"])
    tables = O.TableArrays(np.zeros(n_agents, np.int32), T=d["agent_T"])
    total = 0
    for r, rd in dispatch_rounds(d):
        q = round_queue(rd)
        pool.set_live(rd["live_kv"], rd["running"], rd["waiting"])
        perm, _ = O.sort("fcfs", q, tables, 1)
        rows, cand, st = pool.dispatch_round(q, tables, perm, float(rd["now"][0]))
        assert st == 0
        assert len(rows) == len(rd["dec_uid"]), f"round {r}"
        assert np.array_equal(rows["uid"], rd["dec_uid"])
        assert np.array_equal(rows["target"], rd["dec_target"])
        assert np.array_equal(rows["admitted"], rd["dec_admitted"])
        assert np.array_equal(bits(rows["predicted_peak"]), bits(rd["dec_peak"]))
        assert np.array_equal(bits(cand.ravel()), bits(rd["dec_cand"]))
        assert np.array_equal(pool.suspended, rd["suspended"])
        for j, iid in enumerate(ids):
            got = {s: u for s, u in pool.ledgers[j].slots().items() if u != 0.0}
            exp = ledger_expect(rd, iid)
            assert got.keys() == exp.keys()
            assert all(np.float64(got[s]).view(np.uint64) == np.float64(exp[s]).view(np.uint64) for s in exp)
        for iid, uid, end in zip(rd["fin_inst"], rd["fin_uid"], rd["fin_end"]):
            pool.ledgers[idx_of[int(iid)]].finish(int(uid), float(end))
        total += int(rows["admitted"].sum())
    assert total > 0


@pytest.mark.parametrize("name", ["dp_colocated.kxf", "dp_fanout.kxf", "dp_wide.kxf"])
def test_finalize_matches_reference(name):
    d = kxf.read(name)
    uid, pure, rem = O.finalize(d["wf_offsets"], d["parent"], d["prompt"], d["target"],
                                float(d["prefill_rate"][0]), float(d["decode_rate"][0]))
    assert np.array_equal(uid, d["uid"])
    assert np.array_equal(bits(pure), bits(d["pure_exec"]))
    assert np.array_equal(bits(rem), bits(d["remaining_exec"]))
    assert np.array_equal(bits(rem), bits(d["remaining_by_uid"]))


def test_critical_path_equals_sum_on_chains():
    # tests/test_workload.cpp:114-129: on a chain, remaining = sum of pure_exec.
    off = [0, 4]
    parent = [-1, 0, 1, 2]
    uid, pure, rem = O.finalize(off, parent, [100, 200, 300, 400], [10, 20, 30, 40], 8000.0, 50.0)
    assert rem[0] == pytest.approx(pure.sum())
    assert rem[3] == pure[3]


def test_record_remaining_matches_profiler():
    d = kxf.read("remaining.kxf")
    fin, smp = O.record_remaining(d["rec_offsets"], d["exec_start"], d["exec_end"])
    for a in np.unique(d["samples_agent"]):
        exp = d["samples_sorted"][d["samples_agent"] == a]
        got = np.sort(smp[d["agent"] == a])
        assert np.array_equal(bits(got), bits(exp))


def test_distribution_statistics():
    d = kxf.read("stats.kxf")
    off = d["offsets"]
    for i in range(len(off) - 1):
        v = d["values"][off[i]:off[i + 1]]
        assert bits(O.quantile(v, 0.5)) == bits(d["q50"][i])
        assert bits(O.quantile(v, 0.9)) == bits(d["q90"][i])
        assert bits(O.quantile(v, 0.99)) == bits(d["q99"][i])
        m, fb = O.mode_estimate(v)
        assert bits(m) == bits(d["mode"][i]) and fb == bool(d["median_fallback"][i])
    for i in range(len(d["w1_next"])):
        a = d["values"][off[i]:off[i + 1]]
        b = d["values"][off[i + 1]:off[i + 2]]
        assert bits(O.wasserstein(a, b)) == bits(d["w1_next"][i])
    to = d["table_offsets"]
    for i in range(len(to) - 1):
        got = O.median_anchor_distance(d["table_coords"][to[i]:to[i + 1]], d["table_anchor"][i])
        assert bits(got) == bits(d["table_median"][i])


def test_ledger_unit_values():
    # tests/test_dispatcher.cpp:41-101 golden values.
    L = O.Ledger(0, 0.5, 1000.0)
    assert L.try_place(100.0, 10.0, 0.0, 5.0)[:2] == (True, pytest.approx(150.0))
    L.commit(1, 895.0, 10.0, 1.5, 0.5)
    assert L.slots()[3] == pytest.approx(900.0)
    fits, _, viol = L.try_place(140.0, 10.0, 1.5, 0.5)
    assert not fits and viol == 3
    assert L.commit(2, 140.0, 10.0, 1.5, 0.5) == 2  # logic_error
    L2 = O.Ledger(0, 0.5, 1000.0)
    L2.commit(1, 300.0, 50.0, 0.0, 2.0)
    assert L2.try_place(300.0, 50.0, 0.0, 2.0)[1] == pytest.approx(800.0)
    L2.commit(2, 300.0, 50.0, 0.0, 2.0)
    assert not L2.try_place(300.0, 50.0, 0.0, 2.0)[0]


def test_pairwise_accuracy_matches_reference():
    d = kxf.read("accuracy.kxf")
    off = d["offsets"]
    for t in range(len(off) - 1):
        sl = slice(off[t], off[t + 1])
        for scope_all, key in ((False, "acc_cross"), (True, "acc_all")):
            acc, _ = O.pairwise_accuracy(d["agent"][sl], d["remaining"][sl], d["present"][sl], scope_all)
            exp = d[key][t]
            if np.isnan(exp):
                assert acc is None
            else:
                assert bits(acc) == bits(exp)


def waiting_queue(rd, pre):
    return O.QueueArrays(rd[pre + "agent"], rd[pre + "prompt"], rd[pre + "app_start"], rd[pre + "queue_enter"],
                         rd[pre + "msg_key"], rd[pre + "uid"])


@pytest.mark.parametrize("name", ["dispatch_rr.kxf", "dispatch_static.kxf"])
def test_waiting_rounds_match_reference(name):
    """RoundRobin / StaticThreshold rounds (engine.cpp:259-296): decisions,
    admissions out of the waiting lists and the lists themselves, with the
    lists carried from round to round by the oracle (only the engine's live
    state is reset from the fixture)."""
    d = kxf.read(name)
    ids = d["inst_id"]
    policy = {1: "round_robin", 2: "static_threshold"}[int(d["policy"][0])]
    pool = O.PoolState(ids, d["inst_cap"], d["inst_k"], d["inst_max_batch"])
    depth = d["agent_depth"]
    tables = O.TableArrays(np.zeros(len(depth), np.int32), depth=depth)
    n_adm = 0
    for r, rd in dispatch_rounds(d):
        if r == 0:
            pool.set_waiting(waiting_queue(rd, "w."), rd["w.inst"])
        for i in range(len(ids)):  # the carried lists equal the reference's at round start
            assert np.array_equal(pool.waiting_uids(i), rd["w.uid"][rd["w.inst"] == i]), (r, i)
        pool.set_live(rd["live_kv"], rd["running"])
        q = waiting_queue(rd, "q.")
        perm, _ = O.sort("topo_depth", q, tables, 1)
        rows, adm, st = pool.dispatch_round_waiting(policy, "topo_depth", q, tables, perm, float(rd["now"][0]))
        assert st == 0
        assert np.array_equal(rows["uid"], rd["dec_uid"]), r
        assert np.array_equal(rows["target"], rd["dec_target"]), r
        assert np.array_equal(rows["admitted"], rd["dec_admitted"]), r
        assert np.array_equal(adm["uid"], rd["adm_uid"]), r
        assert np.array_equal(adm["instance"], rd["adm_inst"]), r
        assert np.array_equal(bits(pool.live_kv), bits(rd["end_live_kv"]))
        assert np.array_equal(pool.running, rd["end_running"])
        for i in range(len(ids)):
            assert np.array_equal(pool.waiting_uids(i), rd["end_w.uid"][rd["end_w.inst"] == i]), (r, i)
        n_adm += len(adm)
    assert n_adm > 0


def test_profiler_matches_reference():
    """EmpiricalDistribution restatement vs the reference LatencyProfiler
    (profiler.kxf: sliding 4096 window, doubling checkpoints, W1 convergence,
    take_newly_converged per workflow)."""
    d = kxf.read("profiler.kxf")
    A = int(d["n_agents"][0])
    ex, rm, newly = O.profiler_replay(A, d["off"], d["agent"], d["exec_start"], d["exec_end"])
    assert np.array_equal(newly, d["newly"])
    for kind, dists in (("exec", ex), ("rem", rm)):
        for a in range(A):
            s, tot, cv, last = dists[a].read()
            p = f"{kind}{a}."
            assert np.array_equal(bits(s), bits(d[p + "samples"])), p
            assert tot == int(d[p + "total"][0]) and cv == int(d[p + "converged"][0]), p
            assert bits(last) == bits(d[p + "last"][0]), p
