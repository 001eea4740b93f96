"""K6 on the B200: whole replica simulations against the UNMODIFIED reference
Simulator (engine.cpp:85-486) on identical realize() outputs. Completion
order, every per-call time, counters and metric inputs are bit-exact."""
import numpy as np
import pytest

import ref_sim
from helpers import bits
from paper_2508_06948_b200 import DispatcherConfig, InstanceProfile
from paper_2508_06948_b200 import engine as E

pytestmark = pytest.mark.gpu

DEPTH = np.array([2, 1, 1, 2, 1, 5, 4, 3, 2, 1], np.int32)


def insts(n, cap=3000.0, k=50.0, prefill=8000.0, mb=8):
    return [InstanceProfile(id=10 + 3 * i, capacity_tokens=cap * (1.0 if i % 2 == 0 else 0.9),
                            decode_rate=k if i % 3 else k * 0.8, prefill_rate=prefill, max_batch=mb)
            for i in range(n)]


CASES = [
    # apps, rate, duration, instances, scheduler, dispatcher, recompute
    ("qa", 3.0, 120.0, insts(4), "fcfs", DispatcherConfig("round_robin"), 1.0),
    ("colocated", 4.0, 150.0, insts(4), "fcfs", DispatcherConfig("time_slot", oracle_expected_time=True), 1.0),
    ("colocated", 6.0, 120.0, insts(3, cap=1500.0), "topo_depth", DispatcherConfig("static_threshold"), 1.0),
    ("colocated", 8.0, 100.0, insts(4, cap=1800.0, mb=12), "oracle",
     DispatcherConfig("time_slot", oracle_expected_time=True), 0.5),
    ("cg", 3.0, 120.0, insts(2, cap=1400.0, mb=16), "fcfs", DispatcherConfig("round_robin"), 0.25),
]


def compare(dev, ref, b, r, c0, w0):
    n = int(ref["n_calls"])
    nw = int(ref["n_wf"])
    assert int(dev["counts"][r][0]) == n and int(dev["counts"][r][1]) == nw
    order = dev["call_order"][c0:c0 + n]
    assert np.array_equal(b["uid"][order], ref["uid"][:n]), "completion order"
    assert np.array_equal(bits(dev["exec_start"][c0:c0 + n]), bits(ref["exec_start"][:n]))
    assert np.array_equal(bits(dev["exec_end"][c0:c0 + n]), bits(ref["exec_end"][:n]))
    # per-call fields are indexed by call on the device, by completion on the reference
    assert np.array_equal(bits(dev["first_enqueue"][order]), bits(ref["first_enqueue"][:n]))
    assert np.array_equal(bits(dev["queue_seconds"][order]), bits(ref["queue_seconds"][:n]))
    assert np.array_equal(dev["episodes"][order], ref["episodes"][:n])
    assert np.array_equal(dev["preemptions"][order], ref["preemptions"][:n])
    wo = dev["wf_order"][w0:w0 + nw]
    assert np.array_equal(wo - w0, ref["wf_index"][:nw])
    assert np.array_equal(bits(dev["wf_finish"][wo]), bits(ref["wf_finish"][:nw]))
    assert np.array_equal(dev["wf_output_tokens"][wo], ref["wf_output_tokens"][:nw])
    assert np.array_equal(bits(dev["scalars"][r][:8]), bits(ref["scalars"][:8]))
    # K7: compute_metrics on the device vs the reference (metrics.cpp:13-88)
    m = dev["metrics"][r]
    rs = ref["scalars"]
    pairs = [(2, 8), (3, 9), (4, 10), (5, 11), (6, 12), (7, 13), (8, 14), (11, 15), (13, 16), (12, 17)]
    for mi, ri in pairs:
        assert bits(m[mi]) == bits(rs[ri]), (mi, m[mi], rs[ri])


@pytest.mark.parametrize("case", range(len(CASES)))
def test_replica_engine_matches_reference_simulator(gpu_lib, case):
    apps, rate, dur, inst, sched, disp, rf = CASES[case]
    reals = [E.realize(apps, rate, dur, seed) for seed in (1, 2, 3)]
    b = E.concat(reals)
    dev = E.run_replicas(b, inst, sched, disp, topo_depth=DEPTH, recompute_fraction=rf)
    for r, rz in enumerate(reals):
        one = dict(rz)
        one["prompt"], one["target"] = rz["prompt"], rz["target"]
        ref = ref_sim.run(one, inst, sched, disp, DEPTH, recompute=rf)
        compare(dev, ref, b, r, int(b["wf_offsets"][b["wf_base"][r]]), int(b["wf_base"][r]))


def test_engine_reports_the_reference_livelock(gpu_lib):
    # prompt (<= 240) > (1 - 0.85) * cap: the reference's dispatch_loop
    # would suspend/resume the same instance forever.
    b = E.concat([E.realize("colocated", 8.0, 100.0, 1)])
    with pytest.raises(Exception) as e:
        E.run_replicas(b, insts(4, cap=1400.0, mb=12), "oracle",
                       DispatcherConfig("time_slot", oracle_expected_time=True))
    assert getattr(e.value, "code", None) == 6


def test_engine_rejects_unsupported_configs(gpu_lib):
    b = E.concat([E.realize("qa", 1.0, 20.0, 1)])
    with pytest.raises(Exception):  # agent index outside the agent table
        E.run_replicas(b, insts(2), "fcfs", DispatcherConfig("round_robin"), n_agents=2,
                       topo_depth=np.ones(2, np.int32))
    with pytest.raises(Exception):  # agent_order is not a permutation
        E.run_replicas(b, insts(2), "kairos", DispatcherConfig("time_slot"), agent_order=np.zeros(10))
