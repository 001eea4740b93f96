"""K6 with the KairosScheduler's online priority-table rebuilds
(scheduler.cpp:5-24: W1 matrix + classical MDS over converged agents) and
profile-based expected times (engine.cpp:177-185, ProfilerSnapshot's
mode_estimate), both on the device, against the UNMODIFIED reference
Simulator on identical realize() outputs: completion order, every per-call
time, counters, metrics and the final priority table bit-exact."""
import numpy as np
import pytest

import ref_sim
from helpers import bits
from paper_2508_06948_b200 import DispatcherConfig
from paper_2508_06948_b200 import engine as E
from test_gpu_engine import DEPTH, compare, insts

pytestmark = pytest.mark.gpu

CASES = [
    # apps, rate, duration, instances, scheduler, dispatcher, recompute, rebuild interval
    ("colocated", 4.0, 150.0, insts(4), "kairos", DispatcherConfig("time_slot"), 1.0, 0),
    ("colocated", 6.0, 400.0, insts(4), "kairos", DispatcherConfig("time_slot"), 1.0, 0),
    ("colocated", 6.0, 200.0, insts(4), "kairos", DispatcherConfig("round_robin"), 1.0, 0),
    ("colocated", 6.0, 160.0, insts(3, cap=1500.0), "kairos", DispatcherConfig("static_threshold"), 0.5, 0),
    ("colocated", 5.0, 150.0, insts(4), "kairos", DispatcherConfig("time_slot", oracle_expected_time=True), 1.0, 0),
    ("colocated", 5.0, 200.0, insts(4, cap=1800.0, mb=12), "fcfs", DispatcherConfig("time_slot"), 1.0, 0),
    ("colocated", 5.0, 150.0, insts(4), "topo_depth", DispatcherConfig("time_slot", default_expected_time=2.0), 1.0, 0),
    ("rg", 4.0, 150.0, insts(2), "oracle", DispatcherConfig("time_slot"), 0.25, 0),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_online_profiles_match_reference_simulator(gpu_lib, case):
    apps, rate, dur, inst, sched, disp, rf, interval = CASES[case]
    reals = [E.realize(apps, rate, dur, seed) for seed in (1, 2, 3)]
    b = E.concat(reals)
    dev = E.run_replicas(b, inst, sched, disp, topo_depth=DEPTH, recompute_fraction=rf,
                         rebuild_interval=interval)
    rebuilt = 0
    for r, rz in enumerate(reals):
        ref = ref_sim.run(dict(rz), inst, sched, disp, DEPTH, recompute=rf)
        compare(dev, ref, b, r, int(b["wf_offsets"][b["wf_base"][r]]), int(b["wf_base"][r]))
        if sched == "kairos":
            assert int(dev["table_versions"][r]) == ref["table_version"]
            assert np.array_equal(bits(dev["priority_keys"][r]), bits(ref["priority_keys"]))
            rebuilt += ref["table_version"]
    if sched == "kairos":
        assert rebuilt > 0, "case never rebuilt a priority table"


def test_kairos_rebuild_interval(gpu_lib):
    # a short interval rebuilds every few completions (scheduler.cpp:8)
    reals = [E.realize("colocated", 4.0, 150.0, 7)]
    b = E.concat(reals)
    dev = E.run_replicas(b, insts(4), "kairos", DispatcherConfig("time_slot"), topo_depth=DEPTH,
                         rebuild_interval=16)
    dev256 = E.run_replicas(b, insts(4), "kairos", DispatcherConfig("time_slot"), topo_depth=DEPTH)
    assert int(dev["table_versions"][0]) > int(dev256["table_versions"][0])


def test_c5_shape_replicas_match_reference_simulator(gpu_lib):
    """BASELINE C5's replica shape: the co-located workload at
    12 workflows/s for 720 s on 16 instances, Kairos + profiler T, two
    replicas of a sweep, each bit-exact against the reference Simulator."""
    from paper_2508_06948_b200 import InstanceProfile
    inst = [InstanceProfile(id=i, capacity_tokens=3000.0, decode_rate=50.0, prefill_rate=8000.0, max_batch=8)
            for i in range(16)]
    disp = DispatcherConfig("time_slot")
    reals = [E.realize("colocated", 12.0, 720.0, seed) for seed in (1, 5)]
    b = E.concat(reals)
    dev = E.run_replicas(b, inst, "kairos", disp, topo_depth=DEPTH)
    for r, rz in enumerate(reals):
        ref = ref_sim.run(dict(rz), inst, "kairos", disp, DEPTH)
        assert ref["n_calls"] > 20000
        compare(dev, ref, b, r, int(b["wf_offsets"][b["wf_base"][r]]), int(b["wf_base"][r]))
        assert int(dev["table_versions"][r]) == ref["table_version"] > 0
        assert np.array_equal(bits(dev["priority_keys"][r]), bits(ref["priority_keys"]))
