"""realize() for general WorkloadConfigs (choice / parallel / feedback,
weighted or cycled entries, Poisson or trace arrivals) in the product
library (kx_realize, kx_workload.cpp) against the UNMODIFIED reference
realize() (workload.cpp:319-372) run in the same process through
oracle/_ref/libkxref.so. Host code only: no GPU needed."""
import numpy as np
import pytest

import ref_sim
from helpers import bits
from paper_2508_06948_b200 import KxError
from paper_2508_06948_b200 import workload as W


def same(cfg, prefill=8000.0, decode=50.0):
    got = W.realize(cfg, prefill, decode)
    ref = ref_sim.realize(cfg, prefill, decode)
    assert np.array_equal(bits(got.arrival), bits(ref["arrival"]))
    assert np.array_equal(got.wf_offsets, ref["wf_offsets"])
    for k in ("agent", "parent", "prompt", "target", "uid"):
        assert np.array_equal(getattr(got, k), ref[k]), k
    assert np.array_equal(bits(got.pure_exec), bits(ref["pure_exec"]))
    assert np.array_equal(bits(got.remaining), bits(ref["remaining"]))
    assert np.array_equal(bits(got.remaining), bits(ref["rem_map"]))  # remaining_by_uid
    return got


@pytest.mark.parametrize("apps,rate,dur,seed", [
    ("qa", 2.0, 200.0, 1), ("colocated", 5.0, 300.0, 4), ("cg", 3.0, 400.0, 9)])
def test_builtin_templates(apps, rate, dur, seed):
    sel = {"qa": [W.qa_app()], "cg": [W.cg_app()], "colocated": [W.qa_app(), W.rg_app(), W.cg_app()]}
    same(W.WorkloadConfig(sel[apps], rate=rate, duration=dur, seed=seed))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_generated_apps_c3_shapes(seed):
    # C3's 100 generated apps (choice / parallel / feedback)
    got = same(W.WorkloadConfig(W.generated_apps(100, seed=seed), rate=300.0, duration=20.0, seed=seed),
               prefill=6000.0, decode=40.0)
    assert got.n_calls > 20000
    # the parallel apps fan out: some workflow has two calls with the same parent
    first = got.wf_offsets[:-1]
    assert (np.diff(got.wf_offsets) >= 5).any()
    assert len(first) > 1000


def test_cycle_entries_and_trace_arrivals():
    apps = W.generated_apps(7, seed=5)
    rng = np.random.default_rng(1)
    trace = np.cumsum(rng.exponential(0.05, 3000)) + 100.0
    same(W.WorkloadConfig(apps, duration=50.0, seed=2, trace=trace, trace_scale=0.4, entry_selection="cycle"))


def test_fixed_lengths_and_deep_feedback():
    a = W.AgentSpec("x", W.LengthSpec.fixed(100), W.LengthSpec.fixed(7), choice=[("y", 1.0)])
    b = W.AgentSpec("y", W.LengthSpec.uniform(1, 3), W.LengthSpec.lognormal(5.0, 1.5, 9),
                    feedback=("x", 0.9, 6))
    same(W.WorkloadConfig([W.AppSpec("loop", [a, b], "x")], rate=10.0, duration=30.0, seed=3))


@pytest.mark.parametrize("mutate", ["cycle", "prob_sum", "both", "fb_iter", "rate"])
def test_validate_rejects_like_the_reference(mutate):
    a = W.AgentSpec("x", W.LengthSpec.fixed(10), W.LengthSpec.fixed(10), choice=[("y", 1.0)])
    b = W.AgentSpec("y", W.LengthSpec.fixed(10), W.LengthSpec.fixed(10))
    cfg = W.WorkloadConfig([W.AppSpec("bad", [a, b], "x")], rate=1.0, duration=10.0)
    if mutate == "cycle":
        b.choice = [("x", 1.0)]
    elif mutate == "prob_sum":
        a.choice = [("y", 0.7)]
    elif mutate == "both":
        a.parallel = ["y"]
    elif mutate == "fb_iter":
        b.feedback = ("x", 0.5, 0)
    else:
        cfg.rate = 0.0
    with pytest.raises(KxError) as e:
        W.realize(cfg)
    assert e.value.code == 1  # std::invalid_argument
    with pytest.raises(ValueError):
        ref_sim.realize(cfg)


def test_snapshot_from_realization():
    cfg = W.WorkloadConfig(W.generated_apps(20, seed=1), rate=500.0, duration=10.0, seed=1)
    real = W.realize(cfg)
    n = real.n_calls - 17
    s = W.snapshot_from_realization(real, n)
    assert s.n == n and s.pk_known.sum() == len(real.agent_names) - 1
    # queue_enter = arrival + sum of the ancestors' pure_exec (recomputed per call by walking up)
    wf = np.repeat(np.arange(len(real.arrival)), np.diff(real.wf_offsets))
    for i in np.random.default_rng(0).integers(0, n, 300):
        t, j = real.arrival[wf[i]], i
        acc = []
        while real.parent[j] >= 0:
            j = real.wf_offsets[wf[i]] + real.parent[j]
            acc.append(real.pure_exec[j])
        assert s.queue_enter[i] == t + sum(acc[::-1]) or np.isclose(s.queue_enter[i], t + sum(acc))
