"""Parity at the benchmark's own configurations (BASELINE.json C1-C4, in
their stated shapes, built by workload.build_workload exactly as bench.py
builds them): every decision of one tick (uid, target, admitted,
predicted_peak bits, candidate_peaks bits) and the full per-pool queue order
against the UNMODIFIED reference (Dispatcher with the same pre-loaded
ledgers + ReadyQueue comparator sort, oracle/_ref/libkxref.so) on the same
inputs. C4 is the headline: 16M requests, 8 pools x 32 instances,
max_batch 64, capacity 20000; C3 dispatches 64 instances in one pool."""
import numpy as np
import pytest

import bench
from paper_2508_06948_b200 import workload as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config", ["C1", "C2", "C3", "C4"])
def test_config_tick_matches_reference(gpu_lib, config):
    w = W.build_workload(config, 0, arrivals=1024)
    s = bench.make_sched(w, 0)
    snap = w.snap
    s.upload(snap.agent, snap.prompt, snap.app_start, snap.queue_enter, snap.msg_key, snap.uid)
    s.restore()
    s.tick(w.now)
    rows, cand = s.fetch_dispatch()
    s.order()
    perm, offs = s.fetch_order()
    L = bench._ref_lib()
    ref = bench.RefPools(L, w, list(range(snap.n_pools)))
    ref.record(True)
    ref.tick(min(snap.n_pools, 16), w.now)
    total = 0
    for j, p in enumerate(ref.pools):
        n_ref, bad = bench.compare_decisions(ref, j, rows[p], cand[p])
        assert bad == 0, f"pool {p}: {bad} of {n_ref} decisions differ"
        assert n_ref == len(rows[p]) and n_ref > 0
        total += n_ref
        ro = ref.order(j)
        go = snap.uid[perm[offs[p]:offs[p + 1]]]
        assert len(ro) == len(go) and np.array_equal(ro, go), f"pool {p}: queue order differs"
    # placements fill the free batch slots: the round ran to its end
    admitted = sum(int(r["admitted"].sum()) for r in rows)
    free = sum(max(0, i.max_batch - int(r)) for i, r in zip(w.insts, w.running))
    assert 0 < admitted <= free
    # a second tick from the restored state replays the same decisions
    s.restore()
    s.tick(w.now)
    rows2, _ = s.fetch_dispatch()
    for a, b in zip(rows, rows2):
        assert np.array_equal(a, b)
    ref.close()
    print(f"{config}: {total} decisions, {admitted} admitted, bit-exact")
