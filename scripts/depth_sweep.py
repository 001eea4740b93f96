#!/usr/bin/env python
"""Tick throughput across queue depths (north star: 1K to 16M), one B200.

The C4 instance layout (8 LLM pools x 32 instances, pre-loaded ledgers,
Kairos priority + time-slot dispatch) over queues of 1K, 64K, 1M and 16M
requests split evenly over the pools. Per depth: device time of the step
(state restore + kx_tick, replayed as one CUDA graph; inputs resident in
HBM), scheduled requests/s, and the reference's own CPU path on the same
pools (comparator std::sort + Dispatcher, one pool per host thread).
Prints one JSON line per depth.

    python scripts/depth_sweep.py [--depths 1000,65536,1000000,16000000] [--steps 50]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def one(depth: int, steps: int, warmup: int, cpu: bool):
    import torch
    from paper_2508_06948_b200 import workload as W

    per_pool = max(1, depth // bench.N_POOLS)
    snap = W.snapshot(n_pools=bench.N_POOLS, per_pool=per_pool, seed=1)
    insts = W.instances(bench.N_POOLS, bench.INST_PER_POOL)
    live, running, commits = W.preload(insts, seed=7, now=bench.NOW)
    s = bench.make_sched(snap, insts, live, running, commits, 0)
    s.upload(snap.agent, snap.prompt, snap.app_start, snap.queue_enter, snap.msg_key, snap.uid)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.ExternalStream(s.stream_ptr(), device=dev)

    def step():
        s.restore()
        s.tick(bench.NOW)

    for _ in range(warmup):
        step()
    s.synchronize()
    rows, _ = s.fetch_dispatch()
    decisions = int(sum(len(r) for r in rows))
    s.capture_begin()
    step()
    s.capture_end()
    s.graph_launch()
    s.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # inputs above L2 only at the larger depths: flush L2 between replays
    # below 8M requests so every step reads its queue from HBM
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if snap.n < 8_000_000 else None
    total = 0.0
    for _ in range(steps):
        if flush is not None:
            flush.zero_()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        s.graph_launch()
        e1.record(stream)
        e1.synchronize()
        total += e0.elapsed_time(e1)
    ms = total / steps
    line = {"metric": "scheduled requests/s (score+sort+dispatch)", "queue_depth": snap.n,
            "value": snap.n / (ms / 1e3), "unit": "requests/s", "ms_per_tick": ms,
            "decisions_per_tick": decisions, "pools": bench.N_POOLS, "instances": len(insts),
            "l2": "flushed between ticks" if flush is not None else "inputs larger than L2",
            "steps": steps, "warmup": warmup}
    if cpu:
        t0 = time.time()
        line["cpu_baseline"] = bench.cpu_baseline(snap, insts, live, running, commits)
        line["cpu_baseline"]["build_s"] = time.time() - t0
        line["cpu_baseline"]["sample"] = (
            f"one tick of all {bench.N_POOLS} pools ({snap.n} requests), one pool per host thread: the "
            "reference comparator std::sort (harness.cpp:92-100) + Dispatcher choose/commit over the "
            "dispatched prefix + gc")
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--depths", default="1000,65536,1000000,16000000")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    for d in [int(x) for x in args.depths.split(",")]:
        print(json.dumps(one(d, args.steps, args.warmup, not args.no_cpu)), flush=True)


if __name__ == "__main__":
    main()
