#!/usr/bin/env python
"""Replica sweep (config C5 shape): many independent load-trace replicas of
the co-located QA+RG+CG workload simulated on the device (K6) with their
metrics computed on the device (K7).

Single GPU:   python scripts/replica_sweep.py --replicas 1024 --duration 720
              (--scheduler kairos --profile-T: the paper's policy, online tables)
Multi GPU:    torchrun --nproc-per-node N scripts/replica_sweep.py ...
Replica r is simulated by rank r % N (weak scaling when --replicas scales
with N); NCCL all-gathers each rank's per-replica metric rows and latency
histograms; rank 0 aggregates them in replica order (aggregate_metrics,
metrics.cpp:90-123) and prints one JSON line.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2508_06948_b200 import DispatcherConfig, InstanceProfile  # noqa: E402
from paper_2508_06948_b200 import engine as E  # noqa: E402

DEPTH = np.array([2, 1, 1, 2, 1, 5, 4, 3, 2, 1], np.int32)  # topo_depths of the templates


def instances(n=16):
    return [InstanceProfile(id=i, capacity_tokens=3000.0, decode_rate=50.0, prefill_rate=8000.0,
                            max_batch=8) for i in range(n)]


def sweep(args, rank=0, ws=1, dev=0):
    mine = E.shard(args.replicas, rank, ws)
    t0 = time.time()
    reals = [E.realize("colocated", args.rate, args.duration, seed=1 + r) for r in mine]
    b = E.concat(reals)
    t_gen = time.time() - t0
    disp = DispatcherConfig(args.dispatcher, oracle_expected_time=not args.profile_T)
    sys.path.insert(0, str(ROOT))
    from bench import Clocks  # nvidia-smi sampling over the device run
    clocks = Clocks(dev)
    clocks.mark(True)
    res = E.run_replicas(b, instances(args.instances), args.scheduler, disp, topo_depth=DEPTH,
                         device=dev, warmup_seconds=args.warmup)
    clocks.mark(False)
    res["clocks"] = clocks.stop()
    n_calls = int(res["counts"][:, 0].sum())
    events = int(res["counts"][:, 3].sum())
    return mine, res, n_calls, events, t_gen, b


def parity(args, mine, res, b, n_check):
    """Bit-exact comparison of n_check replicas (spread over the sweep) with
    the UNMODIFIED reference Simulator on the same realize() output:
    completion order, per-call exec times, counters and compute_metrics."""
    sys.path.insert(0, str(ROOT / "tests"))
    import ref_sim  # noqa: E402  (oracle/_ref/libkxref.so)
    disp = DispatcherConfig(args.dispatcher, oracle_expected_time=not args.profile_T)
    picks = sorted({int(round(x)) for x in np.linspace(0, len(mine) - 1, n_check)})

    def one(j):
        r = mine[j]
        rz = E.realize("colocated", args.rate, args.duration, seed=1 + r)
        ref = ref_sim.run(rz, instances(args.instances), args.scheduler, disp, DEPTH)
        c0 = int(b["wf_offsets"][b["wf_base"][j]])
        n = int(ref["n_calls"])
        bad = []
        if int(res["counts"][j][0]) != n:
            return r, n, ["call count"]
        order = res["call_order"][c0:c0 + n]
        bits = lambda a: np.ascontiguousarray(a).view(np.uint64)  # noqa: E731
        if not np.array_equal(b["uid"][order], ref["uid"][:n]):
            bad.append("completion order")
        for k in ("exec_start", "exec_end"):
            if not np.array_equal(bits(res[k][c0:c0 + n]), bits(ref[k][:n])):
                bad.append(k)
        if not np.array_equal(bits(res["scalars"][j][:8]), bits(ref["scalars"][:8])):
            bad.append("counters")
        m, rs = res["metrics"][j], ref["scalars"]
        for mi, ri in [(2, 8), (3, 9), (4, 10), (5, 11), (6, 12), (7, 13), (8, 14), (11, 15), (13, 16), (12, 17)]:
            if bits(np.array([m[mi]]))[0] != bits(np.array([rs[ri]]))[0]:
                bad.append(f"metric {mi}")
        return r, n, bad

    t0 = time.perf_counter()
    with ThreadPoolExecutor(min(len(picks), os.cpu_count() or 1)) as ex:
        outs = list(ex.map(one, picks))
    return {"replicas_checked": [o[0] for o in outs], "requests_checked": sum(o[1] for o in outs),
            "mismatches": sum(len(o[2]) for o in outs), "details": {o[0]: o[2] for o in outs if o[2]},
            "checked": "completion order, exec_start/exec_end bits per call, counters, compute_metrics bits",
            "reference": "unmodified reference Simulator (oracle/_ref/libkxref.so)",
            "seconds": time.perf_counter() - t0}


def cpu_reference(args, sample):
    sys.path.insert(0, str(ROOT / "tests"))
    import ref_sim  # noqa: E402  (the reference Simulator via oracle/_ref/libkxref.so)
    disp = DispatcherConfig(args.dispatcher, oracle_expected_time=not args.profile_T)
    reals = [E.realize("colocated", args.rate, args.duration, seed=1 + r) for r in range(sample)]
    threads = min(sample, os.cpu_count() or 1)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        outs = list(ex.map(lambda rz: ref_sim.run(rz, instances(args.instances), args.scheduler, disp, DEPTH),
                           reals))
    secs = time.perf_counter() - t0
    calls = sum(int(o["n_calls"]) for o in outs)
    return {"value": calls / secs, "unit": "simulated requests/s", "cores": threads, "kind": "reference",
            "sample": f"{sample} replicas through the reference Simulator (engine.cpp:85-123), "
                      f"{threads} threads, {calls} requests, {secs:.2f}s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--replicas", type=int, default=1024)  # C5: 1024 replicas
    ap.add_argument("--rate", type=float, default=12.0)
    ap.add_argument("--duration", type=float, default=720.0)
    ap.add_argument("--instances", type=int, default=16)
    ap.add_argument("--scheduler", default="fcfs")
    ap.add_argument("--dispatcher", default="time_slot")
    ap.add_argument("--warmup", type=float, default=0.0)
    ap.add_argument("--cpu-sample", type=int, default=16)
    ap.add_argument("--parity", type=int, default=0,
                    help="compare this many replicas bit-exact with the reference Simulator")
    ap.add_argument("--profile-T", action="store_true",
                    help="time_slot T from the online profiler (engine.cpp:177-185) instead of the oracle's")
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    import torch
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    if dist:
        dist.barrier()
    mine, res, n_calls, events, t_gen, b = sweep(args, rank, ws, local)
    dev_ms = res["device_ms"]
    # NCCL gather of metric rows and histograms (the only collective).
    if dist:
        rows, hist = E.gather_rows(dist, res["metrics"], res["histogram"], args.replicas, ws, "cuda")
        t = torch.tensor([dev_ms, float(n_calls), float(events)], device="cuda", dtype=torch.float64)
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        dev_ms = float(tmax[0].item())
        n_calls = int(t[1].item())
        events = int(t[2].item())
    else:
        rows = res["metrics"]
        hist = res["histogram"].sum(0)
    if rank == 0:
        agg = E.aggregate(rows)
        cpu = cpu_reference(args, min(args.cpu_sample, args.replicas)) if ws == 1 and args.cpu_sample > 0 else None
        par = parity(args, mine, res, b, args.parity) if ws == 1 and args.parity > 0 else None
        print(json.dumps({
            "metric": "simulated requests/s (replica sweep: DES + per-replica metrics on device)",
            "value": n_calls / (dev_ms / 1e3), "unit": "simulated requests/s", "n_gpus": ws,
            "replicas": args.replicas, "requests": n_calls, "events": events,
            "events_per_s": events / (dev_ms / 1e3), "device_ms": dev_ms, "scaling": "weak",
            "config": {"workload": f"colocated QA+RG+CG, rate {args.rate}/s for {args.duration}s per replica",
                       "instances": args.instances, "scheduler": args.scheduler, "dispatcher": args.dispatcher,
                       "expected_T": "profiler" if args.profile_T else "oracle"},
            "aggregate": dict(zip(E.METRIC_NAMES, [float(x) for x in agg])),
            "histogram_total": int(hist.sum()),
            "cpu_baseline": cpu, "parity": par, "clocks": res.get("clocks"),
            "host_realize_s": t_gen}), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
