"""Replica sweeps on the device (K6): plumbing over kx_replicas_run and the
host realize() restatement (kx_realize_builtin)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import check
from .sched import DispatcherConfig, InstanceProfile

APPS = {"qa": 1, "rg": 2, "cg": 4, "colocated": 7}
SCALAR_NAMES = ["preemption_events", "preempted_requests", "wasted_kv_tokens", "completed_kv_tokens",
                "prefill_seconds", "decode_seconds", "total_events", "end_time"]


def realize(apps="colocated", rate=3.0, duration=720.0, seed=1, prefill_rate=8000.0, decode_rate=50.0):
    """realize() (workload.cpp:319-372) for the built-in templates."""
    lib = _abi.load()
    r = C.c_void_p()
    check(lib.kx_realize_builtin(APPS[apps] if isinstance(apps, str) else apps, rate, duration, seed,
                                 prefill_rate, decode_rate, C.byref(r)))
    nw, nc = C.c_int64(), C.c_int64()
    lib.kx_realization_sizes(r, C.byref(nw), C.byref(nc))
    out = dict(arrival=np.zeros(nw.value), app=np.zeros(nw.value, np.int32),
               wf_offsets=np.zeros(nw.value + 1, np.int64), agent=np.zeros(nc.value, np.int32),
               parent=np.zeros(nc.value, np.int32), prompt=np.zeros(nc.value, np.int64),
               target=np.zeros(nc.value, np.int64), pure_exec=np.zeros(nc.value),
               remaining=np.zeros(nc.value), uid=np.zeros(nc.value, np.uint64))
    lib.kx_realization_copy(r, *[v.ctypes.data for v in out.values()])
    lib.kx_realization_free(r)
    return out


def concat(reals):
    """Concatenate per-replica realizations into one kx_replica_batch layout."""
    wf_base = [0]
    arrays = {k: [] for k in ["arrival", "agent", "parent", "prompt", "target", "pure_exec", "remaining", "uid"]}
    offs = [np.zeros(1, np.int64)]
    c_total = 0
    for rz in reals:
        wf_base.append(wf_base[-1] + len(rz["arrival"]))
        for k in arrays:
            arrays[k].append(rz[k])
        offs.append(rz["wf_offsets"][1:] + c_total)
        c_total += len(rz["agent"])
    out = {k: np.ascontiguousarray(np.concatenate(v)) for k, v in arrays.items()}
    out["wf_base"] = np.array(wf_base, np.int64)
    out["wf_offsets"] = np.concatenate(offs).astype(np.int64)
    return out


METRIC_NAMES = ["instances", "requests", "mean_token_latency", "p90_token_latency", "p95_token_latency",
                "p99_token_latency", "mean_request_token_latency", "mean_queueing_ratio", "preemption_rate",
                "preempted_requests", "preemption_events", "wasted_memory_fraction", "total_queue_seconds",
                "decode_time_fraction", "sim_end_time", "latency_count"]


def builtin_agent_order(n_agents=10):
    """Agent indices in AgentId order (std::map iteration: byte-wise name
    order), the label order of the reference's W1 matrix (priority.cpp:49-65)."""
    lib = _abi.load()
    names = [lib.kx_builtin_agent_name(a).decode() for a in range(n_agents)]
    return np.array(sorted(range(n_agents), key=lambda a: names[a].encode()), np.int32)


def run_replicas(batch, instances: list[InstanceProfile], scheduler="fcfs",
                 dispatcher: DispatcherConfig | None = None, topo_depth=None, n_agents=10,
                 dispatch_period=0.1, recompute_fraction=1.0, heap_capacity=0, device=0,
                 warmup_seconds=0.0, agent_order=None, rebuild_interval=0):
    """Whole replica simulations on the device (K6). scheduler "kairos" runs
    the KairosScheduler's online table rebuilds; time_slot dispatch without
    oracle_expected_time takes T from the device profiler (engine.cpp:177-185)."""
    lib = _abi.load()
    d = dispatcher or DispatcherConfig()
    arr = (_abi.kx_instance * len(instances))()
    for i, p in enumerate(instances):
        arr[i] = _abi.kx_instance(p.id, 0, p.capacity_tokens, p.decode_rate, p.prefill_rate, p.max_batch, 0)
    dc = _abi.kx_dispatcher_config(_abi.DISPATCH[d.policy], int(d.oracle_expected_time), d.slot_len,
                                   d.resume_watermark, d.static_threshold, d.default_expected_time)
    depth = np.ascontiguousarray(topo_depth if topo_depth is not None else np.ones(n_agents), np.int32)
    cfg = _abi.kx_engine_config(len(instances), _abi.SCHED[scheduler], arr, dc, n_agents, 0,
                                depth.ctypes.data, dispatch_period, recompute_fraction, heap_capacity,
                                device, 0, warmup_seconds)
    if agent_order is None:
        agent_order = builtin_agent_order(n_agents) if n_agents == 10 else np.arange(n_agents)
    order = np.ascontiguousarray(agent_order, np.int32)
    cfg.agent_order = order.ctypes.data
    cfg.kairos_rebuild_interval = rebuild_interval
    R = len(batch["wf_base"]) - 1
    W = int(batch["wf_base"][-1])
    Cn = len(batch["agent"])
    cols = [np.ascontiguousarray(batch[k], dt) for k, dt in [
        ("wf_base", np.int64), ("arrival", np.float64), ("wf_offsets", np.int64), ("agent", np.int32),
        ("parent", np.int32), ("prompt", np.int64), ("target", np.int64), ("pure_exec", np.float64),
        ("remaining", np.float64), ("uid", np.uint64)]]
    b = _abi.kx_replica_batch(R, 0, *[c.ctypes.data for c in cols])
    res = dict(call_order=np.zeros(Cn, np.int64), exec_start=np.zeros(Cn), exec_end=np.zeros(Cn),
               instance=np.zeros(Cn, np.int32), first_enqueue=np.zeros(Cn), queue_seconds=np.zeros(Cn),
               episodes=np.zeros(Cn, np.int32), preemptions=np.zeros(Cn, np.int32),
               wf_order=np.zeros(W, np.int64), wf_finish=np.zeros(W), wf_output_tokens=np.zeros(W, np.int64),
               wf_calls=np.zeros(W, np.int32), scalars=np.zeros(R * 8), counts=np.zeros(R * 4, np.int64),
               metrics=np.zeros(R * 16), histogram=np.zeros(R * 256, np.uint32),
               priority_keys=np.zeros(R * n_agents), table_versions=np.zeros(R, np.int64))
    out = _abi.kx_replica_results(*[v.ctypes.data for v in res.values()])
    ms = C.c_double()
    check(lib.kx_replicas_run(C.byref(cfg), C.byref(b), C.byref(out), C.byref(ms)))
    res["device_ms"] = ms.value
    res["scalars"] = res["scalars"].reshape(R, 8)
    res["counts"] = res["counts"].reshape(R, 4)
    res["metrics"] = res["metrics"].reshape(R, 16)
    res["histogram"] = res["histogram"].reshape(R, 256)
    res["priority_keys"] = res["priority_keys"].reshape(R, n_agents)
    return res


def aggregate(metrics_rows):
    """aggregate_metrics (metrics.cpp:90-123) in replica order."""
    lib = _abi.load()
    rows = np.ascontiguousarray(metrics_rows, np.float64)
    out = np.zeros(16)
    check(lib.kx_aggregate_metrics(len(rows), rows.ctypes.data, out.ctypes.data))
    return out


def shard(n_replicas: int, rank: int, world: int) -> list[int]:
    """Replica r runs on rank r % world (independent replicas: no exchange)."""
    return list(range(rank, n_replicas, world))


def gather_rows(dist, rows, hist, n_replicas: int, world: int, device):
    """All-gather per-replica metric rows [R_local, 16] and latency
    histograms [R_local, 256] (NCCL on CUDA tensors, gloo on CPU) and return
    (rows in replica order [R, 16], summed histogram [256]) on every rank."""
    import torch
    m = torch.as_tensor(np.asarray(rows, np.float64), device=device)
    h = torch.as_tensor(np.asarray(hist, np.int64), device=device)
    mx = max(len(shard(n_replicas, k, world)) for k in range(world))
    pm = torch.zeros((mx, 16), dtype=torch.float64, device=device)
    ph = torch.zeros((mx, 256), dtype=torch.int64, device=device)
    pm[:m.shape[0]] = m
    ph[:h.shape[0]] = h
    gm = [torch.zeros_like(pm) for _ in range(world)]
    gh = [torch.zeros_like(ph) for _ in range(world)]
    dist.all_gather(gm, pm)
    dist.all_gather(gh, ph)
    out = np.zeros((n_replicas, 16))
    tot = np.zeros(256, np.int64)
    for k in range(world):
        idx = shard(n_replicas, k, world)
        out[idx] = gm[k][:len(idx)].cpu().numpy()
        tot += gh[k][:len(idx)].sum(0).cpu().numpy()
    return out, tot
