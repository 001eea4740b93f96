#!/usr/bin/env python
"""Benchmark: scheduled requests/s (score + sort + dispatch) of one
scheduling tick, Kairos priority + time-slot dispatch, on 1..N B200s (one
process per GPU, weak scaling: every rank owns its own pools and queue).

  python bench.py [--config C1|C2|C3|C4] [--gpus N] [--steps K] [--warmup W]
                  [--impl mine|reference]

Configs (BASELINE.json `configs`; paper_2508_06948_b200/workload.py):
  C1  QA app, 1 pool x 4 instances, 1K queued requests
  C2  QA+RG+CG co-located, 1 pool x 16 instances, 64K queued requests
  C3  100 generated apps (choice/parallel/feedback, 500 agents), 1 pool x 64
      instances, 1M queued requests
  C4  (default, the headline) 16M queued requests, 8 pools x 32 instances,
      max_batch 64, pre-loaded ledgers
C1-C3 queues are the product's realize() of the config's WorkloadConfig
(bit-identical to the reference's realize(), tests/test_workload_general.py);
C4 is a numpy draw of the co-located shapes at 16M.

One step = restore the pre-tick instance/ledger state (device copy) + kx_tick
(order the whole queue, dispatch every pool) on the handle's stream, replayed
as one CUDA graph. `value` times it with the queue resident in HBM (L2
flushed between steps when the queue is smaller than L2). `e2e` runs the same
step through the C ABI from pinned HOST buffers (queue upload H2D + tick +
decision-log D2H inside the timed region). `parity` compares every decision
of the measured tick (target, admitted, predicted peak bits, candidate peak
bits) and the full queue order with the UNMODIFIED reference (Dispatcher +
comparator sort, oracle/_ref/libkxref.so) run on the same inputs on the host
in the cpu_baseline leg. `--impl reference` times that reference CPU path
alone on this host's cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "scheduled requests/sec (score+sort+dispatch) at 1M–16M queue depth; % HBM roofline"
UNIT = "requests/s"
L2_BYTES = 126 << 20
REF_BUDGET_S = 300.0  # the --impl reference run (warm-up + steps) fits in ~5 minutes
SURVEY_B_ALG = 238.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def tie_elements(snap) -> int:
    """Requests whose (pool, priority key, app_start) -- the compact key's
    discrete part and its primary time -- equals another request's: the
    exact-tuple tie fix can reach msg_key / uid only for these (an upper bound
    of the in-place reads of a mapped upload)."""
    pool = np.asarray(snap.agent_pool)[snap.agent]
    pk = np.asarray(snap.priority_key)[snap.agent]
    o = np.lexsort((snap.app_start, pk, pool))
    p2, k2, a2 = pool[o], pk[o], snap.app_start[o]
    same = (p2[1:] == p2[:-1]) & (k2[1:] == k2[:-1]) & (a2[1:] == a2[:-1])
    tied = np.zeros(len(o), bool)
    tied[1:] |= same
    tied[:-1] |= same
    return int(tied.sum())


class Clocks:
    """SM clock and throttle reasons sampled during the timed region
    (B200_PROFILING.md's clocks line): an NVML polling thread (every 2 ms, so
    even a region of a few milliseconds holds samples) started before the
    warm-up; only the samples inside the marked region are summarised (the
    nearest one if the region is shorter than a period). Falls back to
    `nvidia-smi -lms 50` when NVML is unavailable."""

    REASONS = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80)]

    def __init__(self, index: int):
        import threading
        self.t0 = self.t1 = None
        self.rows = []  # (time, sm_mhz, max_mhz, reason bits)
        self.p = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((time.time(), float(sm), float(mx), int(rs)))
                    except Exception:
                        pass
                    self._stop.wait(0.002)

            self.th = threading.Thread(target=poll, daemon=True)
            self.th.start()
            self.nvml = True
        except Exception:
            self.nvml = False
            self.th = None
            self._start_smi(index)

    def _start_smi(self, index):
        self.path = Path("/tmp") / f"kx_clocks_{os.getpid()}.csv"
        q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def mark(self, start: bool):
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def _smi_rows(self):
        time.sleep(0.15)  # let the sample after the region land
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        import datetime
        rows = []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        bits = dict(self.REASONS)
        for r in self.path.read_text().strip().splitlines():
            c = [x.strip() for x in r.split(",")]
            if len(c) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(c[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                sm, mx = float(c[2]), float(c[3])
            except ValueError:
                continue
            rb = sum(bits[n] for n, v in zip(names, c[6:10]) if v == "Active")
            rows.append((ts, sm, mx, rb))
        return rows

    def stop(self):
        if self.nvml:
            time.sleep(0.01)
            self._stop.set()
            self.th.join(timeout=1)
            rows = list(self.rows)
        elif self.p is not None:
            rows = self._smi_rows()
        else:
            return None
        if not rows:
            return None
        t0 = self.t0 or rows[0][0]
        t1 = self.t1 or rows[-1][0]
        inside = [r for r in rows if t0 <= r[0] <= t1]
        if not inside:  # region shorter than the period: nearest sample
            inside = [min(rows, key=lambda r: abs(r[0] - (t0 + t1) / 2))]
        reasons = sorted({n for r in inside for n, b in self.REASONS if r[3] & b})
        return {"sm_mhz": statistics.median(r[1] for r in inside), "sm_max_mhz": max(r[2] for r in inside),
                "reasons": reasons, "samples": len(inside), "source": "nvml" if self.nvml else "nvidia-smi"}


def config_dict(w, ws):
    snap = w.snap
    qbytes = snap.n * 44
    return {"workload": w.desc, "config": w.name, "queue_depth_per_gpu": snap.n, "pools": snap.n_pools,
            "instances": len(w.insts), "agents": len(snap.agent_names), "policy": "kairos+time_slot",
            "max_batch": w.insts[0].max_batch, "capacity_tokens": w.insts[0].capacity_tokens,
            "l2": ("inputs (%d MB) larger than L2" % (qbytes >> 20)) if qbytes > L2_BYTES else
                  ("L2 flushed between steps (queue %.1f MB < L2)" % (qbytes / 2 ** 20)),
            "step": "state restore + kx_tick (order + dispatch), replayed as one CUDA graph",
            "parallelism": f"pools per rank, weak scaling over {ws} GPU(s)"}


def make_sched(w, device):
    import paper_2508_06948_b200 as kx
    snap = w.snap
    s = kx.DeviceScheduler(w.insts, n_pools=snap.n_pools, queue_capacity=snap.n + w.arrivals.n,
                           max_agents=len(snap.agent_pool), device=device)
    s.set_agent_tables(snap.agent_pool, snap.priority_key, snap.topo_depth, snap.expected_T)
    s.set_scheduler("kairos")
    cm = w.commits
    if cm:
        c = np.array(cm, dtype=np.float64).T
        s.commit_batch(c[0].astype(np.int32), np.array([x[1] for x in cm], np.uint64), c[2], c[3], c[4], c[5])
    s.set_live(w.live, w.running, np.zeros(len(w.insts), np.int32))
    s.gc(w.now)  # the pre-loaded state is the end of the previous round (engine.cpp:212)
    s.checkpoint()
    return s


def run_mine(args):
    import torch
    import paper_2508_06948_b200 as kx
    from paper_2508_06948_b200 import workload as W

    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    t0 = time.time()
    w = W.build_workload(args.config, rank)
    snap = w.snap
    log(f"[rank {rank}] {w.name}: {snap.n} requests, {len(w.insts)} instances, "
        f"{len(snap.agent_names)} agents ({time.time() - t0:.1f}s)")
    s = make_sched(w, local)
    s.upload(snap.agent, snap.prompt, snap.app_start, snap.queue_enter, snap.msg_key, snap.uid)
    stream = torch.cuda.ExternalStream(s.stream_ptr(), device=dev)
    lib = s.lib
    NOW = w.now

    def step():
        s.restore()
        s.tick(NOW)

    clocks = Clocks(local)
    for _ in range(args.warmup):
        step()
    s.synchronize()
    gpu_rows, gpu_cand = s.fetch_dispatch()
    admitted = int(sum(int(r["admitted"].sum()) for r in gpu_rows))
    decisions = int(sum(len(r) for r in gpu_rows))
    s.order()
    gpu_perm, gpu_offs = s.fetch_order()

    # The step (state restore + tick) is captured once into a CUDA graph and
    # replayed: same kernels, one launch per step instead of ~30.
    s.capture_begin()
    step()
    s.capture_end()
    for _ in range(2):
        s.graph_launch()
    s.synchronize()
    r2, _ = s.fetch_dispatch()
    assert int(sum(int(r["admitted"].sum()) for r in r2)) == admitted, "graph replay differs"

    # ---- timed region: device-resident inputs, graph replays ---------------
    flush = None
    if snap.n * 44 <= L2_BYTES:  # queue fits in L2: flush it between steps (not timed)
        flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    s.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clocks.mark(True)
    if flush is None:
        ev0.record(stream)
        for _ in range(args.steps):
            s.graph_launch()
        ev1.record(stream)
        ev1.synchronize()
        ms_total = ev0.elapsed_time(ev1)
    else:
        ms_total = 0.0
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                flush.zero_()
                ev0.record(stream)
                s.graph_launch()
                ev1.record(stream)
                ev1.synchronize()
                ms_total += ev0.elapsed_time(ev1)
    clocks.mark(False)
    s.synchronize()
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    if dist:
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        dist.barrier()

    # ---- per-kernel CUDA-event timing: the same K steps, launched directly ----
    s.profile(True)
    launches0 = lib.kx_launch_count()
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            if flush is not None:
                flush.zero_()
            step()
    s.synchronize()
    launches = lib.kx_launch_count() - launches0  # the graph replays exactly these kernels
    phases = s.profile_read()
    s.profile(False)
    ms_step = ms_total / args.steps
    n_total = snap.n * ws
    value = n_total / (ms_step / 1e3)

    # ---- e2e: pinned host buffers through the C ABI ------------------------
    # KX_MEM_HOST_MAPPED: the columns every request's key needs (agent,
    # app_start, queue_enter) are copied each step; prompt, msg and uid stay
    # in the pinned buffers and are read in place by the kernels that need
    # them (dispatched heads, exact-tuple ties). h2d counts the copied bytes
    # plus an upper bound of those in-place reads: 3 fields of every head a
    # pool can land (its prefix, <= 2048, plus the resumed heads) and msg +
    # uid of every element of an exact-tuple tie run of the compact key.
    pin = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
           for k, v in dict(agent=snap.agent.astype(np.int32), prompt=snap.prompt, app=snap.app_start,
                            qe=snap.queue_enter, msg=snap.msg_key.view(np.int64),
                            uid=snap.uid.view(np.int64)).items()}
    view = kx._abi.kx_queue_view(*[t.data_ptr() for t in
                                   (pin["agent"], pin["prompt"], pin["app"], pin["qe"], pin["msg"],
                                    pin["uid"])], None, None)
    copied = sum(pin[k].numel() * pin[k].element_size() for k in ("agent", "app", "qe"))
    heads_bound = snap.n_pools * 2048 + admitted + snap.n_pools
    key_ties = tie_elements(snap)
    h2d = copied + heads_bound * 3 * 8 + key_ties * 2 * 8

    def e2e_step():
        kx._abi.check(lib.kx_queue_upload(s.h, snap.n, C.byref(view), kx._abi.KX_MEM_HOST_MAPPED))
        s.restore()
        s.tick(NOW)
        r, c = s.fetch_dispatch()
        return sum(x.nbytes for x in r) + sum(x.nbytes for x in c)

    d2h = e2e_step()
    e2e_steps = max(3, min(args.steps, 10))
    if dist:
        dist.barrier()
    s.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    e1.synchronize()
    wall_ms = 1e3 * (time.perf_counter() - w0) / e2e_steps
    # device span between the two events on the handle's stream: covers the
    # H2D copies, validation, tick and D2H plus any host gaps between them
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    # The host link bounds e2e: plain pinned -> device copies of the same
    # copied columns, timed the same way, give its measured bandwidth.
    link_dst = {k: torch.empty_like(pin[k], device=dev) for k in ("agent", "app", "qe")}
    with torch.cuda.stream(stream):
        for _ in range(2):
            for k, d in link_dst.items():
                d.copy_(pin[k], non_blocking=True)
        stream.synchronize()
        l0 = torch.cuda.Event(enable_timing=True)
        l1 = torch.cuda.Event(enable_timing=True)
        l0.record(stream)
        for _ in range(3):
            for k, d in link_dst.items():
                d.copy_(pin[k], non_blocking=True)
        l1.record(stream)
        l1.synchronize()
    link_gbps = 3 * copied / (l0.elapsed_time(l1) / 1e3) / 1e9
    del link_dst

    # ---- steady-state serving loop: the queue stays resident ----------------
    # The reference's ReadyQueue persists across dispatch rounds
    # (engine.cpp:220-268): each step enqueues that step's arrivals from
    # pinned host memory (kx_queue_enqueue), ticks, reads the decision log
    # back and pops the placed requests (kx_queue_remove_admitted); the queue
    # stays at its depth because as many requests arrive as were placed.
    arr = w.arrivals
    apin = [torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for v in
            (arr.agent.astype(np.int32), arr.prompt, arr.app_start, arr.queue_enter,
             arr.msg_key.view(np.int64), arr.uid.view(np.int64))]
    a_bytes_per_req = sum(t.element_size() for t in apin)
    s.graph_release()  # the timed replays are done: the pop may swap the queue's double buffer
    kx._abi.check(lib.kx_queue_upload(s.h, snap.n, C.byref(view), kx._abi.KX_MEM_HOST))
    a_pos = [0]

    def steady_step():
        s.restore()
        s.tick(NOW)
        r, cpk = s.fetch_dispatch()
        m = int(sum(int(x["admitted"].sum()) for x in r))
        s.remove_admitted()
        o = a_pos[0]
        if o + m > arr.n:
            o = 0
        v2 = kx._abi.kx_queue_view(*[t.data_ptr() + o * t.element_size() for t in apin], None, None)
        kx._abi.check(lib.kx_queue_enqueue(s.h, m, C.byref(v2), kx._abi.KX_MEM_HOST))
        a_pos[0] = o + m
        return m * a_bytes_per_req, sum(x.nbytes for x in r) + sum(x.nbytes for x in cpk)

    steady_step()
    st_steps = max(3, min(args.steps, 10))
    st_h2d = st_d2h = 0
    if dist:
        dist.barrier()
    s.synchronize()
    e0.record(stream)
    for _ in range(st_steps):
        hb, db = steady_step()
        st_h2d += hb
        st_d2h += db
    e1.record(stream)
    e1.synchronize()
    st_ms = e0.elapsed_time(e1) / st_steps
    if dist:
        t = torch.tensor([st_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        st_ms = float(t.item())
    depth_after = s.size()

    # ---- roofline of the dominant kernel ------------------------------------
    hbm, peak_src = peaks()
    dom_name, dom = max(((k, v) for k, v in phases.items() if v["alg_bytes"] > 0),
                        key=lambda kv: kv[1]["ms"])
    dom_launch_ms = dom["ms"] / dom["launches"]
    dom_bytes = dom["alg_bytes"] / dom["launches"]
    achieved = dom_bytes / (dom_launch_ms / 1e3) / 1e9
    tot_ms = sum(v["ms"] for v in phases.values())
    kernels = {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                   "share": v["ms"] / tot_ms if tot_ms else None,
                   "alg_GBps": (v["alg_bytes"] / (v["ms"] / 1e3) / 1e9) if v["alg_bytes"] and v["ms"] else None}
               for k, v in phases.items()}
    tick_bytes = sum(v["alg_bytes"] for v in phases.values()) / args.steps
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(args.config, {}).get(dom_name)
        except Exception:
            traffic = None

    cpu = parity = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu, parity = cpu_baseline(w, gpu_rows, gpu_cand, gpu_perm, gpu_offs)

    if rank == 0:
        cfg = config_dict(w, ws)
        cfg.update(admitted_per_step=admitted, decisions_per_step=decisions)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic: the product's realize() of the config's WorkloadConfig (seed 1+rank), "
                     "first N calls queued" if w.name != "C4" else
                     "synthetic (co-located QA/RG/CG workflow shapes drawn with numpy, workload.snapshot)"),
            "config": cfg,
            "parity": parity,
            "e2e": {"value": n_total / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "wall_ms_per_step": wall_ms,
                    # host link: the step's H2D bytes over its time vs plain pinned copies
                    "link": {"achieved_GBps": h2d / (e2e_ms / 1e3) / 1e9, "copy_GBps": link_gbps,
                             "frac": h2d / (e2e_ms / 1e3) / 1e9 / link_gbps}},
            # the serving loop with the queue resident: only arrivals go up
            "e2e_steady": {"value": n_total / (st_ms / 1e3), "unit": UNIT,
                           "h2d_bytes_per_step": st_h2d / st_steps, "d2h_bytes_per_step": st_d2h / st_steps,
                           "ms_per_step": st_ms, "queue_depth_after": depth_after,
                           "step": "kx_queue_enqueue(arrivals, pinned host) + state restore + kx_tick + "
                                   "decision-log read + kx_queue_remove_admitted"},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": hbm,
                         "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                         "alg_bytes_per_launch": dom_bytes, "peak_source": peak_src,
                         "tick_alg_bytes": tick_bytes,
                         "tick_frac": (tick_bytes / (ms_step / 1e3) / 1e9) / hbm,
                         # SURVEY §8(d)'s north-star accounting of score + sort: a 64-bit key
                         # through 8 LSD passes, B_alg = 38 + 8 + 192 = 238 B/request. This path
                         # moves fewer bytes (32-bit compact key; tick_alg_bytes), so this is the
                         # requests/s the target is stated in, not measured traffic.
                         "survey_b_alg_per_request": SURVEY_B_ALG,
                         "survey_frac": value * SURVEY_B_ALG / 1e9 / hbm},
            "kernels": kernels,
            "gpu_launches": int(launches),
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


# ---- the reference's CPU path ------------------------------------------------
def _ref_lib():
    so = ROOT / "oracle" / "_ref" / "libkxref.so"
    if not so.exists():
        return None
    L = C.CDLL(str(so))
    P = C.c_void_p
    L.kxref_pool_new.restype = P
    L.kxref_pool_new.argtypes = [C.c_int, P, P, P, P, C.c_double, C.c_double, C.c_int, C.c_int, P, P,
                                 P, P, P]
    L.kxref_pool_free.argtypes = [P]
    L.kxref_pool_set_live.argtypes = [P, P, P, P]
    L.kxref_pool_commit.argtypes = [P, C.c_int32, C.c_uint64, C.c_int64, C.c_double, C.c_double]
    L.kxref_pool_gc.argtypes = [P, C.c_double]
    L.kxref_pool_set_queue.argtypes = [P, C.c_int64, P, P, P, P, P, P, P]
    L.kxref_pool_reset.argtypes = [P]
    L.kxref_pool_tick.restype = C.c_int64
    L.kxref_pool_tick.argtypes = [P, C.c_double]
    L.kxref_pools_tick.restype = C.c_double
    L.kxref_pools_tick.argtypes = [C.POINTER(P), C.c_int, C.c_double, C.c_int]
    L.kxref_pool_record.argtypes = [P, C.c_int]
    L.kxref_pool_log.restype = C.c_int64
    L.kxref_pool_log.argtypes = [P, P, P, P, P, P]
    L.kxref_pool_order.restype = C.c_int64
    L.kxref_pool_order.argtypes = [P, P]
    return L


class RefPools:
    """The reference's data structures (Dispatcher with pre-loaded ledgers,
    PendingRequest queue, policy table) for `pools` pools of the workload."""

    def __init__(self, L, w, pools, max_per_pool=None):
        self.L = L
        snap, insts = w.snap, w.insts
        names = [n.encode() for n in snap.agent_names]
        self.cnames = (C.c_char_p * len(names))(*names)
        self.handles, self.pools, self.ni = [], list(pools), []
        self.n = 0
        self._keep = []
        all_ids = np.array([i.id for i in insts])
        for p in pools:
            sel = np.array([i.pool == p for i in insts])
            ids = all_ids[sel].astype(np.int32)
            caps = np.array([i.capacity_tokens for i in insts])[sel]
            ks = np.array([i.decode_rate for i in insts])[sel]
            mb = np.array([i.max_batch for i in insts], np.int32)[sel]
            arrs = [ids, caps, ks, mb, snap.priority_key, snap.pk_known, snap.topo_depth, snap.expected_T]
            self._keep += arrs
            h = L.kxref_pool_new(len(ids), ids.ctypes.data, caps.ctypes.data, ks.ctypes.data, mb.ctypes.data,
                                 0.5, 0.85, 0, len(names), C.cast(self.cnames, C.c_void_p),
                                 snap.priority_key.ctypes.data, snap.pk_known.ctypes.data,
                                 snap.topo_depth.ctypes.data, snap.expected_T.ctypes.data)
            for (iid, uid, P, k, t0, T) in w.commits:
                if iid in ids:
                    L.kxref_pool_commit(h, int(iid), int(uid), int(P), t0, T)
            L.kxref_pool_gc(h, w.now)
            lv = np.ascontiguousarray(w.live[sel])
            rn = np.ascontiguousarray(w.running[sel], np.int32)
            wt = np.zeros(len(ids), np.int32)
            self._keep += [lv, rn, wt]
            L.kxref_pool_set_live(h, lv.ctypes.data, rn.ctypes.data, wt.ctypes.data)
            m = np.flatnonzero(snap.agent_pool[snap.agent] == p)
            if max_per_pool is not None:
                m = m[:max_per_pool]  # a prefix of the pool's queue (bounded reference sample)
            cols = [np.ascontiguousarray(x[m]) for x in (snap.agent, snap.prompt, snap.app_start,
                                                         snap.queue_enter, snap.msg_counter, snap.uid)]
            L.kxref_pool_set_queue(h, len(cols[0]), *[c.ctypes.data for c in cols], C.cast(self.cnames, C.c_void_p))
            self.n += len(cols[0])
            self.handles.append(h)
            self.ni.append(len(ids))
        self.arr = (C.c_void_p * len(self.handles))(*self.handles)

    def tick(self, threads, now):
        return self.L.kxref_pools_tick(self.arr, len(self.handles), now, threads)

    def record(self, on: bool):
        for h in self.handles:
            self.L.kxref_pool_record(h, int(on))

    def log(self, j):
        h, ni = self.handles[j], self.ni[j]
        n = self.L.kxref_pool_log(h, None, None, None, None, None)
        uid = np.zeros(n, np.uint64)
        tgt = np.zeros(n, np.int32)
        adm = np.zeros(n, np.int32)
        peak = np.zeros(n)
        cand = np.zeros((n, ni))
        self.L.kxref_pool_log(h, uid.ctypes.data, tgt.ctypes.data, adm.ctypes.data, peak.ctypes.data,
                              cand.ctypes.data)
        return uid, tgt, adm, peak, cand

    def order(self, j):
        n = self.L.kxref_pool_order(self.handles[j], None)
        out = np.zeros(n, np.uint64)
        self.L.kxref_pool_order(self.handles[j], out.ctypes.data)
        return out

    def close(self):
        for h in self.handles:
            self.L.kxref_pool_free(h)


def compare_decisions(ref, j, rows, cand):
    """Mismatching decision rows of pool ref.pools[j]: uid, target, admitted,
    predicted_peak bits, candidate_peaks bits (engine.cpp:242-246)."""
    uid, tgt, adm, peak, rc = ref.log(j)
    n = min(len(uid), len(rows))
    ni = rc.shape[1]
    bad = np.zeros(n, bool)
    if n:
        bad |= rows["uid"][:n] != uid[:n]
        bad |= rows["target"][:n] != tgt[:n]
        bad |= rows["admitted"][:n] != adm[:n]
        bad |= rows["predicted_peak"][:n].view(np.uint64) != peak[:n].view(np.uint64)
        bad |= (np.ascontiguousarray(cand[:n, :ni]).view(np.uint64) != rc[:n].view(np.uint64)).any(axis=1)
    return len(uid), int(bad.sum()) + abs(len(uid) - len(rows))


def cpu_baseline(w, gpu_rows=None, gpu_cand=None, gpu_perm=None, gpu_offs=None):
    """One tick of the reference's own CPU path (every pool on its own host
    thread), timed; with the GPU's decisions/order given, also their parity."""
    L = _ref_lib()
    if L is None:
        return ({"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                 "sample": "unavailable: oracle/_ref/libkxref.so not built"}, None)
    ncpu = os.cpu_count() or 1
    P = w.snap.n_pools
    k = min(P, ncpu)
    t0 = time.time()
    ref = RefPools(L, w, list(range(k)))
    log(f"cpu baseline: built reference queues for {k} pools ({ref.n} requests) in {time.time() - t0:.1f}s")
    ref.record(gpu_rows is not None)
    threads = min(k, ncpu)
    secs = ref.tick(threads, w.now)
    cpu = {"value": ref.n / secs, "unit": UNIT, "cores": threads, "kind": "reference",
           "sample": f"one tick of {k} of the {P} pool(s) ({ref.n} requests), one pool per host thread: "
                     f"reference comparator std::sort (harness.cpp:92-100) + Dispatcher choose/commit over "
                     f"the dispatched prefix (engine.cpp:220-268) + gc, decision log recorded "
                     f"({secs:.2f}s)", "seconds": secs, "host_cpus": ncpu}
    parity = None
    if gpu_rows is not None:
        t1 = time.time()
        dec = mis = omis = 0
        for j, p in enumerate(ref.pools):
            d, m = compare_decisions(ref, j, gpu_rows[p], gpu_cand[p])
            dec += d
            mis += m
            ro = ref.order(j)
            go = w.snap.uid[gpu_perm[gpu_offs[p]:gpu_offs[p + 1]]]
            omis += int((ro != go).sum()) if len(ro) == len(go) else max(len(ro), len(go))
        parity = {"pools_checked": k, "pools": P, "decisions": dec, "mismatches": mis,
                  "order_checked": int(ref.n), "order_mismatches": omis,
                  "checked": "target, admitted, predicted_peak bits, candidate_peaks bits per decision; "
                             "full per-pool queue order (uids)",
                  "reference": "unmodified reference Dispatcher + ReadyQueue comparator (oracle/_ref)",
                  "seconds": time.time() - t1}
    ref.close()
    return cpu, parity


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    L = _ref_lib()
    if L is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libkxref.so is not built"}))
        return
    from paper_2508_06948_b200 import workload as W
    w = W.build_workload(args.config, 0)
    ncpu = os.cpu_count() or 1
    P = w.snap.n_pools
    ref = RefPools(L, w, list(range(P)))
    threads = min(P, ncpu)
    first = ref.tick(threads, w.now)  # warm-up 1, also sizes the sample
    per_round = first
    m = None
    if first * (args.steps + args.warmup) > REF_BUDGET_S:
        # bounded sample: every pool keeps its instances and ledgers, each
        # step ticks a prefix of every pool's queue (the tick's sort is
        # n log n, so a shorter queue is slightly faster per request)
        per_pool = ref.n // P
        m = per_pool
        for _ in range(4):  # the tick is not linear in the queue length: re-measure and shrink
            m = max(10_000, int(m * REF_BUDGET_S / ((args.steps + args.warmup) * first)))
            ref.close()
            ref = RefPools(L, w, list(range(P)), max_per_pool=m)
            first = ref.tick(threads, w.now)
            if first * (args.steps + args.warmup) <= REF_BUDGET_S or m == 10_000:
                break
    for _ in range(max(0, args.warmup - 1)):
        ref.tick(threads, w.now)
    times = [ref.tick(threads, w.now) for _ in range(args.steps)]
    ms = 1e3 * sum(times) / len(times)
    value = ref.n / (ms / 1e3)
    k = P
    sample = (f"{k} of {P} pool(s) per step ({ref.n} requests"
              + (f": the first {m} of each pool's queue" if m else "") +
              f"), {threads} host threads (one pool per "
              f"thread, the reference's one-Simulator-per-thread model, harness.cpp:189-206): reference "
              f"comparator std::sort (harness.cpp:92-100) + reference Dispatcher over the dispatched "
              f"prefix + gc. The prefix walk replaces the reference's O(N) best_index scan per placement "
              f"(priority.hpp:89-103), so this baseline is faster than the stock path")
    cfg = config_dict(w, ws)
    del per_round
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, the same inputs as the mine arm (workload.build_workload)",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    ref.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4"])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mine(args)


if __name__ == "__main__":
    main()
