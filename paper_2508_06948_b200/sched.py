"""Thin Python handle over the C ABI (tests / benchmark plumbing).

`DeviceScheduler` owns one kx_sched: the device-resident ready queue of P
pools, the per-agent tables, and each instance's live view and slot ledger.
Method names follow the reference API they replace (scheduler.hpp,
priority.hpp, dispatcher.hpp, engine.cpp:220-268).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._abi import check, ptr


@dataclass
class InstanceProfile:
    """InstanceProfile (engine.hpp:25-31) + the pool it serves."""
    id: int
    pool: int = 0
    capacity_tokens: float = 3000.0
    decode_rate: float = 50.0
    prefill_rate: float = 8000.0
    max_batch: int = 64


@dataclass
class DispatcherConfig:
    """DispatcherConfig (dispatcher.hpp:112-121)."""
    policy: str = "time_slot"
    slot_len: float = 0.5
    resume_watermark: float = 0.85
    static_threshold: float = 0.90
    default_expected_time: float = 1.0
    oracle_expected_time: bool = False


DECISION_DTYPE = np.dtype([("time", "<f8"), ("predicted_peak", "<f8"), ("uid", "<u8"),
                           ("queue_index", "<i8"), ("agent", "<i4"), ("target", "<i4"),
                           ("pool", "<i4"), ("admitted", "<i4")])
assert DECISION_DTYPE.itemsize == C.sizeof(_abi.kx_decision)
ADMISSION_DTYPE = np.dtype([("time", "<f8"), ("uid", "<u8"), ("queue_index", "<i8"), ("instance", "<i4"),
                            ("pool", "<i4")])


class DeviceScheduler:
    def __init__(self, instances: list[InstanceProfile], n_pools: int = 1,
                 dispatcher: DispatcherConfig | None = None, queue_capacity: int = 1 << 16,
                 max_agents: int = 1024, slot_ring: int = 256, device: int = 0,
                 log_capacity_per_pool: int = 0):
        self.lib = _abi.load()
        d = dispatcher or DispatcherConfig()
        self.instances = list(instances)
        self.n_pools = n_pools
        arr = (_abi.kx_instance * len(instances))()
        for i, p in enumerate(instances):
            arr[i] = _abi.kx_instance(p.id, p.pool, p.capacity_tokens, p.decode_rate,
                                      p.prefill_rate, p.max_batch, 0)
        dc = _abi.kx_dispatcher_config(_abi.DISPATCH[d.policy], int(d.oracle_expected_time),
                                       d.slot_len, d.resume_watermark, d.static_threshold,
                                       d.default_expected_time)
        cfg = _abi.kx_sched_config(n_pools, len(instances), arr, dc, queue_capacity, max_agents,
                                   slot_ring, device, log_capacity_per_pool)
        self._arr = arr
        h = C.c_void_p()
        check(self.lib.kx_sched_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.ring = slot_ring
        self._keep = []

    def close(self):
        if getattr(self, "h", None):
            self.lib.kx_sched_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing -----------------------------------------------------------
    def stream_ptr(self) -> int:
        s = C.c_void_p()
        check(self.lib.kx_sched_stream(self.h, C.byref(s)))
        return s.value or 0

    def synchronize(self):
        check(self.lib.kx_sched_synchronize(self.h))

    # -- scheduler policy / tables -------------------------------------------
    def set_scheduler(self, kind: str):
        check(self.lib.kx_set_scheduler(self.h, _abi.SCHED[kind]))

    def set_agent_tables(self, agent_pool, priority_key=None, topo_depth=None, expected_T=None,
                         version: int = 0):
        ap = np.ascontiguousarray(agent_pool, dtype=np.int32)
        pk = None if priority_key is None else np.ascontiguousarray(priority_key, dtype=np.float64)
        dp = None if topo_depth is None else np.ascontiguousarray(topo_depth, dtype=np.int32)
        T = None if expected_T is None else np.ascontiguousarray(expected_T, dtype=np.float64)
        check(self.lib.kx_set_agent_tables(self.h, len(ap), ptr(ap), ptr(pk), ptr(dp), ptr(T),
                                           version))

    def set_remaining_table(self, uid_base: int, remaining, present):
        rem = np.ascontiguousarray(remaining, dtype=np.float64)
        pr = np.ascontiguousarray(present, dtype=np.uint8)
        check(self.lib.kx_set_remaining_table(self.h, uid_base, len(rem), ptr(rem), ptr(pr),
                                              _abi.KX_MEM_HOST))

    # -- queue ---------------------------------------------------------------
    def _view(self, agent, prompt_tokens, app_start, queue_enter, msg_key, uid, kept_tokens, pure_exec, device):
        if device:
            cols = [agent, prompt_tokens, app_start, queue_enter, msg_key, uid, kept_tokens, pure_exec]
            return cols, int(agent.numel()), _abi.KX_MEM_DEVICE
        cols = [np.ascontiguousarray(agent, np.int32), np.ascontiguousarray(prompt_tokens, np.int64),
                np.ascontiguousarray(app_start, np.float64), np.ascontiguousarray(queue_enter, np.float64),
                np.ascontiguousarray(msg_key, np.uint64), np.ascontiguousarray(uid, np.uint64),
                None if kept_tokens is None else np.ascontiguousarray(kept_tokens, np.int64),
                None if pure_exec is None else np.ascontiguousarray(pure_exec, np.float64)]
        return cols, len(cols[0]), _abi.KX_MEM_HOST

    def upload(self, agent, prompt_tokens, app_start, queue_enter, msg_key, uid, kept_tokens=None,
               pure_exec=None, device: bool = False, mapped: bool = False):
        """Replace the queue. Host numpy arrays, or torch CUDA tensors with device=True, or
        pinned host torch tensors with mapped=True (KX_MEM_HOST_MAPPED: prompt, kept, msg and
        uid are read in place; keep the tensors alive and unchanged until the next upload)."""
        if mapped:
            cols = [agent, prompt_tokens, app_start, queue_enter, msg_key, uid, kept_tokens, pure_exec]
            for c in cols:
                if c is not None and not c.is_pinned():
                    raise ValueError("mapped upload needs pinned host tensors")
            self._mapped_cols = cols  # the device reads them until the next upload
            n, mem = int(agent.numel()), _abi.KX_MEM_HOST_MAPPED
        else:
            cols, n, mem = self._view(agent, prompt_tokens, app_start, queue_enter, msg_key, uid, kept_tokens,
                                      pure_exec, device)
        v = _abi.kx_queue_view(*[ptr(c) for c in cols])
        check(self.lib.kx_queue_upload(self.h, n, C.byref(v), mem))
        self.n = n

    def enqueue(self, agent, prompt_tokens, app_start, queue_enter, msg_key, uid, kept_tokens=None,
                pure_exec=None, device: bool = False):
        """ReadyQueue::enqueue (priority.hpp:72) for each request, in order: append."""
        cols, n, mem = self._view(agent, prompt_tokens, app_start, queue_enter, msg_key, uid, kept_tokens,
                                  pure_exec, device)
        v = _abi.kx_queue_view(*[ptr(c) for c in cols])
        check(self.lib.kx_queue_enqueue(self.h, n, C.byref(v), mem))
        self.n = self.size()

    def size(self) -> int:
        n = C.c_int64()
        check(self.lib.kx_queue_size(self.h, C.byref(n)))
        return n.value

    def remove_admitted(self):
        check(self.lib.kx_queue_remove_admitted(self.h))
        self.n = self.size()

    # -- K2/K3/K4 --------------------------------------------------------------
    def score(self):
        n = self.size()
        k = np.zeros((3, n), np.float64)
        check(self.lib.kx_score(self.h, ptr(k[0]), ptr(k[1]), ptr(k[2]), _abi.KX_MEM_HOST))
        return k

    def order(self):
        check(self.lib.kx_order(self.h))

    def fetch_order(self):
        n = self.size()
        perm = np.zeros(n, np.uint32)
        offs = np.zeros(self.n_pools + 1, np.int64)
        check(self.lib.kx_order_fetch(self.h, ptr(perm), ptr(offs), _abi.KX_MEM_HOST))
        return perm, offs

    # -- K5 ---------------------------------------------------------------------
    def dispatch_round(self, now: float):
        check(self.lib.kx_dispatch_round(self.h, now))

    def tick(self, now: float):
        check(self.lib.kx_tick(self.h, now))

    def fetch_dispatch(self):
        """Returns (rows per pool list of structured arrays, candidate peaks per pool)."""
        cnt = np.zeros(self.n_pools, np.int64)
        rs, ps = C.c_int64(), C.c_int64()
        check(self.lib.kx_dispatch_fetch(self.h, ptr(cnt), None, None, C.byref(rs), C.byref(ps)))
        # only each pool's first cnt[p] rows are written (and returned)
        rows = np.empty(self.n_pools * rs.value, DECISION_DTYPE)
        cand = np.empty(self.n_pools * rs.value * ps.value, np.float64)
        check(self.lib.kx_dispatch_fetch(self.h, ptr(cnt), ptr(rows), ptr(cand), C.byref(rs),
                                         C.byref(ps)))
        rows = rows.reshape(self.n_pools, rs.value)
        cand = cand.reshape(self.n_pools, rs.value, ps.value)
        return [rows[p, :cnt[p]] for p in range(self.n_pools)], \
               [cand[p, :cnt[p]] for p in range(self.n_pools)]

    # -- waiting lists (round_robin / static_threshold) ---------------------------
    def set_waiting(self, instance_pos, agent, prompt_tokens, app_start, queue_enter, msg_key, uid,
                    kept_tokens=None):
        """Replace every waiting list: entry j joins the instance at position instance_pos[j]."""
        pos = np.ascontiguousarray(instance_pos, np.int32)
        cols = [np.ascontiguousarray(agent, np.int32), np.ascontiguousarray(prompt_tokens, np.int64),
                np.ascontiguousarray(app_start, np.float64), np.ascontiguousarray(queue_enter, np.float64),
                np.ascontiguousarray(msg_key, np.uint64), np.ascontiguousarray(uid, np.uint64),
                None if kept_tokens is None else np.ascontiguousarray(kept_tokens, np.int64), None]
        v = _abi.kx_queue_view(*[ptr(c) for c in cols])
        check(self.lib.kx_waiting_upload(self.h, len(pos), ptr(pos), C.byref(v)))

    def waiting_uids(self, instance_pos: int):
        n = C.c_int64()
        check(self.lib.kx_waiting_fetch(self.h, instance_pos, 0, None, C.byref(n)))
        out = np.zeros(n.value, np.uint64)
        check(self.lib.kx_waiting_fetch(self.h, instance_pos, n.value, ptr(out), C.byref(n)))
        return out

    def fetch_admissions(self):
        """Admissions out of the waiting lists in the last round, per pool."""
        cnt = np.zeros(self.n_pools, np.int64)
        rs = C.c_int64()
        check(self.lib.kx_admissions_fetch(self.h, ptr(cnt), None, C.byref(rs)))
        rows = np.zeros(self.n_pools * rs.value, ADMISSION_DTYPE)
        check(self.lib.kx_admissions_fetch(self.h, ptr(cnt), ptr(rows), C.byref(rs)))
        rows = rows.reshape(self.n_pools, rs.value)
        return [rows[p, :cnt[p]] for p in range(self.n_pools)]

    def rr_next(self, set_to=None):
        got = np.zeros(self.n_pools, np.int64)
        st = None if set_to is None else np.ascontiguousarray(set_to, np.int64)
        check(self.lib.kx_rr_next(self.h, ptr(got), ptr(st)))
        return got

    # -- instance / ledger state ----------------------------------------------------
    def set_live(self, live_kv=None, running=None, waiting=None):
        lk = None if live_kv is None else np.ascontiguousarray(live_kv, np.float64)
        rn = None if running is None else np.ascontiguousarray(running, np.int32)
        wt = None if waiting is None else np.ascontiguousarray(waiting, np.int32)
        check(self.lib.kx_instances_set_live(self.h, ptr(lk), ptr(rn), ptr(wt)))

    def get_live(self):
        n = len(self.instances)
        lk = np.zeros(n, np.float64)
        rn = np.zeros(n, np.int32)
        wt = np.zeros(n, np.int32)
        sp = np.zeros(n, np.uint8)
        check(self.lib.kx_instances_get_live(self.h, ptr(lk), ptr(rn), ptr(wt), ptr(sp)))
        return lk, rn, wt, sp

    def try_place(self, instance_id, P, k, t0, T):
        fits, peak, viol = C.c_int32(), C.c_double(), C.c_int64()
        check(self.lib.kx_ledger_try_place(self.h, instance_id, P, k, t0, T, C.byref(fits),
                                           C.byref(peak), C.byref(viol)))
        return bool(fits.value), peak.value, viol.value

    def commit(self, instance_id, uid, P, k, t0, T):
        check(self.lib.kx_ledger_commit(self.h, instance_id, uid, P, k, t0, T))

    def commit_batch(self, instance_id, uid, P, k, t0, T):
        """Batched SlotLedger::commit (skips entries that do not fit); returns fit flags."""
        arrs = [np.ascontiguousarray(instance_id, np.int32), np.ascontiguousarray(uid, np.uint64),
                np.ascontiguousarray(P, np.float64), np.ascontiguousarray(k, np.float64),
                np.ascontiguousarray(t0, np.float64), np.ascontiguousarray(T, np.float64)]
        fits = np.zeros(len(arrs[0]), np.uint8)
        check(self.lib.kx_ledger_commit_batch(self.h, len(arrs[0]), *[ptr(a) for a in arrs], ptr(fits)))
        return fits

    def on_request_finished(self, instance_id, uid, actual_end):
        check(self.lib.kx_on_request_finished(self.h, instance_id, uid, actual_end))

    def on_overload(self, instance_id):
        check(self.lib.kx_on_overload(self.h, instance_id))

    def on_live_usage(self, instance_id, live_kv):
        check(self.lib.kx_on_live_usage(self.h, instance_id, live_kv))

    def gc(self, now):
        check(self.lib.kx_gc(self.h, now))

    def ledger(self, instance_id):
        base = C.c_int64()
        na = C.c_int32()
        usage = np.zeros(self.ring, np.float64)
        ex = np.zeros(self.ring, np.uint8)
        check(self.lib.kx_ledger_read(self.h, instance_id, C.byref(base), ptr(usage), ptr(ex),
                                      C.byref(na)))
        return {int(base.value + i): float(usage[i]) for i in range(self.ring) if ex[i]}, na.value

    def profile(self, enable: bool = True):
        check(self.lib.kx_profile_enable(self.h, int(enable)))

    def profile_read(self):
        arr = (_abi.kx_phase_stat * 64)()
        n = C.c_int32()
        check(self.lib.kx_profile_read(self.h, arr, 64, C.byref(n)))
        return {arr[i].name.decode(): {"ms": arr[i].total_ms, "launches": arr[i].launches,
                                       "alg_bytes": arr[i].alg_bytes} for i in range(n.value)}

    def capture_begin(self):
        """Start capturing this handle's asynchronous calls into a CUDA graph."""
        check(self.lib.kx_graph_capture_begin(self.h))

    def capture_end(self):
        check(self.lib.kx_graph_capture_end(self.h))

    def graph_release(self):
        check(self.lib.kx_graph_release(self.h))

    def graph_launch(self):
        """Replay the captured calls (one launch)."""
        check(self.lib.kx_graph_launch(self.h))

    def checkpoint(self):
        check(self.lib.kx_state_checkpoint(self.h))

    def restore(self):
        check(self.lib.kx_state_restore(self.h))


def orchestrator_dp(wf_offsets, parent, prompt_tokens, target_tokens, prefill_rate=8000.0,
                    decode_rate=50.0, uid_base=1):
    """K1 over many workflows (finalize_instance, workload.cpp:292-315)."""
    lib = _abi.load()
    off = np.ascontiguousarray(wf_offsets, np.int64)
    par = np.ascontiguousarray(parent, np.int32)
    pr = np.ascontiguousarray(prompt_tokens, np.int64)
    tg = np.ascontiguousarray(target_tokens, np.int64)
    n = len(par)
    uid = np.zeros(n, np.uint64)
    pure = np.zeros(n, np.float64)
    rem = np.zeros(n, np.float64)
    check(lib.kx_orchestrator_dp(len(off) - 1, ptr(off), ptr(par), ptr(pr), ptr(tg), prefill_rate,
                                 decode_rate, uid_base, ptr(uid), ptr(pure), ptr(rem),
                                 _abi.KX_MEM_HOST))
    return uid, pure, rem


def record_remaining(rec_offsets, exec_start, exec_end):
    """K1b: per-workflow finish and remaining samples (profiler.cpp:31-50)."""
    lib = _abi.load()
    off = np.ascontiguousarray(rec_offsets, np.int64)
    es = np.ascontiguousarray(exec_start, np.float64)
    ee = np.ascontiguousarray(exec_end, np.float64)
    fin = np.zeros(len(off) - 1, np.float64)
    smp = np.zeros(len(es), np.float64)
    check(lib.kx_record_remaining(len(off) - 1, ptr(off), ptr(es), ptr(ee), ptr(fin), ptr(smp),
                                  _abi.KX_MEM_HOST))
    return fin, smp


def sorting_accuracy(agent, remaining, present=None, scope="cross_agent"):
    """K8: pairwise_sorting_accuracy (priority.cpp:165-189); returns
    (accuracy or None, pairs, correct)."""
    lib = _abi.load()
    a = np.ascontiguousarray(agent, np.int32)
    r = np.ascontiguousarray(remaining, np.float64)
    pr = None if present is None else np.ascontiguousarray(present, np.uint8)
    pairs, correct, acc = C.c_uint64(), C.c_double(), C.c_double()
    check(lib.kx_sorting_accuracy(len(a), ptr(a), ptr(r), ptr(pr), 1 if scope == "all" else 0,
                                  C.byref(pairs), C.byref(correct), C.byref(acc)))
    return (None if pairs.value == 0 else acc.value), pairs.value, correct.value


class Profiler:
    """LatencyProfiler (profiler.hpp:49-90) on the device (K9): per agent an
    execution and a remaining-latency EmpiricalDistribution. Configs are
    (min_samples, relative_threshold, window_cap) (distribution.hpp:36-40)."""

    EXECUTION, REMAINING = 0, 1

    def __init__(self, n_agents: int, exec_cfg=(16, 0.05, 0), remaining_cfg=(16, 0.05, 4096),
                 capacity: int = 8192, device: int = 0):
        self.lib = _abi.load()
        self.n_agents = n_agents
        ec = _abi.kx_convergence_config(*exec_cfg)
        rc = _abi.kx_convergence_config(*remaining_cfg)
        h = C.c_void_p()
        check(self.lib.kx_profiler_create(n_agents, C.byref(ec), C.byref(rc), capacity, device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.kx_profiler_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def record_execution(self, agent, latency):
        a = np.ascontiguousarray(agent, np.int32)
        v = np.ascontiguousarray(latency, np.float64)
        check(self.lib.kx_profiler_record_execution(self.h, len(a), ptr(a), ptr(v)))

    def record_remaining(self, rec_offsets, agent, exec_start, exec_end):
        """Completed workflows in order; returns take_newly_converged() per workflow."""
        off = np.ascontiguousarray(rec_offsets, np.int64)
        a = np.ascontiguousarray(agent, np.int32)
        es = np.ascontiguousarray(exec_start, np.float64)
        ee = np.ascontiguousarray(exec_end, np.float64)
        newly = np.zeros(max(len(off) - 1, 0), np.uint8)
        check(self.lib.kx_profiler_record_remaining(self.h, len(off) - 1, ptr(off), ptr(a), ptr(es), ptr(ee),
                                                    ptr(newly)))
        return newly

    def read(self, kind: int, agent: int):
        """(sorted samples, total_added, converged, last_checkpoint_distance)."""
        n, tot, cv, last = C.c_int64(), C.c_uint64(), C.c_int32(), C.c_double()
        check(self.lib.kx_profiler_read(self.h, kind, agent, 0, None, C.byref(n), C.byref(tot), C.byref(cv),
                                        C.byref(last)))
        out = np.zeros(n.value, np.float64)
        check(self.lib.kx_profiler_read(self.h, kind, agent, n.value, ptr(out), C.byref(n), C.byref(tot),
                                        C.byref(cv), C.byref(last)))
        return out, tot.value, bool(cv.value), last.value


def w1_matrix(sample_sets):
    """§8(f)2: build_distance_matrix_from_samples (priority.cpp:15-65) on the
    device. sample_sets: per-agent sorted sample arrays in label order; returns
    the (n + 1) x (n + 1) matrix with the anchor {0.0} as the last label,
    bit-identical to the reference."""
    lib = _abi.load()
    sets = [np.ascontiguousarray(x, np.float64) for x in sample_sets]
    off = np.zeros(len(sets) + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in sets]) if sets else []
    flat = np.concatenate(sets) if sets else np.zeros(0)
    m = len(sets) + 1
    out = np.zeros((m, m), np.float64)
    check(lib.kx_w1_matrix(len(sets), ptr(off), ptr(flat), ptr(out)))
    return out
