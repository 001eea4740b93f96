"""ctypes binding of the oracle's C restatement (oracle/kx_oracle.c).

TEST INFRASTRUCTURE ONLY: the checker for the CUDA path. Built on demand by
`make -C oracle restatement` (gcc only; no reference sources needed).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
SO = ROOT / "oracle" / "_ref" / "kx_oracle.so"

KAIROS, FCFS, TOPO, ORACLE = 0, 1, 2, 3
POLICY = {"kairos": KAIROS, "fcfs": FCFS, "topo_depth": TOPO, "oracle": ORACLE}


class Queue(C.Structure):
    _fields_ = [("n", C.c_int64), ("agent", C.c_void_p), ("prompt", C.c_void_p),
                ("app_start", C.c_void_p), ("queue_enter", C.c_void_p), ("msg_key", C.c_void_p),
                ("uid", C.c_void_p), ("kept", C.c_void_p), ("pure_exec", C.c_void_p)]


class Tables(C.Structure):
    _fields_ = [("n_agents", C.c_int32), ("pool", C.c_void_p), ("pk", C.c_void_p),
                ("depth", C.c_void_p), ("T", C.c_void_p), ("rem_base", C.c_uint64),
                ("rem_n", C.c_int64), ("rem", C.c_void_p), ("rem_present", C.c_void_p)]


class Pool(C.Structure):
    _fields_ = [("n_inst", C.c_int32), ("id", C.c_void_p), ("cap", C.c_void_p), ("k", C.c_void_p),
                ("max_batch", C.c_void_p), ("live_kv", C.c_void_p), ("running", C.c_void_p),
                ("waiting", C.c_void_p), ("suspended", C.c_void_p), ("ledgers", C.c_void_p),
                ("slot_len", C.c_double), ("watermark", C.c_double), ("oracle_T", C.c_int32)]


DECISION = np.dtype([("time", "<f8"), ("predicted_peak", "<f8"), ("uid", "<u8"),
                     ("queue_index", "<i8"), ("agent", "<i4"), ("target", "<i4"),
                     ("pool", "<i4"), ("admitted", "<i4")])

WAITREC = np.dtype([("app_start", "<f8"), ("queue_enter", "<f8"), ("msg", "<u8"), ("uid", "<u8"),
                    ("prompt", "<i8"), ("kept", "<i8"), ("qidx", "<i8"), ("agent", "<i4"),
                    ("round", "<i4")])
ADMISSION = np.dtype([("time", "<f8"), ("uid", "<u8"), ("queue_index", "<i8"), ("instance", "<i4"),
                      ("pool", "<i4")])
DISPATCH_POLICY = {"time_slot": 0, "round_robin": 1, "static_threshold": 2}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not SO.exists():
            subprocess.run(["make", "-C", str(ROOT / "oracle"), "restatement"], check=True,
                           capture_output=True)
        L = C.CDLL(str(SO))
        P = C.c_void_p
        L.kxo_quantile_sorted.restype = C.c_double
        L.kxo_quantile_sorted.argtypes = [P, C.c_int64, C.c_double]
        L.kxo_histogram_mode.restype = C.c_double
        L.kxo_histogram_mode.argtypes = [P, C.c_int64]
        L.kxo_mode_estimate.restype = C.c_double
        L.kxo_mode_estimate.argtypes = [P, C.c_int64, C.c_int64, C.POINTER(C.c_int)]
        L.kxo_wasserstein_1d.restype = C.c_double
        L.kxo_wasserstein_1d.argtypes = [P, C.c_int64, P, C.c_int64]
        L.kxo_median_anchor_distance.restype = C.c_double
        L.kxo_median_anchor_distance.argtypes = [P, C.c_int64, C.c_double]
        L.kxo_order_keys.argtypes = [C.c_int, C.POINTER(Queue), C.POINTER(Tables), P, P, P]
        L.kxo_sort.argtypes = [C.c_int, C.POINTER(Queue), C.POINTER(Tables), C.c_int32, P, P]
        L.kxo_ledger_new.restype = P
        L.kxo_ledger_new.argtypes = [C.c_int32, C.c_double, C.c_double]
        L.kxo_ledger_free.argtypes = [P]
        L.kxo_try_place.argtypes = [P, C.c_double, C.c_double, C.c_double, C.c_double,
                                    C.POINTER(C.c_int32), C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.kxo_commit.argtypes = [P, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double]
        L.kxo_finish.argtypes = [P, C.c_uint64, C.c_double]
        L.kxo_gc.argtypes = [P, C.c_double]
        L.kxo_ledger_dump.restype = C.c_int64
        L.kxo_ledger_dump.argtypes = [P, P, P, C.c_int64]
        L.kxo_ledger_active.restype = C.c_int64
        L.kxo_ledger_active.argtypes = [P]
        L.kxo_dispatch_round.restype = C.c_int64
        L.kxo_dispatch_round.argtypes = [C.POINTER(Pool), C.POINTER(Queue), C.POINTER(Tables), P,
                                         C.c_int64, C.c_double, C.c_int32, P, P, C.c_int64,
                                         C.POINTER(C.c_int32)]
        L.kxo_dispatch_round_waiting.restype = C.c_int64
        L.kxo_dispatch_round_waiting.argtypes = [
            C.POINTER(Pool), C.c_int, C.c_double, C.c_int, C.POINTER(C.c_int64), P, C.c_int64, C.c_int32,
            C.POINTER(Queue), C.POINTER(Tables), P, C.c_int64, C.c_double, C.c_int32, P, C.c_int64, P,
            C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        L.kxo_dist_new.restype = P
        L.kxo_dist_new.argtypes = [C.c_uint64, C.c_double, C.c_int64]
        L.kxo_dist_free.argtypes = [P]
        L.kxo_dist_add.argtypes = [P, C.c_double]
        L.kxo_dist_read.restype = C.c_int64
        L.kxo_dist_read.argtypes = [P, P, C.c_int64, C.POINTER(C.c_uint64), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_double)]
        L.kxo_pairwise_accuracy.argtypes = [C.c_int64, P, P, P, C.c_int32, C.POINTER(C.c_double),
                                            C.POINTER(C.c_uint64)]
        L.kxo_finalize.argtypes = [C.c_int64, P, P, P, P, C.c_double, C.c_double, C.c_uint64, P, P, P]
        L.kxo_record_remaining.argtypes = [C.c_int64, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


class QueueArrays:
    """Owns contiguous arrays + the kxo_queue view."""

    def __init__(self, agent, prompt, app_start, queue_enter, msg_key, uid, kept=None, pure_exec=None):
        self.agent = np.ascontiguousarray(agent, np.int32)
        self.prompt = np.ascontiguousarray(prompt, np.int64)
        self.app_start = np.ascontiguousarray(app_start, np.float64)
        self.queue_enter = np.ascontiguousarray(queue_enter, np.float64)
        self.msg_key = np.ascontiguousarray(msg_key, np.uint64)
        self.uid = np.ascontiguousarray(uid, np.uint64)
        self.kept = None if kept is None else np.ascontiguousarray(kept, np.int64)
        self.pure_exec = None if pure_exec is None else np.ascontiguousarray(pure_exec, np.float64)
        self.view = Queue(len(self.agent), _p(self.agent), _p(self.prompt), _p(self.app_start),
                          _p(self.queue_enter), _p(self.msg_key), _p(self.uid), _p(self.kept),
                          _p(self.pure_exec))


class TableArrays:
    def __init__(self, pool, pk=None, depth=None, T=None, rem_base=0, rem=None, rem_present=None):
        n = len(pool)
        self.pool = np.ascontiguousarray(pool, np.int32)
        self.pk = np.ascontiguousarray(pk if pk is not None else np.zeros(n), np.float64)
        self.depth = np.ascontiguousarray(depth if depth is not None else np.ones(n), np.int32)
        self.T = np.ascontiguousarray(T if T is not None else np.ones(n), np.float64)
        self.rem = None if rem is None else np.ascontiguousarray(rem, np.float64)
        self.rem_present = None if rem_present is None else np.ascontiguousarray(rem_present, np.uint8)
        self.view = Tables(n, _p(self.pool), _p(self.pk), _p(self.depth), _p(self.T), rem_base,
                           0 if self.rem is None else len(self.rem), _p(self.rem), _p(self.rem_present))


def order_keys(policy, q: QueueArrays, t: TableArrays):
    n = len(q.agent)
    k = np.zeros((3, n), np.float64)
    lib().kxo_order_keys(POLICY.get(policy, policy), C.byref(q.view), C.byref(t.view),
                         _p(k[0]), _p(k[1]), _p(k[2]))
    return k


def sort(policy, q: QueueArrays, t: TableArrays, n_pools: int):
    n = len(q.agent)
    perm = np.zeros(n, np.uint32)
    offs = np.zeros(n_pools + 1, np.int64)
    rc = lib().kxo_sort(POLICY.get(policy, policy), C.byref(q.view), C.byref(t.view), n_pools,
                        _p(perm), _p(offs))
    assert rc == 0
    return perm, offs


class Ledger:
    def __init__(self, id_, slot_len, cap):
        self.h = lib().kxo_ledger_new(id_, slot_len, cap)

    def __del__(self):
        if getattr(self, "h", None):
            lib().kxo_ledger_free(self.h)

    def try_place(self, P, k, t0, T):
        f, pk, v = C.c_int32(), C.c_double(), C.c_int64()
        lib().kxo_try_place(self.h, P, k, t0, T, C.byref(f), C.byref(pk), C.byref(v))
        return bool(f.value), pk.value, v.value

    def commit(self, uid, P, k, t0, T):
        return lib().kxo_commit(self.h, uid, P, k, t0, T)

    def finish(self, uid, end):
        return lib().kxo_finish(self.h, uid, end)

    def gc(self, now):
        lib().kxo_gc(self.h, now)

    def slots(self):
        cap = 4096
        s = np.zeros(cap, np.int64)
        u = np.zeros(cap, np.float64)
        n = lib().kxo_ledger_dump(self.h, _p(s), _p(u), cap)
        return {int(a): float(b) for a, b in zip(s[:n], u[:n])}

    def active(self):
        return lib().kxo_ledger_active(self.h)


class PoolState:
    """One pool's Dispatcher + engine live view for the oracle dispatch loop."""

    def __init__(self, ids, caps, ks, max_batch, slot_len=0.5, watermark=0.85, oracle_T=False):
        n = len(ids)
        self.id = np.ascontiguousarray(ids, np.int32)
        self.cap = np.ascontiguousarray(caps, np.float64)
        self.k = np.ascontiguousarray(ks, np.float64)
        self.max_batch = np.ascontiguousarray(max_batch, np.int32)
        self.live_kv = np.zeros(n, np.float64)
        self.running = np.zeros(n, np.int32)
        self.waiting = np.zeros(n, np.int32)
        self.suspended = np.zeros(n, np.uint8)
        self.ledgers = [Ledger(int(ids[i]), slot_len, float(caps[i])) for i in range(n)]
        self._lp = (C.c_void_p * n)(*[l.h for l in self.ledgers])
        self.view = Pool(n, _p(self.id), _p(self.cap), _p(self.k), _p(self.max_batch),
                         _p(self.live_kv), _p(self.running), _p(self.waiting), _p(self.suspended),
                         C.cast(self._lp, C.c_void_p), slot_len, watermark, int(oracle_T))

    def set_live(self, live_kv, running, waiting=None):
        self.live_kv[:] = live_kv
        self.running[:] = running
        if waiting is not None:
            self.waiting[:] = waiting

    # ---- waiting lists (round_robin / static_threshold) ----
    wcap = 0
    rr_next = 0
    round = 0

    def set_waiting(self, q: "QueueArrays", inst_pos, wcap=4096):
        """Replaces every waiting list: entry j joins instance inst_pos[j]."""
        n = len(self.id)
        self.wcap = wcap
        self.wrec = np.zeros(n * wcap, WAITREC)
        self.waiting[:] = 0
        for j, i in enumerate(np.asarray(inst_pos)):
            r = self.wrec[int(i) * wcap + int(self.waiting[i])]
            r["app_start"], r["queue_enter"] = q.app_start[j], q.queue_enter[j]
            r["msg"], r["uid"], r["prompt"] = q.msg_key[j], q.uid[j], q.prompt[j]
            r["kept"] = 0 if q.kept is None else q.kept[j]
            r["qidx"], r["agent"], r["round"] = -1, q.agent[j], -1
            self.wrec[int(i) * wcap + int(self.waiting[i])] = r
            self.waiting[i] += 1

    def waiting_uids(self, i):
        return self.wrec["uid"][i * self.wcap:i * self.wcap + int(self.waiting[i])].copy()

    def dispatch_round_waiting(self, dispatch_policy, sched_policy, q: "QueueArrays", t: "TableArrays", perm,
                               now, static_thr=0.90, pool_index=0, row_cap=1 << 16):
        if self.wcap == 0:
            self.set_waiting(q, [])
        self.round += 1
        perm = np.ascontiguousarray(perm, np.uint32)
        rows = np.zeros(row_cap, DECISION)
        adm = np.zeros(row_cap, ADMISSION)
        rr = C.c_int64(self.rr_next)
        nadm = C.c_int64()
        st = C.c_int32()
        n = lib().kxo_dispatch_round_waiting(
            C.byref(self.view), DISPATCH_POLICY.get(dispatch_policy, dispatch_policy), static_thr,
            POLICY.get(sched_policy, sched_policy), C.byref(rr), self.wrec.ctypes.data, self.wcap, self.round,
            C.byref(q.view), C.byref(t.view), _p(perm), len(perm), now, pool_index, rows.ctypes.data, row_cap,
            adm.ctypes.data, row_cap, C.byref(nadm), C.byref(st))
        self.rr_next = rr.value
        return rows[:n], adm[:nadm.value], st.value

    def dispatch_round(self, q: QueueArrays, t: TableArrays, perm, now, pool_index=0, row_cap=1 << 16):
        perm = np.ascontiguousarray(perm, np.uint32)
        rows = np.zeros(row_cap, DECISION)
        cand = np.zeros(row_cap * len(self.id), np.float64)
        st = C.c_int32()
        n = lib().kxo_dispatch_round(C.byref(self.view), C.byref(q.view), C.byref(t.view), _p(perm),
                                     len(perm), now, pool_index, rows.ctypes.data, _p(cand), row_cap,
                                     C.byref(st))
        return rows[:n], cand[:n * len(self.id)].reshape(n, len(self.id)), st.value


def finalize(off, parent, prompt, target, prefill, decode, uid_base=1):
    off = np.ascontiguousarray(off, np.int64)
    parent = np.ascontiguousarray(parent, np.int32)
    prompt = np.ascontiguousarray(prompt, np.int64)
    target = np.ascontiguousarray(target, np.int64)
    n = len(parent)
    uid = np.zeros(n, np.uint64)
    pure = np.zeros(n, np.float64)
    rem = np.zeros(n, np.float64)
    rc = lib().kxo_finalize(len(off) - 1, _p(off), _p(parent), _p(prompt), _p(target), prefill,
                            decode, uid_base, _p(uid), _p(pure), _p(rem))
    assert rc == 0
    return uid, pure, rem


def record_remaining(off, es, ee):
    off = np.ascontiguousarray(off, np.int64)
    es = np.ascontiguousarray(es, np.float64)
    ee = np.ascontiguousarray(ee, np.float64)
    fin = np.zeros(len(off) - 1, np.float64)
    smp = np.zeros(len(es), np.float64)
    lib().kxo_record_remaining(len(off) - 1, _p(off), _p(es), _p(ee), _p(fin), _p(smp))
    return fin, smp


def quantile(sorted_vals, p):
    a = np.ascontiguousarray(sorted_vals, np.float64)
    return lib().kxo_quantile_sorted(_p(a), len(a), p)


def mode_estimate(sorted_vals, min_samples=16):
    a = np.ascontiguousarray(sorted_vals, np.float64)
    fb = C.c_int()
    v = lib().kxo_mode_estimate(_p(a), len(a), min_samples, C.byref(fb))
    return v, bool(fb.value)


def wasserstein(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return lib().kxo_wasserstein_1d(_p(a), len(a), _p(b), len(b))


def median_anchor_distance(coords, anchor):
    c = np.ascontiguousarray(coords, np.float64)
    return lib().kxo_median_anchor_distance(_p(c), len(c), anchor)


def pairwise_accuracy(agent, rem, present=None, scope_all=False):
    a = np.ascontiguousarray(agent, np.int32)
    r = np.ascontiguousarray(rem, np.float64)
    p = None if present is None else np.ascontiguousarray(present, np.uint8)
    acc, pairs = C.c_double(), C.c_uint64()
    rc = lib().kxo_pairwise_accuracy(len(a), _p(a), _p(r), _p(p), int(scope_all), C.byref(acc), C.byref(pairs))
    return (None if rc else acc.value), pairs.value


class Dist:
    """EmpiricalDistribution restatement (kxo_dist)."""

    def __init__(self, min_samples=16, threshold=0.05, window_cap=0):
        self.h = lib().kxo_dist_new(min_samples, threshold, window_cap)

    def __del__(self):
        if getattr(self, "h", None):
            lib().kxo_dist_free(self.h)
            self.h = None

    def add(self, v):
        return lib().kxo_dist_add(self.h, float(v))

    def read(self):
        tot, cv, last = C.c_uint64(), C.c_int32(), C.c_double()
        n = lib().kxo_dist_read(self.h, None, 0, C.byref(tot), C.byref(cv), C.byref(last))
        out = np.zeros(n, np.float64)
        lib().kxo_dist_read(self.h, _p(out), n, C.byref(tot), C.byref(cv), C.byref(last))
        return out, tot.value, cv.value, last.value


def profiler_replay(n_agents, off, agent, es, ee, exec_cfg=(16, 0.05, 0), rem_cfg=(16, 0.05, 4096)):
    """LatencyProfiler replay: record_execution of every record, then
    record_remaining per workflow; returns (exec dists, rem dists, newly[w])."""
    ex = [Dist(*exec_cfg) for _ in range(n_agents)]
    rm = [Dist(*rem_cfg) for _ in range(n_agents)]
    newly = np.zeros(len(off) - 1, np.uint8)
    for w in range(len(off) - 1):
        b, e = int(off[w]), int(off[w + 1])
        for r in range(b, e):
            assert ex[agent[r]].add(ee[r] - es[r]) >= 0
        if b == e:
            continue
        fin = ee[b]
        for r in range(b, e):
            fin = ee[r] if fin < ee[r] else fin
        for r in range(b, e):
            got = rm[agent[r]].add(fin - es[r])
            assert got >= 0
            if got == 1:
                newly[w] = 1
    return ex, rm, newly
