"""ctypes wrapper of kxref_sim_run: the UNMODIFIED reference Simulator
(oracle/_ref/libkxref.so). TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
SO = ROOT / "oracle" / "_ref" / "libkxref.so"
# the drop-in build: the same reference Simulator with its time-slot dispatch
# round and Dispatcher events on the B200 (oracle/dropin_sim.cpp)
DROPIN_SO = ROOT / "oracle" / "_ref" / "libkxdropin.so"
SCHED = {"kairos": 0, "fcfs": 1, "topo_depth": 2, "oracle": 3}
DISPATCH = {"time_slot": 0, "round_robin": 1, "static_threshold": 2}
_libs = {}


def lib(so=SO):
    if so not in _libs:
        if not Path(so).exists():
            subprocess.run(["make", "-C", str(ROOT / "oracle")], check=True, capture_output=True)
        L = C.CDLL(str(so))
        L.kxref_sim_run.restype = C.c_int
        _libs[so] = L
    return _libs[so]


def run(batch_one, instances, scheduler, dispatcher, topo_depth, period=0.1, recompute=1.0, so=SO):
    """One replica through the reference Simulator (the stock build, or
    with so=DROPIN_SO the drop-in build); returns a dict like
    engine.run_replicas."""
    b = batch_one
    W = len(b["arrival"])
    Cn = len(b["agent"])
    cols = [np.ascontiguousarray(b[k], dt) for k, dt in [
        ("arrival", np.float64), ("wf_offsets", np.int64), ("agent", np.int32), ("parent", np.int32),
        ("prompt", np.int64), ("target", np.int64), ("pure_exec", np.float64), ("remaining", np.float64),
        ("uid", np.uint64)]]
    ids = np.array([p.id for p in instances], np.int32)
    caps = np.array([p.capacity_tokens for p in instances])
    ks = np.array([p.decode_rate for p in instances])
    pf = np.array([p.prefill_rate for p in instances])
    mb = np.array([p.max_batch for p in instances], np.int32)
    depth = np.ascontiguousarray(topo_depth, np.int32)
    out = dict(uid=np.zeros(Cn, np.uint64), exec_start=np.zeros(Cn), exec_end=np.zeros(Cn),
               instance=np.zeros(Cn, np.int32), first_enqueue=np.zeros(Cn), queue_seconds=np.zeros(Cn),
               episodes=np.zeros(Cn, np.int32), preemptions=np.zeros(Cn, np.int32),
               wf_index=np.zeros(W, np.int64), wf_finish=np.zeros(W), wf_output_tokens=np.zeros(W, np.int64),
               wf_calls=np.zeros(W, np.int64), scalars=np.zeros(18))
    pk = np.zeros(10)
    version = C.c_int64(0)
    nc, nw = C.c_int64(), C.c_int64()
    d = dispatcher
    P = C.c_void_p
    args = [C.c_int64(W)] + [P(c.ctypes.data) for c in cols] + [
        C.c_int(len(instances)), P(ids.ctypes.data), P(caps.ctypes.data), P(ks.ctypes.data),
        P(pf.ctypes.data), P(mb.ctypes.data), C.c_int(SCHED[scheduler]), C.c_int(DISPATCH[d.policy]),
        C.c_int(int(d.oracle_expected_time)), C.c_double(d.slot_len), C.c_double(d.resume_watermark),
        C.c_double(d.static_threshold), C.c_double(d.default_expected_time), C.c_double(period),
        C.c_double(recompute), P(depth.ctypes.data)] + [P(v.ctypes.data) for v in out.values()] + [
        C.byref(nc), C.byref(nw), P(pk.ctypes.data), C.byref(version)]
    rc = lib(so).kxref_sim_run(*args)
    assert rc == 0, "reference simulation failed"
    out["n_calls"] = nc.value
    out["n_wf"] = nw.value
    out["priority_keys"] = pk
    out["table_version"] = version.value
    return out


def realize(cfg, prefill=8000.0, decode=50.0):
    """The reference realize() (workload.cpp:319-372) on the same
    WorkloadConfig (built through the C ABI struct, agent i named "a<i>");
    returns a dict of flat arrays, or raises ValueError with the reference's
    exception message."""
    from paper_2508_06948_b200 import workload as W
    L = lib()
    P = C.c_void_p
    L.kxref_realize.restype = P
    L.kxref_realize.argtypes = [P, C.c_uint64, C.c_double, C.c_double]
    L.kxref_realize_error.restype = C.c_char_p
    L.kxref_realize_error.argtypes = [P]
    L.kxref_realize_sizes.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.kxref_realize_copy.argtypes = [P] * 11
    L.kxref_realize_free.argtypes = [P]
    c, keep, names = W.workload_abi(cfg)
    h = L.kxref_realize(C.addressof(c), cfg.seed, prefill, decode)
    try:
        err = L.kxref_realize_error(h).decode()
        if err:
            raise ValueError(err)
        nw, nc = C.c_int64(), C.c_int64()
        L.kxref_realize_sizes(h, C.byref(nw), C.byref(nc))
        Wn, N = nw.value, nc.value
        out = dict(arrival=np.zeros(Wn), wf_offsets=np.zeros(Wn + 1, np.int64), agent=np.zeros(N, np.int32),
                   parent=np.zeros(N, np.int32), prompt=np.zeros(N, np.int64), target=np.zeros(N, np.int64),
                   pure_exec=np.zeros(N), remaining=np.zeros(N), uid=np.zeros(N, np.uint64),
                   rem_map=np.zeros(N))
        L.kxref_realize_copy(h, *[v.ctypes.data for v in out.values()])
    finally:
        L.kxref_realize_free(h)
    return out
