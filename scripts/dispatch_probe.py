"""Dispatch-kernel probe: one bench configuration (C1-C4, built exactly as
bench.py builds it), ticked a few times with the library's phase profiler
on; prints per-phase device times, then the same round without the overlap
(full order first, then the dispatch alone). With a KX_DISPATCH_TIMERS
build it also prints pool 0's in-kernel stamps.

    python scripts/dispatch_probe.py C4 3
"""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2508_06948_b200 import workload as W  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "C4"
ticks = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = W.build_workload(config, 0, arrivals=1024)
s = bench.make_sched(w, 0)
snap = w.snap
s.upload(snap.agent, snap.prompt, snap.app_start, snap.queue_enter, snap.msg_key, snap.uid)


STAGES = ["load_head+loop", "row wait", "fence+row loads", "fix / rr eval+select", "select / rr commit", "staging",
          "ledger booking", "admit state", "fence+publish", "rr decisions", "exact-path heads"]


def trace():
    if not hasattr(s.lib, "kx_debug_dispatch_trace"):
        return
    buf = (C.c_uint64 * 128)()
    s.lib.kx_debug_dispatch_trace(buf)
    t = list(buf)
    if not any(t):
        return
    names = ["top", "eval", "flags", "argmin", "staging", "commit", "admit", "publish", "load_head"]
    for it in range(8):
        row = t[it * 16: it * 16 + 9]
        if not all(row):
            continue
        d = [row[k] - row[k - 1] for k in range(1, 9)]
        nxt = t[(it + 1) * 16] - row[8] if it < 7 and t[(it + 1) * 16] else 0
        print("  step trace cycles: " + " ".join(f"{n} {v}" for n, v in zip(names[1:], d)) + f" | to next top {nxt}")


def timers():
    trace()
    buf = (C.c_uint64 * 16)()
    if hasattr(s.lib, "kx_debug_dispatch_stages"):
        s.lib.kx_debug_dispatch_stages(buf)
        st = list(buf)
        if st[12]:
            kd = (C.c_uint64 * 1)()
            s.lib.kx_debug_keys_done(kd)
            pt = (C.c_uint64 * 128)()
            s.lib.kx_debug_dispatch_pool_times(pt)
            npool = len(w.snap.pool_names) if hasattr(w.snap, "pool_names") else w.snap.n_pools
            starts = [(pt[i] - kd[0]) / 1e3 for i in range(npool)]
            ends = [(pt[64 + i] - kd[0]) / 1e3 for i in range(npool)]
            print("  phase-3 per pool, us after keygen: start " + " ".join(f"{x:.1f}" for x in starts) +
                  " | end " + " ".join(f"{x:.1f}" for x in ends))
            print(f"  phase-3 prologue us: start after keygen {(st[12] - kd[0]) / 1e3:.2f}, ring staging "
                  f"{(st[13] - st[12]) / 1e3:.2f}, umax {(st[14] - st[13]) / 1e3:.2f}, prefix sort "
                  f"{(st[15] - st[14]) / 1e3:.2f} (network {(st[11] - st[14]) / 1e3:.2f})")
        if any(st[:12]):
            s.lib.kx_debug_dispatch_timers(buf)
            n = max(1, list(buf)[5])
            print("  resolver stage cycles per record: " + ", ".join(f"{k} {v / n:.0f}" for k, v in zip(STAGES, st)))
    if hasattr(s.lib, "kx_debug_dispatch_timers"):
        s.lib.kx_debug_dispatch_timers(buf)
        t = list(buf)
        if t[0]:
            print(f"  chain kernel (pool 0) us: prologue {(t[1] - t[0]) / 1e3:.2f} loop {(t[2] - t[1]) / 1e3:.2f} "
                  f"epilogue {(t[3] - t[2]) / 1e3:.2f} records {t[5]}  "
                  f"us/record {(t[2] - t[1]) / 1e3 / max(1, t[5]):.3f}")
            n = max(1, t[10])
            print(f"  resolver cycles per admission ({t[10]}): head+row wait {t[6] / n:.0f} "
                  f"fix {t[7] / n:.0f} ({t[11] / n:.2f} entries) select {t[8] / n:.0f} commit {t[9] / n:.0f}")


s.profile(True)
for _ in range(ticks):
    s.restore()
    s.tick(w.now)
s.synchronize()
rows, _ = s.fetch_dispatch()
print(config, "decisions", sum(len(r) for r in rows), "admitted", sum(int(r["admitted"].sum()) for r in rows))
for k, v in s.profile_read().items():
    print(f"{k:14s} {v['ms'] / ticks:8.3f} ms/tick  launches {v['launches'] / ticks:.0f}")
timers()

s.profile(False)
s.profile(True)
for _ in range(ticks):
    s.restore()
    s.order()
    s.dispatch_round(w.now)
s.synchronize()
print("-- order, then dispatch (no overlap)")
for k, v in s.profile_read().items():
    print(f"{k:14s} {v['ms'] / ticks:8.3f} ms/tick  launches {v['launches'] / ticks:.0f}")
timers()

s.profile(False)
s.capture_begin()
s.restore()
s.tick(w.now)
s.capture_end()
for _ in range(ticks):
    s.graph_launch()
s.synchronize()
print("-- graph replay (the bench's step)")
timers()
s.graph_release()
