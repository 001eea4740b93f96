"""Dispatch-kernel probe: the C4 instance layout (8 pools x 32 instances,
pre-loaded ledgers) over a smaller queue, for ncu captures of
k_dispatch_timeslot. Prints per-phase device times."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2508_06948_b200 import workload as W  # noqa: E402

per_pool = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
ticks = int(sys.argv[2]) if len(sys.argv) > 2 else 3
snap = W.snapshot(n_pools=8, per_pool=per_pool, seed=1)
insts = W.instances(8, 32)
live, running, commits = W.preload(insts, seed=7, now=bench.NOW)
s = bench.make_sched(snap, insts, live, running, commits, 0)
s.upload(snap.agent, snap.prompt, snap.app_start, snap.queue_enter, snap.msg_key, snap.uid)
s.profile(True)
for _ in range(ticks):
    s.restore()
    s.tick(bench.NOW)
s.synchronize()
rows, _ = s.fetch_dispatch()
print("decisions", sum(len(r) for r in rows), "admitted", sum(int(r["admitted"].sum()) for r in rows))
for k, v in s.profile_read().items():
    print(f"{k:14s} {v['ms'] / ticks:8.3f} ms/tick  launches {v['launches'] / ticks:.0f}")

# the same round without the overlap: full order first, then the dispatch alone
s.profile(False)
s.profile(True)
for _ in range(ticks):
    s.restore()
    s.order()
    s.dispatch_round(bench.NOW)
s.synchronize()
print("-- order, then dispatch (no overlap)")
for k, v in s.profile_read().items():
    print(f"{k:14s} {v['ms'] / ticks:8.3f} ms/tick  launches {v['launches'] / ticks:.0f}")

import ctypes as C
buf = (C.c_uint64 * 16)()
if hasattr(s.lib, "kx_debug_dispatch_timers"):
    s.lib.kx_debug_dispatch_timers(buf)
    t = list(buf)
    print("batch kernel (pool 0) us: stage", (t[1] - t[0]) / 1e3, "loop", (t[2] - t[1]) / 1e3,
          "epilogue", (t[3] - t[2]) / 1e3, "writeback", (t[4] - t[3]) / 1e3, "rows", t[5])
    print("epilogue us: flush", (t[13] - t[2]) / 1e3, "gc slots", (t[14] - t[13]) / 1e3, "active gc",
          (t[15] - t[14]) / 1e3, "rest", (t[3] - t[15]) / 1e3)
    print("cycles: phaseA", t[6], "phaseB", t[7], "batches", t[11], "fix", t[8], "select", t[9], "stage", t[10], "commit", t[12])
