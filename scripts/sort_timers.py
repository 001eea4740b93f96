"""Per-pass tile phase breakdown of the radix passes inside the C4 tick
(library built with -DKX_SORT_TIMERS=1; scripts/gpu_sort_timers.sh)."""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2508_06948_b200 import workload as W  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "C4"
ticks = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = W.build_workload(config, 0, arrivals=1024)
s = bench.make_sched(w, 0)
snap = w.snap
s.upload(snap.agent, snap.prompt, snap.app_start, snap.queue_enter, snap.msg_key, snap.uid)
buf = (C.c_uint64 * 64)()
for overlap in (True, False):
    s.lib.kx_debug_sort_timers(buf, 1)
    for _ in range(ticks):
        s.restore()
        if overlap:
            s.tick(w.now)
        else:
            s.order()
    s.synchronize()
    s.lib.kx_debug_sort_timers(buf, 1)
    t = list(buf)
    print("-- tick (overlapped dispatch)" if overlap else "-- order alone")
    for p in range(4):
        g = t[p * 8:p * 8 + 8]
        n = max(g[5], 1)
        print(f"pass {p}: tiles/launch {g[5] / ticks:.0f}  per-tile ns: load {g[0] / n:.0f} rank {g[1] / n:.0f} "
              f"scan+lookback {g[2] / n:.0f} stage {g[3] / n:.0f} write {g[4] / n:.0f}")
