import ctypes as C, sys
sys.path.insert(0, '.')
import bench
from paper_2508_06948_b200 import workload as W
for cfg in ['C3', 'C4', 'C2', 'C1']:
    w = W.build_workload(cfg, 0, arrivals=16)
    s = bench.make_sched(w, 0)
    snap = w.snap
    s.upload(snap.agent, snap.prompt, snap.app_start, snap.queue_enter, snap.msg_key, snap.uid)
    cnt = (C.c_uint64 * 2)()
    s.lib.kx_debug_dispatch_counts(cnt, 1)
    for _ in range(3):
        s.restore(); s.tick(w.now)
    s.synchronize()
    s.lib.kx_debug_dispatch_counts(cnt, 1)
    rows, _ = s.fetch_dispatch()
    print(cfg, 'rr decisions', cnt[0] // 3, 'exact-path heads', cnt[1] // 3, 'rows', sum(len(r) for r in rows), 'admitted', sum(int(r['admitted'].sum()) for r in rows))
