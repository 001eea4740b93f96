import sys, time, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
import bench
import paper_2508_06948_b200 as kx
from paper_2508_06948_b200 import workload as W
snap, insts, live, running, commits = bench.build_c4(0)
s = bench.make_sched(snap, insts, live, running, commits, 0)
s.upload(snap.agent, snap.prompt, snap.app_start, snap.queue_enter, snap.msg_key, snap.uid)
arr = W.snapshot(n_pools=8, per_pool=8192, seed=101, msg_base=8_000_000, uid_base=100_000_001)
T = {}
def tm(name, f):
    s.synchronize(); t = time.perf_counter(); r = f(); s.synchronize(); T.setdefault(name, []).append(time.perf_counter() - t); return r
pos = 0
for it in range(6):
    tm("restore", s.restore)
    tm("tick", lambda: s.tick(bench.NOW))
    r, c = tm("fetch", s.fetch_dispatch)
    m = int(sum(int(x["admitted"].sum()) for x in r))
    tm("remove", s.remove_admitted)
    sl = slice(pos, pos + m); pos += m
    tm("enqueue", lambda: s.enqueue(arr.agent[sl], arr.prompt[sl], arr.app_start[sl], arr.queue_enter[sl], arr.msg_key[sl], arr.uid[sl]))
for k, v in T.items():
    print(f"{k:8s} {1e3*np.median(v[1:]):8.3f} ms")
