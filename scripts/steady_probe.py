"""Serving-loop breakdown (bench.py's e2e_steady step, host-timed parts):
state restore, tick, decision-log read, pop of the admitted requests and
enqueue of as many arrivals, for one bench configuration.

    python scripts/steady_probe.py [C4]
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2508_06948_b200 import workload as W  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "C4"
w = W.build_workload(config, 0)
s = bench.make_sched(w, 0)
snap, arr = w.snap, w.arrivals
s.upload(snap.agent, snap.prompt, snap.app_start, snap.queue_enter, snap.msg_key, snap.uid)
T = {}


def tm(name, f):
    s.synchronize()
    t = time.perf_counter()
    r = f()
    s.synchronize()
    T.setdefault(name, []).append(time.perf_counter() - t)
    return r


pos = 0
for it in range(6):
    tm("restore", s.restore)
    tm("tick", lambda: s.tick(w.now))
    r, c = tm("fetch", s.fetch_dispatch)
    m = int(sum(int(x["admitted"].sum()) for x in r))
    tm("remove", s.remove_admitted)
    sl = slice(pos, pos + m)
    pos += m
    tm("enqueue", lambda: s.enqueue(arr.agent[sl], arr.prompt[sl], arr.app_start[sl], arr.queue_enter[sl],
                                    arr.msg_key[sl], arr.uid[sl]))
for k, v in T.items():
    print(f"{k:8s} {1e3 * np.median(v[1:]):8.3f} ms")
