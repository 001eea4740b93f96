import sys, time, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import kxf, paper_2508_06948_b200 as kx
from helpers import dispatch_rounds, round_queue
d = kxf.read("dispatch_small.kxf")
ids = d["inst_id"]
inst = [kx.InstanceProfile(id=int(ids[i]), pool=0, capacity_tokens=float(d["inst_cap"][i]),
                           decode_rate=float(d["inst_k"][i]), max_batch=int(d["inst_max_batch"][i])) for i in range(len(ids))]
s = kx.DeviceScheduler(inst, n_pools=1, queue_capacity=4096, max_agents=16)
n_agents = len(d["agent_T"])
s.set_agent_tables(np.zeros(n_agents, np.int32), expected_T=d["agent_T"])
s.set_scheduler("fcfs")
for i, uid, P, t0, T in zip(d["pre_inst"], d["pre_uid"], d["pre_P"], d["pre_t0"], d["pre_T"]):
    k = float(d["inst_k"][list(ids).index(int(i))])
    s.commit(int(i), int(uid), P, k, t0, T)
for r, rd in dispatch_rounds(d):
    q = round_queue(rd)
    s.upload(q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid)
    s.set_live(rd["live_kv"], rd["running"], rd["waiting"])
    t0 = time.time()
    s.tick(float(rd["now"][0]))
    try:
        rows, cand = s.fetch_dispatch()
        print("round", r, "ok", len(rows[0]), "rows", time.time() - t0)
    except Exception as e:
        print("round", r, "ERR", e, time.time() - t0, "n", len(q.agent))
        break
    for iid, uid, end in zip(rd["fin_inst"], rd["fin_uid"], rd["fin_end"]):
        s.on_request_finished(int(iid), int(uid), float(end))
import ctypes as C
buf = (C.c_uint64 * 16)()
s.lib.kx_debug_dispatch_timers(buf)
print("timeout: observed", buf[12], "target", buf[13], "ptr", hex(buf[14]))
print("order markers: keygen entered", buf[0], "keygen signalled", buf[1], "signal kernel", buf[2])
