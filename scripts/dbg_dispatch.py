import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import kxf, paper_2508_06948_b200 as kx
from helpers import dispatch_rounds, round_queue
d = kxf.read("dispatch_small.kxf")
ids = d["inst_id"]
for mode in ["tick","order+dispatch"]:
    inst = [kx.InstanceProfile(id=int(ids[i]), pool=0, capacity_tokens=float(d["inst_cap"][i]),
                               decode_rate=float(d["inst_k"][i]), max_batch=int(d["inst_max_batch"][i])) for i in range(len(ids))]
    s = kx.DeviceScheduler(inst, n_pools=1, queue_capacity=4096, max_agents=16)
    n_agents = len(d["agent_T"])
    s.set_agent_tables(np.zeros(n_agents, np.int32), expected_T=d["agent_T"])
    s.set_scheduler("fcfs")
    for i, uid, P, t0, T in zip(d["pre_inst"], d["pre_uid"], d["pre_P"], d["pre_t0"], d["pre_T"]):
        k = float(d["inst_k"][list(ids).index(int(i))])
        s.commit(int(i), int(uid), P, k, t0, T)
    r, rd = next(iter(dispatch_rounds(d)))
    q = round_queue(rd)
    s.upload(q.agent, q.prompt, q.app_start, q.queue_enter, q.msg_key, q.uid)
    s.set_live(rd["live_kv"], rd["running"], rd["waiting"])
    if mode=="tick": s.tick(float(rd["now"][0]))
    else:
        s.order(); s.dispatch(float(rd["now"][0])) if hasattr(s,'dispatch') else s.dispatch_round(float(rd["now"][0]))
    rows, cand = s.fetch_dispatch()
    rows=rows[0]
    print(mode, "n", len(rows), "exp", len(rd["dec_uid"]))
    print(" uid", rows["uid"][:6], "exp", rd["dec_uid"][:6])
    print(" tgt", rows["target"][:6], "exp", rd["dec_target"][:6])
    print(" qidx", rows["queue_index"][:6], "agent", rows["agent"][:6])
