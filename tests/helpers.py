"""Fixture plumbing shared by the oracle (CPU) and device (GPU) tests."""
from __future__ import annotations

import numpy as np

import kxf
import oracle_ffi as O

POLICIES = ["kairos", "fcfs", "topo_depth", "oracle"]


def order_fixture(name):
    d = kxf.read(name)
    q = O.QueueArrays(d["agent"], d["prompt"], d["app_start"], d["queue_enter"], d["msg_key"], d["uid"])
    t = O.TableArrays(d["agent_pool"], d["pk"], d["depth"], None, int(d["rem_base"][0]), d["rem"],
                      d["rem_present"])
    return d, q, t, int(d["n_pools"][0])


def dispatch_rounds(d):
    r = 0
    while f"r{r}.now" in d:
        p = f"r{r}."
        yield r, {k[len(p):]: v for k, v in d.items() if k.startswith(p)}
        r += 1


def round_queue(rd):
    return O.QueueArrays(rd["q.agent"], rd["q.prompt"], rd["q.app_start"], rd["q.queue_enter"],
                         rd["q.msg_key"], rd["q.uid"])


def ledger_expect(rd, inst_id):
    m = rd["ledger_inst"] == inst_id
    return {int(s): float(u) for s, u in zip(rd["ledger_slot"][m], rd["ledger_used"][m])}


def bits(x):
    return np.asarray(x, np.float64).view(np.uint64)


def random_queue(rng, n, n_agents, n_pools, tie_grain=0.0, msg_space=None, uid_base=1):
    """Random queue + tables; tie_grain > 0 quantises times to force ties."""
    agent = rng.integers(0, n_agents, n).astype(np.int32)
    app = rng.uniform(0.0, 10.0, n)
    qe = app + rng.uniform(0.0, 5.0, n)
    if tie_grain > 0:
        app = np.floor(app / tie_grain) * tie_grain
        qe = np.floor(qe / tie_grain) * tie_grain
    ms = msg_space or max(1, n // 3)
    msg = rng.integers(0, ms, n).astype(np.uint64)
    uid = (uid_base + rng.permutation(n)).astype(np.uint64)
    prompt = rng.integers(1, 300, n).astype(np.int64)
    pool = (np.arange(n_agents) % n_pools).astype(np.int32)
    pk = np.round(rng.uniform(0.0, 5.0, n_agents), 1)
    depth = rng.integers(1, 6, n_agents).astype(np.int32)
    T = rng.uniform(0.2, 8.0, n_agents)
    rem = np.round(rng.uniform(0.0, 20.0, n), 2)
    present = (rng.uniform(size=n) < 0.9).astype(np.uint8)
    # remaining table dense over [uid_base, uid_base + n)
    rem_tab = np.zeros(n)
    pres_tab = np.zeros(n, np.uint8)
    rem_tab[(uid - uid_base).astype(np.int64)] = rem
    pres_tab[(uid - uid_base).astype(np.int64)] = present
    q = O.QueueArrays(agent, prompt, app, qe, msg, uid)
    t = O.TableArrays(pool, pk, depth, T, uid_base, rem_tab, pres_tab)
    return q, t
