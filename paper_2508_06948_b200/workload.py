"""Synthetic queue snapshots with the shape of the reference's workloads.

The reference synthesises traces with realize() (workload.cpp:319-372) from
the QA / RG / CG templates (workload.cpp:462-560). For million-request queue
snapshots this module draws the same workflow
shapes and token-length distributions vectorised with numpy — synthetic data
of the reference's shape, not a bit-replica of its mt19937 stream (the
parity tests use the reference's own realize() through golden fixtures).

Snapshot semantics: every call of each workflow is queued, with
queue_enter = app_start + sum of its ancestors' pure_exec, app_start drawn
uniformly over a burst window ("excessive load").
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# (name, prompt lo, prompt hi, output median, sigma, cap) — workload.cpp:462-531
AGENTS = [
    ("Router", 40, 80, 10.0, 0.25, 40),
    ("Math", 60, 120, 70.0, 0.35, 400),
    ("Humanities", 60, 120, 240.0, 0.35, 900),
    ("Researcher", 80, 160, 150.0, 0.35, 700),
    ("Writer", 120, 240, 380.0, 0.30, 1100),
    ("ProductManager", 80, 160, 70.0, 0.35, 300),
    ("Architect", 80, 160, 110.0, 0.35, 450),
    ("ProjectManager", 80, 160, 50.0, 0.30, 200),
    ("Engineer", 100, 200, 300.0, 0.40, 1100),
    ("QAEngineer", 80, 160, 40.0, 0.30, 160),
]
A = {n[0]: i for i, n in enumerate(AGENTS)}

# Workflow templates (chains) with probabilities: QA routes 50/50, RG is a
# fixed chain, CG's QA->Engineer feedback fires with p=0.3 up to 3 times
# (workload.cpp:247-256, 538-541). Co-located apps are equally weighted.
_CG = ["ProductManager", "Architect", "ProjectManager", "Engineer", "QAEngineer"]
TEMPLATES = [
    (["Router", "Math"], 1 / 6),
    (["Router", "Humanities"], 1 / 6),
    (["Researcher", "Writer"], 1 / 3),
    (_CG, 1 / 3 * 0.7),
    (_CG + ["Engineer", "QAEngineer"], 1 / 3 * 0.3 * 0.7),
    (_CG + ["Engineer", "QAEngineer"] * 2, 1 / 3 * 0.09 * 0.7),
    (_CG + ["Engineer", "QAEngineer"] * 3, 1 / 3 * 0.027),
]


@dataclass
class QueueSnapshot:
    agent: np.ndarray        # int32 dense agent index (pool-major: pool p owns agents [10p, 10p+10))
    prompt: np.ndarray       # int64
    app_start: np.ndarray    # f64
    queue_enter: np.ndarray  # f64
    msg_counter: np.ndarray  # u64: msg_id is "m-<counter>"
    msg_key: np.ndarray      # u64: lexicographic key of msg_id
    uid: np.ndarray          # u64
    pure_exec: np.ndarray    # f64
    agent_pool: np.ndarray   # int32 per agent
    agent_names: list
    priority_key: np.ndarray  # per agent (cold-start median applied)
    pk_known: np.ndarray      # uint8: agent present in the priority table
    topo_depth: np.ndarray    # per agent
    expected_T: np.ndarray    # per agent
    n_pools: int

    @property
    def n(self):
        return len(self.agent)


def msg_key_decimal(counter: np.ndarray) -> np.ndarray:
    """Order-preserving u64 key of the strings "m-<counter>" (lexicographic,
    SURVEY H1): digits encoded base 11 (digit+1, 0 = end), 18 digits max.
    Same encoding as kairos_b200::MsgKeyer (include/kairos_b200.hpp)."""
    c = counter.astype(np.uint64)
    ndig = np.ones(len(c), np.int64)
    t = c // np.uint64(10)
    while np.any(t > 0):
        ndig += (t > 0)
        t //= np.uint64(10)
    if len(c) and ndig.max() > 18:
        raise ValueError("msg counter with more than 18 digits")
    inner = np.zeros(len(c), np.uint64)
    pw = np.uint64(1)
    t = c.copy()
    for i in range(int(ndig.max()) if len(c) else 0):
        inner += np.where(i < ndig, (t % np.uint64(10) + np.uint64(1)) * pw, np.uint64(0))
        t //= np.uint64(10)
        pw *= np.uint64(11)
    pow11 = np.array([11 ** k for k in range(19)], np.uint64)
    key = inner * pow11[18 - ndig]
    return key


def _quantile_sorted(s: np.ndarray, p: float) -> float:
    # distribution.cpp:33-44
    n = len(s)
    if p <= 0:
        return float(s[0])
    if p >= 1:
        return float(s[-1])
    pos = p * (n - 1)
    lo = int(pos)
    frac = pos - lo
    if lo + 1 >= n:
        return float(s[-1])
    return float(s[lo] + frac * (s[lo + 1] - s[lo]))


def snapshot(n_pools: int = 8, per_pool: int = 2_000_000, seed: int = 1, burst: float = 10.0,
             prefill_rate: float = 8000.0, decode_rate: float = 50.0,
             cold_start_agent: str = "Humanities", msg_base: int = 0, uid_base: int = 1) -> QueueSnapshot:
    rng = np.random.default_rng(seed)
    lens = np.array([len(t[0]) for t in TEMPLATES])
    probs = np.array([t[1] for t in TEMPLATES])
    probs = probs / probs.sum()
    tmpl_agents = [np.array([A[a] for a in t[0]], np.int32) for t in TEMPLATES]
    mean_len = float((lens * probs).sum())
    cols = {k: [] for k in ["agent", "prompt", "target", "app", "wf"]}
    wf_base = msg_base
    for p in range(n_pools):
        n_wf = int(per_pool / mean_len * 1.05) + 16
        t_id = rng.choice(len(TEMPLATES), size=n_wf, p=probs)
        L = lens[t_id]
        ends = np.cumsum(L)
        keep = np.searchsorted(ends, per_pool, side="left") + 1
        t_id, L = t_id[:keep], L[:keep]
        total = int(L.sum())
        starts = np.concatenate([[0], np.cumsum(L)[:-1]])
        pos = np.arange(total) - np.repeat(starts, L)
        wf = np.repeat(np.arange(keep), L)
        ag = np.empty(total, np.int32)
        for t in range(len(TEMPLATES)):
            m = t_id[wf] == t
            ag[m] = tmpl_agents[t][pos[m]]
        app = np.sort(rng.uniform(0.0, burst, keep))
        cols["agent"].append(ag[:per_pool] + 10 * p)
        cols["app"].append(app[wf[:per_pool]])
        cols["wf"].append(wf[:per_pool] + wf_base)
        wf_base += keep
    agent = np.concatenate(cols["agent"]).astype(np.int32)
    local = agent % 10
    lo = np.array([a[1] for a in AGENTS])[local]
    hi = np.array([a[2] for a in AGENTS])[local]
    prompt = rng.integers(lo, hi + 1).astype(np.int64)
    mu = np.log(np.array([a[3] for a in AGENTS]))[local]
    sig = np.array([a[4] for a in AGENTS])[local]
    cap = np.array([a[5] for a in AGENTS])[local]
    target = np.clip(np.rint(np.exp(rng.normal(mu, sig))), 1, cap).astype(np.int64)
    pure = prompt / prefill_rate + target / decode_rate
    wf = np.concatenate(cols["wf"])
    app_start = np.concatenate(cols["app"])
    # queue_enter = app_start + exclusive prefix of pure_exec within the chain
    cs = np.cumsum(pure)
    first = np.ones(len(wf), bool)
    first[1:] = wf[1:] != wf[:-1]
    base = np.maximum.accumulate(np.where(first, np.arange(len(wf)), 0))
    excl = cs - pure - np.where(base > 0, cs[np.maximum(base - 1, 0)], 0.0)
    excl[first] = 0.0
    queue_enter = app_start + excl
    msg_counter = wf.astype(np.uint64)
    # per-agent tables
    n_agents = 10 * n_pools
    agent_pool = (np.arange(n_agents) // 10).astype(np.int32)
    names = [f"{AGENTS[a % 10][0]}_p{a // 10}" for a in range(n_agents)]
    # remaining latency per call = suffix sum of pure_exec within the chain
    last = np.ones(len(wf), bool)
    last[:-1] = wf[:-1] != wf[1:]
    rev_cs = np.cumsum(pure[::-1])[::-1]
    nxt = np.minimum.accumulate(np.where(last, np.arange(len(wf)), len(wf))[::-1])[::-1]
    remaining = rev_cs - np.where(nxt + 1 < len(wf), rev_cs[np.minimum(nxt + 1, len(wf) - 1)], 0.0)
    mean_rem = np.bincount(agent, weights=remaining, minlength=n_agents) / np.maximum(
        np.bincount(agent, minlength=n_agents), 1)
    known = np.array([AGENTS[a % 10][0] != cold_start_agent for a in range(n_agents)], np.uint8)
    pk = mean_rem.copy()
    if known.sum() > 0:
        med = _quantile_sorted(np.sort(pk[known == 1]), 0.5)  # priority.cpp:121-130
        pk[known == 0] = med
    depth = np.array([{"Router": 2, "Researcher": 2, "ProductManager": 5, "Architect": 4,
                       "ProjectManager": 3, "Engineer": 2}.get(AGENTS[a % 10][0], 1)
                      for a in range(n_agents)], np.int32)
    samp = rng.integers(0, len(agent), min(len(agent), 1 << 20))
    sa, sp = agent[samp], pure[samp]
    order = np.lexsort((sp, sa))
    sa, sp = sa[order], sp[order]
    bounds = np.searchsorted(sa, np.arange(n_agents + 1))
    T = np.array([np.median(sp[bounds[a]:bounds[a + 1]]) if bounds[a + 1] > bounds[a] else 1.0
                  for a in range(n_agents)])
    uid = (uid_base + np.arange(len(agent))).astype(np.uint64)
    return QueueSnapshot(agent, prompt, app_start, queue_enter, msg_counter, msg_key_decimal(msg_counter),
                         uid, pure, agent_pool, names, pk, known, depth, T, n_pools)


def instances(n_pools: int = 8, per_pool: int = 32, capacity: float = 20000.0, max_batch: int = 64,
              decode_rate: float = 50.0, prefill_rate: float = 8000.0):
    """InstanceProfile list, pool-grouped (engine.hpp:25-31)."""
    from .sched import InstanceProfile
    out = []
    for p in range(n_pools):
        for j in range(per_pool):
            out.append(InstanceProfile(id=p * per_pool + j, pool=p, capacity_tokens=capacity,
                                       decode_rate=decode_rate, prefill_rate=prefill_rate,
                                       max_batch=max_batch))
    return out


def preload(insts, seed: int = 7, now: float = 10.0):
    """Pre-loaded engine state: per instance a running count,
    live KV and the ledger commits of its running requests. Returns
    (live_kv, running, commits[(instance_id, uid, prompt, decode_rate, t0, T)])."""
    rng = np.random.default_rng(seed)
    live, running, commits = [], [], []
    uid = 10 ** 12
    for inst in insts:
        r = int(rng.integers(inst.max_batch // 2, inst.max_batch - 4))
        kv = 0.0
        for _ in range(r):
            P = int(rng.integers(60, 240))
            t0 = float(now - rng.uniform(0.0, 6.0))
            T = float(rng.uniform(1.0, 14.0))
            commits.append((inst.id, uid, P, inst.decode_rate, t0, T))
            uid += 1
            kv += P + inst.decode_rate * (now - t0)
        live.append(min(kv, 0.6 * inst.capacity_tokens))
        running.append(r)
    return np.array(live), np.array(running, np.int32), commits
