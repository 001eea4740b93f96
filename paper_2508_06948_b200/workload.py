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


def preload(insts, seed: int = 7, now: float = 10.0, light: bool = False):
    """Pre-loaded engine state: per instance a running count,
    live KV and the ledger commits of its running requests. Returns
    (live_kv, running, commits[(instance_id, uid, prompt, decode_rate, t0, T)]).
    `light` (small max_batch, C1-C3): 1 .. max_batch / 2 running requests."""
    rng = np.random.default_rng(seed)
    live, running, commits = [], [], []
    uid = 10 ** 12
    for inst in insts:
        if light:
            r = int(rng.integers(1, max(2, inst.max_batch // 2 + 1)))
        else:
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


# ---- general workloads: WorkloadConfig -> realize() (kx_realize) ------------
# The reference's workload model (workload.hpp:18-83): agents with a
# probabilistic choice, a parallel group or a bounded feedback edge, apps
# with an entry agent and a weight, Poisson or trace arrivals. realize() runs
# in the product library (kx_workload.cpp), restated from workload.cpp:227-372
# and checked bit for bit against the reference's realize()
# (tests/test_workload_general.py).

@dataclass
class LengthSpec:
    """LengthSpec (workload.hpp:18-33)."""
    kind: int = 0          # 0 fixed, 1 uniform int, 2 lognormal int
    a: float = 1.0
    b: float = 0.0
    min_tokens: int = 1
    max_tokens: int = 1 << 20

    @staticmethod
    def fixed(v: int) -> "LengthSpec":
        return LengthSpec(0, float(v), 0.0, v, v)

    @staticmethod
    def uniform(lo: int, hi: int) -> "LengthSpec":
        return LengthSpec(1, float(lo), float(hi), lo, hi)

    @staticmethod
    def lognormal(median: float, sigma: float, cap: int) -> "LengthSpec":
        import math
        return LengthSpec(2, math.log(median), sigma, 1, cap)


@dataclass
class AgentSpec:
    """AgentSpec (workload.hpp:39-52)."""
    name: str
    prompt_len: LengthSpec
    output_len: LengthSpec
    choice: list = None      # [(agent name, probability)]
    parallel: list = None    # [agent name]
    feedback: tuple = None   # (target name, probability, max_iterations)


@dataclass
class AppSpec:
    """AppSpec (workload.hpp:55-60)."""
    name: str
    agents: list
    entry: str
    weight: float = 1.0


@dataclass
class WorkloadConfig:
    """WorkloadConfig (workload.hpp:69-83). `trace` holds raw arrival
    timestamps (ArrivalSpec::TraceFile, already parsed) or None for Poisson."""
    apps: list
    rate: float = 1.0
    duration: float = 60.0
    seed: int = 1
    trace: np.ndarray = None
    trace_scale: float = 1.0
    entry_selection: str = "weighted"

    def agent_names(self) -> list:
        return [a.name for app in self.apps for a in app.agents]


def qa_app() -> AppSpec:
    """qa_app (workload.cpp:462-481)."""
    return AppSpec("qa", [
        AgentSpec("Router", LengthSpec.uniform(40, 80), LengthSpec.lognormal(10.0, 0.25, 40),
                  choice=[("Math", 0.5), ("Humanities", 0.5)]),
        AgentSpec("Math", LengthSpec.uniform(60, 120), LengthSpec.lognormal(70.0, 0.35, 400)),
        AgentSpec("Humanities", LengthSpec.uniform(60, 120), LengthSpec.lognormal(240.0, 0.35, 900))],
        "Router")


def rg_app() -> AppSpec:
    """rg_app (workload.cpp:483-498)."""
    return AppSpec("rg", [
        AgentSpec("Researcher", LengthSpec.uniform(80, 160), LengthSpec.lognormal(150.0, 0.35, 700),
                  choice=[("Writer", 1.0)]),
        AgentSpec("Writer", LengthSpec.uniform(120, 240), LengthSpec.lognormal(380.0, 0.30, 1100))],
        "Researcher")


def cg_app() -> AppSpec:
    """cg_app (workload.cpp:500-521)."""
    def chain(name, median, sigma, cap, nxt, prompt=(80, 160)):
        return AgentSpec(name, LengthSpec.uniform(*prompt), LengthSpec.lognormal(median, sigma, cap),
                         choice=[(nxt, 1.0)] if nxt else None)
    qa = chain("QAEngineer", 40.0, 0.30, 160, None)
    qa.feedback = ("Engineer", 0.3, 3)
    return AppSpec("cg", [chain("ProductManager", 70.0, 0.35, 300, "Architect"),
                          chain("Architect", 110.0, 0.35, 450, "ProjectManager"),
                          chain("ProjectManager", 50.0, 0.30, 200, "Engineer"),
                          chain("Engineer", 300.0, 0.40, 1100, "QAEngineer", prompt=(100, 200)), qa],
                   "ProductManager")


def generated_apps(n_apps: int = 100, seed: int = 2508) -> list:
    """C3: n_apps generated applications of 5 agents each, named
    a<i>_<role>, covering the reference's three structural features
    (workload.hpp:36-38): app i % 3 == 0 routes by a probabilistic choice,
    == 1 fans out to a parallel group, == 2 is a chain whose critic loops
    back through a feedback edge. Lengths are drawn per app from the ranges
    of the built-in templates (workload.cpp:462-531)."""
    rng = np.random.default_rng(seed)
    apps = []
    for i in range(n_apps):
        nm = lambda r: f"a{i}_{r}"  # noqa: E731
        def ln():
            lo = int(rng.integers(40, 121))
            return LengthSpec.uniform(lo, lo + int(rng.integers(40, 121)))
        def out():
            med = float(rng.choice([10.0, 40.0, 70.0, 110.0, 150.0, 240.0, 300.0, 380.0]))
            return LengthSpec.lognormal(med, float(rng.choice([0.25, 0.30, 0.35, 0.40])), int(med * 4))
        kind = i % 3
        plan = AgentSpec(nm("planner"), ln(), out())
        wa = AgentSpec(nm("worker_a"), ln(), out())
        wb = AgentSpec(nm("worker_b"), ln(), out())
        crit = AgentSpec(nm("critic"), ln(), out())
        wr = AgentSpec(nm("writer"), ln(), out())
        if kind == 0:
            p = float(np.round(rng.uniform(0.2, 0.8), 3))
            plan.choice = [(wa.name, p), (wb.name, 1.0 - p)]
            wa.choice = [(crit.name, 1.0)]
            wb.choice = [(wr.name, 1.0)]
            crit.choice = [(wr.name, 1.0)]
        elif kind == 1:
            plan.parallel = [wa.name, wb.name]
            wa.choice = [(wr.name, 1.0)]
            wb.choice = [(crit.name, 1.0)]
            crit.choice = [(wr.name, 1.0)]
        else:
            plan.choice = [(wa.name, 1.0)]
            wa.choice = [(wb.name, 1.0)]
            wb.choice = [(crit.name, 1.0)]
            crit.choice = [(wr.name, 1.0)]
            crit.feedback = (wa.name, float(np.round(rng.uniform(0.1, 0.4), 3)), int(rng.integers(1, 4)))
        apps.append(AppSpec(f"app{i}", [plan, wa, wb, crit, wr], plan.name,
                            float(np.round(rng.uniform(0.5, 2.0), 3))))
    return apps


def workload_abi(cfg: WorkloadConfig):
    """kx_workload_config for `cfg` (plus the buffers it points to)."""
    from . import _abi
    import ctypes as C
    names = cfg.agent_names()
    idx = {n: i for i, n in enumerate(names)}
    if len(idx) != len(names):
        raise ValueError("duplicate agent name")  # WorkloadConfig::validate (workload.cpp:113)
    keep = []

    def arr(x, dt):
        a = np.ascontiguousarray(np.array(x, dt))
        keep.append(a)
        return a.ctypes.data if len(a) else None

    agents = (_abi.kx_agent_spec * len(names))()
    for app in cfg.apps:
        for a in app.agents:
            s = agents[idx[a.name]]
            for f, l in (("prompt_len", a.prompt_len), ("output_len", a.output_len)):
                setattr(s, f, _abi.kx_length_spec(l.kind, 0, l.a, l.b, l.min_tokens, l.max_tokens))
            ch = a.choice or []
            s.n_choice = len(ch)
            s.choice_to = arr([idx[t] for t, _ in ch], np.int32)
            s.choice_p = arr([p for _, p in ch], np.float64)
            par = a.parallel or []
            s.n_parallel = len(par)
            s.parallel_to = arr([idx[t] for t in par], np.int32)
            if a.feedback:
                s.feedback_target = idx[a.feedback[0]]
                s.feedback_probability = a.feedback[1]
                s.feedback_max_iterations = a.feedback[2]
            else:
                s.feedback_target = -1
    apps = (_abi.kx_app_spec * len(cfg.apps))()
    for k, app in enumerate(cfg.apps):
        apps[k].entry = idx[app.entry]
        apps[k].n_members = len(app.agents)
        apps[k].members = arr([idx[a.name] for a in app.agents], np.int32)
        apps[k].weight = app.weight
    c = _abi.kx_workload_config()
    c.n_agents, c.n_apps = len(names), len(cfg.apps)
    c.agents, c.apps = agents, apps
    c.arrival_kind = 1 if cfg.trace is not None else 0
    c.entry_selection = 1 if cfg.entry_selection == "cycle" else 0
    c.rate = cfg.rate
    if cfg.trace is not None:
        c.n_trace = len(cfg.trace)
        c.trace = arr(cfg.trace, np.float64)
    c.trace_scale = cfg.trace_scale
    c.duration = cfg.duration
    keep += [agents, apps]
    return c, keep, names


@dataclass
class Realization:
    """WorkloadRealization (workload.hpp:115-121), flattened: workflow w owns
    calls [wf_offsets[w], wf_offsets[w + 1]) in node order; msg id "m-<w>"."""
    arrival: np.ndarray
    app: np.ndarray
    wf_offsets: np.ndarray
    agent: np.ndarray
    parent: np.ndarray
    prompt: np.ndarray
    target: np.ndarray
    pure_exec: np.ndarray
    remaining: np.ndarray
    uid: np.ndarray
    agent_names: list

    @property
    def n_calls(self):
        return len(self.agent)


def realize(cfg: WorkloadConfig, prefill_rate: float = 8000.0, decode_rate: float = 50.0) -> Realization:
    """realize() (workload.cpp:319-372) in the product library."""
    from . import _abi
    import ctypes as C
    lib = _abi.load()
    c, keep, names = workload_abi(cfg)
    h = C.c_void_p()
    _abi.check(lib.kx_realize(C.byref(c), cfg.seed, prefill_rate, decode_rate, C.byref(h)))
    try:
        nw, nc = C.c_int64(), C.c_int64()
        _abi.check(lib.kx_realization_sizes(h, C.byref(nw), C.byref(nc)))
        W, N = nw.value, nc.value
        out = dict(arrival=np.zeros(W), app=np.zeros(W, np.int32), wf_offsets=np.zeros(W + 1, np.int64),
                   agent=np.zeros(N, np.int32), parent=np.zeros(N, np.int32), prompt=np.zeros(N, np.int64),
                   target=np.zeros(N, np.int64), pure_exec=np.zeros(N), remaining=np.zeros(N),
                   uid=np.zeros(N, np.uint64))
        _abi.check(lib.kx_realization_copy(h, *[v.ctypes.data for v in out.values()]))
    finally:
        lib.kx_realization_free(h)
    return Realization(agent_names=names, **out)


def snapshot_from_realization(real: Realization, n: int, cold_start: int = 1, msg_base: int = 0,
                              uid_offset: int = 0) -> QueueSnapshot:
    """Queue snapshot of a realization: the first n calls in uid
    order all queued, app_start = the workflow's arrival, queue_enter =
    app_start + the pure_exec of its ancestors (the time it would have been
    released under zero queueing). Single pool. Priority key per agent =
    mean remaining_exec of its calls, with the `cold_start` least-called
    agents left out of the table (cold start: the median of the known keys,
    priority.cpp:121-130); expected T = median pure_exec per agent."""
    if n > real.n_calls:
        raise ValueError(f"realization has {real.n_calls} calls, {n} requested")
    W = int(np.searchsorted(real.wf_offsets, n, side="left"))
    wf = np.repeat(np.arange(len(real.arrival)), np.diff(real.wf_offsets))[:n]
    start = real.wf_offsets[wf]
    # ancestors' pure_exec: parents come first, so one forward sweep
    pure = real.pure_exec[:n]
    par = real.parent[:n]
    above = np.zeros(n)
    has = par >= 0
    gp = np.where(has, start + par, 0)
    for i in np.flatnonzero(has):  # parents-first: above[parent] is final
        j = gp[i]
        above[i] = above[j] + pure[j]
    app_start = real.arrival[wf]
    queue_enter = app_start + above
    agent = real.agent[:n].astype(np.int32)
    n_agents = len(real.agent_names)
    counts = np.bincount(agent, minlength=n_agents)
    mean_rem = np.bincount(agent, weights=real.remaining[:n], minlength=n_agents) / np.maximum(counts, 1)
    known = np.ones(n_agents, np.uint8)
    if cold_start:
        present = np.flatnonzero(counts > 0)
        leave = present[np.argsort(counts[present], kind="stable")[:cold_start]]
        known[leave] = 0
    pk = mean_rem.copy()
    if known.sum():
        pk[known == 0] = _quantile_sorted(np.sort(pk[known == 1]), 0.5)
    order = np.lexsort((pure, agent))
    bounds = np.searchsorted(agent[order], np.arange(n_agents + 1))
    T = np.array([np.median(pure[order[bounds[a]:bounds[a + 1]]]) if bounds[a + 1] > bounds[a] else 1.0
                  for a in range(n_agents)])
    msg_counter = (wf + msg_base).astype(np.uint64)
    del W
    return QueueSnapshot(agent, real.prompt[:n].copy(), app_start, queue_enter, msg_counter,
                         msg_key_decimal(msg_counter), real.uid[:n] + np.uint64(uid_offset), pure.copy(),
                         np.zeros(n_agents, np.int32), list(real.agent_names), pk, known,
                         np.ones(n_agents, np.int32), T, 1)


# ---- the benchmark configurations (BASELINE.json configs C1-C4) -------------
CONFIGS = {
    "C1": dict(workload="C1: QA app (Router/Humanities/Math agents), 1 shared LLM, 4 instances, "
                        "1K queued requests", apps="qa", n=1_000, pools=1, per_pool=4, cap=3000.0, mb=8),
    "C2": dict(workload="C2: 3 mixed multi-agent apps (QA+RG+CG) sharing 1 LLM, 16 instances, 64K queued "
                        "requests, excessive-load burst", apps="colocated", n=65_536, pools=1, per_pool=16,
               cap=3000.0, mb=8),
    "C3": dict(workload="C3: 100 generated workflows with dynamic call graphs (choice/parallel/feedback, "
                        "500 agents), 1M queued requests, 64 instances", apps="generated", n=1_000_000,
               pools=1, per_pool=64, cap=3000.0, mb=8),
    "C4": dict(workload="C4: 16M queued requests, 8 LLM pools x 32 instances, Kairos priority + time-slot "
                        "dispatch, pre-loaded ledgers", apps="c4", n=16_000_000, pools=8, per_pool=32,
               cap=20000.0, mb=64),
}
BURST = 10.0  # seconds over which a snapshot's workflows arrive


@dataclass
class BenchWorkload:
    name: str
    desc: str
    snap: QueueSnapshot
    arrivals: QueueSnapshot  # later calls of the same workload (serving-loop enqueues)
    insts: list
    live: np.ndarray
    running: np.ndarray
    commits: list
    now: float


def _realize_calls(apps, n: int, seed: int) -> Realization:
    """realize() of `apps` with the Poisson rate chosen so that at least n
    calls arrive within BURST seconds."""
    pilot = realize(WorkloadConfig(apps, rate=200.0, duration=BURST, seed=seed))
    per_wf = max(1.0, pilot.n_calls / max(1, len(pilot.arrival)))
    rate = n / per_wf / BURST * 1.05
    for _ in range(8):
        real = realize(WorkloadConfig(apps, rate=rate, duration=BURST, seed=seed))
        if real.n_calls >= n:
            return real
        rate *= 1.1 * n / max(1, real.n_calls)
    raise RuntimeError("could not realize enough calls")


def build_workload(name: str, rank: int = 0, arrivals: int = 65_536) -> BenchWorkload:
    """The queue snapshot, instances and pre-tick engine state of config
    `name` (rank r of a weak-scaling run draws its own seed)."""
    c = CONFIGS[name]
    now = BURST
    if c["apps"] == "c4":
        snap = snapshot(n_pools=c["pools"], per_pool=c["n"] // c["pools"], seed=1 + rank,
                        msg_base=rank * 10_000_000, uid_base=1 + rank * 10 ** 9)
        arr = snapshot(n_pools=c["pools"], per_pool=max(1, arrivals // c["pools"]), seed=101 + rank,
                       msg_base=rank * 10_000_000 + 8_000_000, uid_base=1 + rank * 10 ** 9 + 100_000_000)
    else:
        apps = {"qa": lambda: [qa_app()], "colocated": lambda: [qa_app(), rg_app(), cg_app()],
                "generated": lambda: generated_apps(100)}[c["apps"]]()
        real = _realize_calls(apps, c["n"] + arrivals, seed=1 + rank)
        full = snapshot_from_realization(real, c["n"] + arrivals, uid_offset=rank * 10 ** 9,
                                         msg_base=rank * 10_000_000)
        n = c["n"]
        cut = lambda a, lo, hi: a[lo:hi]  # noqa: E731
        fields = ("agent", "prompt", "app_start", "queue_enter", "msg_counter", "msg_key", "uid", "pure_exec")
        mk = lambda lo, hi: QueueSnapshot(*[cut(getattr(full, f), lo, hi) for f in fields],  # noqa: E731
                                          full.agent_pool, full.agent_names, full.priority_key, full.pk_known,
                                          full.topo_depth, full.expected_T, full.n_pools)
        snap, arr = mk(0, n), mk(n, n + arrivals)
    insts = instances(c["pools"], c["per_pool"], capacity=c["cap"], max_batch=c["mb"])
    live, running, commits = preload(insts, seed=7 + rank, now=now, light=c["apps"] != "c4")
    return BenchWorkload(name, c["workload"], snap, arr, insts, live, running, commits, now)
