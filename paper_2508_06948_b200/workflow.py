"""Trace CSV I/O and workflow reconstruction.

`Trace` parses a whole trace file on the device (kx_trace_parse: read_trace
+ parse_trace_line + validate, trace.cpp:14-127) and writes it back
(kx_trace_format: write_trace, trace.cpp:29-48). `Trace.analyze()` folds
every instance into the call graph on the device (kx_workflow_reconstruct:
WorkflowAnalyzer::ingest_trace, workflow.cpp:319-343, with
WorkflowGraph::ingest / ingest_instance / classify_fanout,
workflow.cpp:19-111) and returns a `WorkflowGraph` with the reference's
query API (workflow.hpp:55-111). The queries over the reduced graph
(feedback edges, downstream paths, topological depth, the report) are
small walks over a few hundred nodes; they run here, restated from
workflow.cpp:154-299.
"""
from __future__ import annotations

import ctypes as C
from collections import defaultdict
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import check


@dataclass
class FanoutPattern:
    """FanoutPattern (workflow.hpp:44-52)."""
    node: str
    downstreams: list = field(default_factory=list)  # sorted (std::set)
    kind: str = "single"
    parallel_obs: int = 0
    sequential_obs: int = 0
    single_obs: int = 0


class Trace:
    """A trace file parsed on the device. Raises KxError (code 1, the
    reference's std::invalid_argument message) on the first bad line."""

    def __init__(self, data: bytes | str, device: int = 0):
        lib = _abi.load()
        if isinstance(data, str):
            data = data.encode()
        self._lib = lib
        self._data = data
        h = C.c_void_p()
        check(lib.kx_trace_parse(data, len(data), device, C.byref(h)))
        self._h = h
        n, a, m, nb = C.c_int64(), C.c_int32(), C.c_int64(), C.c_int64()
        check(lib.kx_trace_sizes(h, C.byref(n), C.byref(a), C.byref(m), C.byref(nb)))
        self.n, self.n_msgs = n.value, m.value
        names = C.create_string_buffer(max(1, nb.value))
        offs = np.zeros(a.value + 1, np.int64)
        check(lib.kx_trace_agents(h, names, offs.ctypes.data))
        raw = names.raw
        self.agents = [raw[offs[i]:offs[i + 1]].decode() for i in range(a.value)]

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.kx_trace_free(self._h)
            self._h = None

    def columns(self) -> dict:
        """RequestRecord fields (types.hpp) in file order."""
        n = self.n
        out = dict(msg=np.zeros(n, np.int64), agent=np.zeros(n, np.int32), upstream=np.zeros(n, np.int32),
                   exec_start=np.zeros(n), exec_end=np.zeros(n), prompt_tokens=np.zeros(n, np.int64),
                   output_tokens=np.zeros(n, np.int64), app_start=np.zeros(n))
        check(self._lib.kx_trace_columns(self._h, *[v.ctypes.data for v in out.values()]))
        return out

    def msg_id(self, i: int) -> str:
        n = C.c_int64()
        check(self._lib.kx_trace_msg_id(self._h, i, None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(1, n.value))
        check(self._lib.kx_trace_msg_id(self._h, i, buf, n.value, C.byref(n)))
        return buf.raw[:n.value].decode()

    def msg_ids(self, msgs) -> list:
        """msg_id strings of many msg indices (one device gather)."""
        msgs = np.ascontiguousarray(msgs, dtype=np.int64)
        off = np.zeros(len(msgs), np.int64)
        ln = np.zeros(len(msgs), np.int32)
        check(self._lib.kx_trace_msg_spans(self._h, len(msgs), msgs.ctypes.data, off.ctypes.data, ln.ctypes.data))
        d = self._data
        return [d[o:o + n].decode() for o, n in zip(off.tolist(), ln.tolist())]

    def format(self) -> bytes:
        """write_trace (trace.cpp:44-48) of the records, formatted on the device."""
        n = C.c_int64()
        check(self._lib.kx_trace_format(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(self._lib.kx_trace_format(self._h, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    def analyze(self) -> "WorkflowGraph":
        """WorkflowAnalyzer::ingest_trace (workflow.cpp:336-342) + snapshot()."""
        sz = _abi.kx_workflow_sizes()
        check(self._lib.kx_workflow_reconstruct(self._h, C.byref(sz)))
        A = len(self.agents)
        ef, et = np.zeros(sz.n_edges, np.int32), np.zeros(sz.n_edges, np.int32)
        ec = np.zeros(sz.n_edges, np.uint64)
        ent = np.zeros(A, np.uint8)
        par, seq, sgl = (np.zeros(A, np.uint64) for _ in range(3))
        dm = np.zeros(sz.n_diagnostics, np.int64)
        de, do = np.zeros(sz.n_diagnostics, np.int32), np.zeros(sz.n_diagnostics, np.int32)
        check(self._lib.kx_workflow_fetch(self._h, *[v.ctypes.data for v in
                                                     (ef, et, ec, ent, par, seq, sgl, dm, de, do)]))
        g = WorkflowGraph()
        g._nodes = list(self.agents)
        g._edges = {(self.agents[f], self.agents[t]): int(c) for f, t, c in zip(ef, et, ec)}
        g._entries = [self.agents[a] for a in range(A) if ent[a]]
        for a in range(A):
            p, s, z = int(par[a]), int(seq[a]), int(sgl[a])
            if p + s + z == 0:
                continue
            kind = "single" if p + s == 0 else ("parallel" if p >= s else "sequential")
            down = sorted(t for (f, t) in g._edges if f == self.agents[a])
            g._fanouts[self.agents[a]] = FanoutPattern(self.agents[a], down, kind, p, s, z)
        ids = self.msg_ids(dm)
        g._diagnostics = [f"msg {ids[i]}: conflicting entries '{self.agents[e]}' and '{self.agents[o]}'"
                          for i, (e, o) in enumerate(zip(de, do))]
        g._instances = int(sz.instances)
        return g


class WorkflowGraph:
    """The reconstructed call graph (workflow.hpp:55-111)."""

    def __init__(self):
        self._nodes: list[str] = []
        self._edges: dict[tuple[str, str], int] = {}
        self._entries: list[str] = []
        self._fanouts: dict[str, FanoutPattern] = {}
        self._diagnostics: list[str] = []
        self._instances = 0

    def nodes(self):
        return list(self._nodes)

    def edges(self):
        return [(f, t, c) for (f, t), c in sorted(self._edges.items())]

    def edge_observations(self, frm, to):
        return self._edges.get((frm, to), 0)

    def has_edge(self, frm, to):
        return (frm, to) in self._edges

    def entries(self):
        return list(self._entries)

    def entry(self):
        if len(self._entries) != 1:
            raise RuntimeError(f"graph has {len(self._entries)} entries, expected exactly one")
        return self._entries[0]

    def fanouts(self):
        return dict(sorted(self._fanouts.items()))

    def diagnostics(self):
        return list(self._diagnostics)

    def instances_ingested(self):
        return self._instances

    def downstream_agents(self, frm):
        """workflow.cpp:146-152 (edges_ order)."""
        return [t for (f, t) in sorted(self._edges) if f == frm]

    def feedback_edges(self):
        """Iterative DFS from the entries, then every node (workflow.cpp:154-191)."""
        feedback, done, on_stack = set(), set(), set()

        def dfs(root):
            if root in done:
                return
            stack = [[root, self.downstream_agents(root), 0]]
            on_stack.add(root)
            while stack:
                f = stack[-1]
                if f[2] < len(f[1]):
                    to = f[1][f[2]]
                    f[2] += 1
                    if to in on_stack:
                        feedback.add((f[0], to))
                    elif to not in done:
                        on_stack.add(to)
                        stack.append([to, self.downstream_agents(to), 0])
                else:
                    done.add(f[0])
                    on_stack.discard(f[0])
                    stack.pop()

        for e in sorted(self._entries):
            dfs(e)
        for n in sorted(self._nodes):
            dfs(n)
        return sorted(feedback)

    def _reaches(self, frm, to):
        seen, stack = set(), [frm]
        while stack:
            n = stack.pop()
            if n in seen:
                continue
            seen.add(n)
            for nxt in self.downstream_agents(n):
                if nxt == to:
                    return True
                stack.append(nxt)
        return False

    def downstream_paths(self, agent, max_loop=3):
        """workflow.cpp:214-260."""
        if agent not in self._nodes:
            raise ValueError("unknown agent: " + agent)
        feedback = set(self.feedback_edges())

        def budget(frm, to):
            if (frm, to) in feedback:
                return max_loop
            on_cycle = frm == to or self._reaches(to, frm)
            return max_loop + 1 if on_cycle else 1

        paths, current, used = [], [agent], defaultdict(int)

        def walk(node):
            extended = False
            for to in self.downstream_agents(node):
                edge = (node, to)
                if used[edge] >= budget(node, to):
                    continue
                used[edge] += 1
                current.append(to)
                walk(to)
                current.pop()
                used[edge] -= 1
                if edge not in feedback:
                    extended = True
            if not extended:
                paths.append(list(current))

        walk(agent)
        out = []
        for p in sorted(paths):
            if not out or out[-1] != p:
                out.append(p)
        return out

    def topo_depth(self, agent):
        """workflow.cpp:262-269."""
        return max([1] + [len(p) for p in self.downstream_paths(agent, 1)])

    def report(self):
        """WorkflowGraph::report (workflow.cpp:271-313), byte for byte."""
        out = [f"workflow graph: {len(self._nodes)} nodes, {len(self._edges)} edges, "
               f"{self._instances} instances\n", "entries:"]
        out += [f" {e}" for e in sorted(self._entries)]
        out.append("\nedges:\n")
        out += [f"  {f} -> {t}  (x{c})\n" for f, t, c in self.edges()]
        fb = self.feedback_edges()
        if fb:
            out.append("feedback edges:\n")
            out += [f"  {f} -> {t}\n" for f, t in fb]
        out.append("fanouts:\n")
        for node, pat in sorted(self._fanouts.items()):
            out.append(f"  {node}: {pat.kind} {{{', '.join(pat.downstreams)}}}  [par={pat.parallel_obs} "
                       f"seq={pat.sequential_obs} single={pat.single_obs}]\n")
        if self._diagnostics:
            out.append("diagnostics:\n")
            out += [f"  {d}\n" for d in self._diagnostics]
        return "".join(out)
