"""§8(f)4 throughput: trace CSV parse + workflow reconstruction on the device
(kx_trace_parse + kx_workflow_reconstruct through the Python host API, host
bytes in, graph out: H2D of the file inside the timing) against the
unmodified reference read_trace + WorkflowAnalyzer::ingest_trace +
WorkflowGraph::report (oracle/_ref/libkxref.so, one host thread) on the same
bytes; the reports must be identical. Prints one JSON line.

    python scripts/trace_probe.py [--workflows 300000] [--repeats 5]
"""
import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import bench  # noqa: E402
import ref_sim  # noqa: E402  (test infrastructure: the reference, as the checker / CPU baseline)
from test_gpu_trace import device_report, synthetic  # noqa: E402
from paper_2508_06948_b200.workflow import Trace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workflows", type=int, default=300_000)
ap.add_argument("--repeats", type=int, default=5)
a = ap.parse_args()
data = synthetic(7, n_wf=a.workflows, blank=False)
lines = data.count(b"\n") - 1


def device_once():
    t0 = time.perf_counter()
    t = Trace(data)
    t1 = time.perf_counter()
    g = t.analyze()
    t2 = time.perf_counter()
    rep = device_report(t)  # report() + depth and downstream paths of every node, as the reference bridge
    t3 = time.perf_counter()
    return rep, (t1 - t0, t2 - t1, t3 - t2)


device_once()  # warm-up (module load, allocations)
clk = bench.Clocks(0)
clk.mark(True)
times, parts = [], []
for _ in range(a.repeats):
    t0 = time.perf_counter()
    rep_dev, pp = device_once()
    times.append(time.perf_counter() - t0)
    parts.append(pp)
clk.mark(False)
clocks = clk.stop()
dev_s = min(times)
best = parts[times.index(dev_s)]

L = ref_sim.lib()
f = L.kxref_trace_report
f.restype = C.c_int64
f.argtypes = [C.c_char_p, C.c_int64, C.c_int, C.c_void_p, C.c_int64]
cap = 1 << 26
buf = C.create_string_buffer(cap)
ref_times = []
for _ in range(2):
    t0 = time.perf_counter()
    n = f(data, len(data), 3, C.cast(buf, C.c_void_p), cap)
    ref_times.append(time.perf_counter() - t0)
ref_s = min(ref_times)
rep_ref = buf.raw[:n].decode()
same = rep_ref == rep_dev
print(json.dumps({
    "metric": "trace lines parsed + workflows reconstructed per second (read_trace + WorkflowAnalyzer)",
    "lines": lines, "bytes": len(data), "workflows": a.workflows,
    "device": {"seconds": dev_s, "lines_per_s": lines / dev_s, "GB_per_s": len(data) / dev_s / 1e9,
               "parse_s": best[0], "reconstruct_s": best[1], "host_report_s": best[2],
               "path": "host bytes -> kx_trace_parse (H2D + newline scan + per-line parse/validate + interning) "
                       "-> kx_workflow_reconstruct -> graph fetch"},
    "reference": {"seconds": ref_s, "lines_per_s": lines / ref_s, "threads": 1,
                  "path": "read_trace + WorkflowAnalyzer::ingest_trace + report (+ depths/paths), oracle/_ref"},
    "speedup": ref_s / dev_s, "report_identical": same, "clocks": clocks}))
