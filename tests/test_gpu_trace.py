"""§8(f)4 on the B200: trace CSV parse/format (trace.cpp:14-127) and workflow
reconstruction (workflow.cpp:19-343) against the UNMODIFIED reference
(read_trace, write_trace, WorkflowAnalyzer, oracle/_ref/libkxref.so) on the
same bytes: every parsed field bit-exact, the written trace byte-identical,
WorkflowGraph::report() plus topo_depth and downstream_paths of every node
identical, and the first bad line's error message identical."""
import ctypes as C

import numpy as np
import pytest

import ref_sim
from helpers import bits
from paper_2508_06948_b200 import KxError
from paper_2508_06948_b200 import engine as E
from paper_2508_06948_b200.workflow import Trace

pytestmark = pytest.mark.gpu
HEADER = "msg_id,agent,upstream,exec_start,exec_end,prompt_tokens,output_tokens,app_start"


def ref_call(name, data: bytes, *extra):
    L = ref_sim.lib()
    f = getattr(L, name)
    f.restype = C.c_int64
    f.argtypes = [C.c_char_p, C.c_int64] + [C.c_int] * len(extra) + [C.c_void_p, C.c_int64]
    cap = 1 << 26
    buf = C.create_string_buffer(cap)
    n = f(data, len(data), *extra, C.cast(buf, C.c_void_p), cap)
    if n < 0:
        return None, buf.raw[:-n - 1].decode()
    return buf.raw[:n], None


def ref_columns(data: bytes, n):
    L = ref_sim.lib()
    L.kxref_trace_columns.restype = C.c_int64
    L.kxref_trace_columns.argtypes = [C.c_char_p, C.c_int64, C.c_int64] + [C.c_void_p] * 5
    out = [np.zeros(max(n, 1)), np.zeros(max(n, 1)), np.zeros(max(n, 1)), np.zeros(max(n, 1), np.int64),
           np.zeros(max(n, 1), np.int64)]
    got = L.kxref_trace_columns(data, len(data), n, *[a.ctypes.data for a in out])
    out = [a[:n] for a in out]
    assert got == n
    return out


def device_report(t: Trace, max_loop=3):
    g = t.analyze()
    s = g.report()
    for node in g.nodes():
        s += f"depth {node} {g.topo_depth(node)}\n"
        for p in g.downstream_paths(node, max_loop):
            s += f"path {node}:" + "".join(" " + x for x in p) + "\n"
    return s


def synthetic(seed, n_wf=300, header=True, blank=True, shuffle=True):
    """Workflows of four fixed call-graph templates (a branch, a fan-out whose
    spans overlap or not, a pipeline with a feedback loop, a single call),
    random timing, a few conflicting entries; lines shuffled."""
    rng = np.random.default_rng(seed)
    lines = []
    for w in range(n_wf):
        msg = f"m-{w}" if w % 7 else f"job_{w:05d}"
        app = float(rng.uniform(0, 500))
        t = app + float(rng.uniform(0, 1))
        kind = int(rng.integers(0, 4))
        recs = []

        def call(agent, up, start, dur):
            recs.append((agent, up, start, start + dur))
            return start + dur

        if kind == 0:  # QA branch
            e = call("Router", "", t, float(rng.uniform(0.1, 1)))
            call("Math" if rng.random() < 0.5 else "Humanities", "Router", e, float(rng.uniform(0.5, 3)))
        elif kind == 1:  # fan-out: mostly parallel under Researcher, mostly sequential under Planner
            up = "Researcher" if rng.random() < 0.5 else "Planner"
            e = call(up, "", t, float(rng.uniform(0.5, 2)))
            kids = ["Writer", "écrit", "a1"][: int(rng.integers(2, 4))]
            if (up == "Researcher") == (rng.random() < 0.8):
                for k in kids:
                    call(k, up, e + float(rng.uniform(0, 0.3)), float(rng.uniform(1, 2)))
            else:  # touching endpoints are not simultaneity
                s0 = e
                for k in kids:
                    s0 = call(k, up, s0, float(rng.uniform(0.2, 1))) + (0.0 if rng.random() < 0.4 else 0.1)
        elif kind == 2:  # pipeline with a QA -> Engineer feedback loop
            e = call("ProductManager", "", t, 1.0)
            e = call("Architect", "ProductManager", e, 1.0)
            e = call("Engineer", "Architect", e, 2.0)
            for _ in range(int(rng.integers(1, 4))):
                e = call("QA", "Engineer", e, 0.5)
                if rng.random() < 0.6:
                    e = call("Engineer", "QA", e, 1.5)
        else:  # one call
            call("Z_last", "", t, float(rng.uniform(0.1, 1)))
        if rng.random() < 0.04:  # a conflicting entry
            recs.append(("Router" if recs[0][0] != "Router" else "Z_last", "", t, t + 0.5))
        for a, u, s0, s1 in recs:
            lines.append(f"{msg},{a},{u},{s0:.9f},{s1:.9f},{int(rng.integers(1, 900))},"
                         f"{int(rng.integers(1, 400))},{app:.9f}")
    if shuffle:
        rng.shuffle(lines)
    if blank:
        for _ in range(5):
            lines.insert(int(rng.integers(0, len(lines))), "")
    return ("\n".join(([HEADER] if header else []) + lines) + "\n").encode()


def engine_trace(seed=3):
    """A simulated trace: the device engine's per-call exec times of one
    co-located replica, upstream = the parent call's agent."""
    from paper_2508_06948_b200 import DispatcherConfig, InstanceProfile
    rz = E.realize("colocated", 6.0, 200.0, seed)
    b = E.concat([rz])
    inst = [InstanceProfile(id=i, capacity_tokens=3000.0, max_batch=8) for i in range(4)]
    res = E.run_replicas(b, inst, "fcfs", DispatcherConfig("time_slot", oracle_expected_time=True),
                         topo_depth=np.ones(10, np.int32))
    n = int(res["counts"][0][0])
    order = res["call_order"][:n]
    names = [E._abi.load().kx_builtin_agent_name(a).decode() for a in range(10)]
    wf = np.repeat(np.arange(len(rz["arrival"])), np.diff(rz["wf_offsets"]))
    lines = [HEADER]
    for j, c in enumerate(order):
        w = wf[c]
        p = rz["parent"][c]
        up = names[rz["agent"][rz["wf_offsets"][w] + p]] if p >= 0 else ""
        lines.append(f"m-{w},{names[rz['agent'][c]]},{up},{res['exec_start'][j]:.9f},{res['exec_end'][j]:.9f},"
                     f"{rz['prompt'][c]},{rz['target'][c]},{rz['arrival'][w]:.9f}")
    return ("\n".join(lines) + "\n").encode()


def check_against_reference(data):
    t = Trace(data)
    ref_txt, err = ref_call("kxref_trace_report", data, 3)
    assert err is None, err
    cols = t.columns()
    es, ee, as_, pt, ot = ref_columns(data, t.n)
    assert np.array_equal(bits(cols["exec_start"]), bits(es))
    assert np.array_equal(bits(cols["exec_end"]), bits(ee))
    assert np.array_equal(bits(cols["app_start"]), bits(as_))
    assert np.array_equal(cols["prompt_tokens"], pt) and np.array_equal(cols["output_tokens"], ot)
    ref_w, err = ref_call("kxref_trace_write", data)
    assert err is None and t.format() == ref_w, "write_trace bytes differ"
    assert device_report(t) == ref_txt.decode(), "workflow reconstruction differs"
    return t


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_synthetic_traces_match_reference(gpu_lib, seed):
    t = check_against_reference(synthetic(seed, header=seed != 2, blank=seed != 3))
    g = t.analyze()
    kinds = {p.kind for p in g.fanouts().values()}
    assert {"parallel", "sequential", "single"} <= kinds
    assert g.diagnostics() and g.feedback_edges()


def test_simulated_trace_matches_reference(gpu_lib):
    check_against_reference(engine_trace())


def test_number_forms_match_reference(gpu_lib):
    # forms std::stod accepts inside the exact fast path
    lines = [HEADER, "m-1,A,,1e-3, 2.5,+3,0007,0", "m-1,B,A,.5,1.,1,1,0.000000001",
             "m-2,A,,12345678.123456789,12345679,5,5,12345678.0", "m-3,A,,-0.0,0,1,1,-0.0",
             "m-4,C,,9007199.254740993,9999999999.999999999,2,2,9007199.254740993",
             "m-5,C,,0.1234567890123456789,1234567890123456789e-9,1,1,0.000000000000000000001e3",
             "m-6,C,,4503599627370497.5,4503599627370497.500000000,1,1,1e15"]
    check_against_reference(("\n".join(lines)).encode())  # no trailing newline


BAD = [
    ("m-1,A,,1,2,3,4", "expected 8 fields"),
    ("m-1,A,,1,2,3,4,0,9", "expected 8 fields"),
    ("m-1,A,,x,2,3,4,0", "bad numeric field 'exec_start'"),
    ("m-1,A,,1,,3,4,0", "bad numeric field 'exec_end'"),
    ("m-1,A,,1,2,3.5,4,0", "bad count field 'prompt_tokens'"),
    ("m-1,A,,1,2,3,99999999999999999999,0", "bad count field 'output_tokens'"),
    ("m-1,A,,1,2,3,4,1e", "bad numeric field 'app_start'"),
    ("m-1,A,,1,2,3,4,0\r", "bad numeric field 'app_start'"),
    (",A,,1,2,3,4,0", "empty msg_id"),
    ("m-1,,,1,2,3,4,0", "empty agent"),
    ("m-1,A,,1,2,3,4,-1", "app_start < 0"),
    ("m-1,A,,1,2,3,4,1.5", "exec_start < app_start"),
    ("m-1,A,,2,1,3,4,0", "exec_end < exec_start"),
    ("m-1,A,,1,2,0,4,0", "prompt_tokens < 1"),
    ("m-1,A,,1,2,3,0,0", "output_tokens < 1"),
]


@pytest.mark.parametrize("line,what", BAD)
def test_bad_lines_match_reference_message(gpu_lib, line, what):
    data = "\n".join([HEADER, "m-0,A,,1,2,3,4,0", "", line, "m-1,A,,x"]).encode()
    _, ref_err = ref_call("kxref_trace_report", data, 3)
    assert ref_err is not None and what in ref_err
    with pytest.raises(KxError) as e:
        Trace(data)
    assert e.value.code == 1
    assert str(e.value).split("] ", 1)[1] == ref_err


@pytest.mark.parametrize("num", ["0x1p3", "inf", "nan", "1.00000000000000000001", "1e30"])
def test_numbers_outside_the_exact_forms_are_refused(gpu_lib, num):
    data = f"{HEADER}\nm-1,A,,0,{num},1,1,0\n".encode()
    _, ref_err = ref_call("kxref_trace_write", data)  # the reference accepts (or rejects) them
    with pytest.raises(KxError) as e:
        Trace(data)
    assert "exact decimal forms" in str(e.value) or (ref_err is not None and ref_err in str(e.value))


def test_empty_and_header_only_traces(gpu_lib):
    for data in [b"", (HEADER + "\n").encode(), b"\n\n"]:
        t = Trace(data)
        assert t.n == 0
        ref_txt, err = ref_call("kxref_trace_report", data, 3)
        assert err is None and device_report(t) == ref_txt.decode()
        assert t.format() == ref_call("kxref_trace_write", data)[0]
