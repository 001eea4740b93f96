"""The product's host-side realize() restatement (kx_workload.cpp) against
the reference's realize() output (tests/golden/dp_*.kxf, made by
oracle/gen_golden.cpp). Host code only: no GPU needed."""
import ctypes as C

import numpy as np
import pytest

import kxf
import paper_2508_06948_b200 as kx
from paper_2508_06948_b200 import _abi
from helpers import bits


def realize(mask, rate, duration, seed, prefill, decode):
    lib = kx.load()
    r = C.c_void_p()
    _abi.check(lib.kx_realize_builtin(mask, rate, duration, seed, prefill, decode, C.byref(r)))
    nw, nc = C.c_int64(), C.c_int64()
    lib.kx_realization_sizes(r, C.byref(nw), C.byref(nc))
    out = dict(arrival=np.zeros(nw.value), app=np.zeros(nw.value, np.int32),
               wf_offsets=np.zeros(nw.value + 1, np.int64), agent=np.zeros(nc.value, np.int32),
               parent=np.zeros(nc.value, np.int32), prompt=np.zeros(nc.value, np.int64),
               target=np.zeros(nc.value, np.int64), pure_exec=np.zeros(nc.value),
               remaining=np.zeros(nc.value), uid=np.zeros(nc.value, np.uint64))
    lib.kx_realization_copy(r, *[v.ctypes.data for v in out.values()])
    lib.kx_realization_free(r)
    return out


@pytest.mark.parametrize("name,mask,rate,duration,seed,prefill,decode", [
    ("dp_colocated.kxf", 7, 3.0, 400.0, 3, 8000.0, 50.0),
    ("dp_cg.kxf", 4, 2.0, 300.0, 11, 6000.0, 40.0),
])
def test_realize_port_is_the_reference_stream(name, mask, rate, duration, seed, prefill, decode):
    d = kxf.read(name)
    got = realize(mask, rate, duration, seed, prefill, decode)
    assert np.array_equal(bits(got["arrival"]), bits(d["arrival"]))
    assert np.array_equal(got["wf_offsets"], d["wf_offsets"])
    assert np.array_equal(got["agent"], d["builtin_agent"])
    assert np.array_equal(got["parent"], d["parent"])
    assert np.array_equal(got["prompt"], d["prompt"])
    assert np.array_equal(got["target"], d["target"])
    assert np.array_equal(got["uid"], d["uid"])
    assert np.array_equal(bits(got["pure_exec"]), bits(d["pure_exec"]))
    assert np.array_equal(bits(got["remaining"]), bits(d["remaining_exec"]))


def test_builtin_agent_names():
    lib = kx.load()
    names = [lib.kx_builtin_agent_name(i).decode() for i in range(10)]
    assert names[0] == "Router" and names[9] == "QAEngineer"
    assert lib.kx_builtin_agent_name(10) is None


def test_invalid_rate_is_invalid_argument():
    lib = kx.load()
    r = C.c_void_p()
    assert lib.kx_realize_builtin(7, 0.0, 10.0, 1, 8000.0, 50.0, C.byref(r)) == _abi.KX_ERR_INVALID
