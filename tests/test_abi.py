"""C-ABI boundary checks that need no GPU: the library loads, exports every
entry point declared in include/kairos_b200.h, its struct layouts match the
header as compiled by gcc, and compute calls fail loudly without a device."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

import paper_2508_06948_b200 as kx
from paper_2508_06948_b200 import _abi

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "kairos_b200.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int64_t|int|void|const char\*)\s+(kx_\w+)\s*\(", text, re.M)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert len(names) >= 30
    assert set(names) == set(_abi.SIGNATURES), set(names) ^ set(_abi.SIGNATURES)


def test_library_exports_every_symbol():
    lib = kx.load()
    out = subprocess.run(["nm", "-D", "--defined-only", str(_abi.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (kx_\w+)", out))
    missing = set(declared_functions()) - exported
    assert not missing, missing
    assert lib.kx_abi_version() == 1


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu\\n", sizeof(kx_instance), sizeof(kx_dispatcher_config),
         sizeof(kx_sched_config), sizeof(kx_queue_view), sizeof(kx_decision));
  printf("%zu %zu %zu\\n", offsetof(kx_sched_config, queue_capacity),
         offsetof(kx_decision, agent), offsetof(kx_sched_config, log_capacity_per_pool));
  return 0;
}}""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", str(src), "-o", str(exe)], check=True)
    sizes, offs = subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n")[:2]
    assert [int(x) for x in sizes.split()] == [C.sizeof(_abi.kx_instance),
                                               C.sizeof(_abi.kx_dispatcher_config),
                                               C.sizeof(_abi.kx_sched_config),
                                               C.sizeof(_abi.kx_queue_view),
                                               C.sizeof(_abi.kx_decision)]
    assert [int(x) for x in offs.split()] == [_abi.kx_sched_config.queue_capacity.offset,
                                              _abi.kx_decision.agent.offset,
                                              _abi.kx_sched_config.log_capacity_per_pool.offset]


def test_cpp_adapter_header_compiles(tmp_path):
    src = tmp_path / "use.cpp"
    src.write_text('#include "kairos_b200.hpp"\nint main() { return 0; }\n')
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{ROOT / 'include'}", str(src)], check=True)


def test_no_device_fails_loudly():
    lib = kx.load()
    if lib.kx_device_available():
        pytest.skip("a GPU is visible; the no-device path is not reachable")
    with pytest.raises(kx.KxError) as e:
        kx.DeviceScheduler([kx.InstanceProfile(0)])
    assert e.value.code == _abi.KX_ERR_CUDA
    with pytest.raises(kx.KxError):
        kx.orchestrator_dp([0, 1], [-1], [10], [10])


def test_invalid_config_maps_to_invalid_argument():
    lib = kx.load()
    cfg = _abi.kx_sched_config()
    cfg.n_pools = 1
    cfg.n_instances = 0  # dispatcher needs matching instance lists
    h = C.c_void_p()
    assert lib.kx_sched_create(C.byref(cfg), C.byref(h)) == _abi.KX_ERR_INVALID
    assert b"instance" in lib.kx_last_error()
