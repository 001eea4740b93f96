"""K1 on the B200: finalize_instance's uid / pure_exec / remaining_exec and
record_remaining's samples, bit-exact against the reference fixtures."""
import numpy as np
import pytest

import kxf
import oracle_ffi as O
import paper_2508_06948_b200 as kx
from helpers import bits

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["dp_colocated.kxf", "dp_fanout.kxf", "dp_wide.kxf"])
def test_orchestrator_dp_matches_reference(gpu_lib, name):
    d = kxf.read(name)
    uid, pure, rem = kx.orchestrator_dp(d["wf_offsets"], d["parent"], d["prompt"], d["target"],
                                        float(d["prefill_rate"][0]), float(d["decode_rate"][0]), 1)
    assert np.array_equal(uid, d["uid"])
    assert np.array_equal(bits(pure), bits(d["pure_exec"]))
    assert np.array_equal(bits(rem), bits(d["remaining_exec"]))


def random_forest(rng, n_wf, max_calls):
    off, parent = [0], []
    for _ in range(n_wf):
        n = int(rng.integers(1, max_calls + 1))
        parent += [-1] + [int(rng.integers(0, c)) for c in range(1, n)]
        off.append(len(parent))
    m = len(parent)
    return (np.array(off), np.array(parent, np.int32), rng.integers(1, 500, m), rng.integers(1, 900, m))


@pytest.mark.parametrize("n_wf,max_calls", [(1, 1), (10_000, 11), (2000, 80), (200_000, 6)])
def test_orchestrator_dp_matches_oracle_random(gpu_lib, n_wf, max_calls):
    rng = np.random.default_rng(n_wf)
    off, parent, pr, tg = random_forest(rng, n_wf, max_calls)
    got = kx.orchestrator_dp(off, parent, pr, tg, 8000.0, 50.0, 7)
    exp = O.finalize(off, parent, pr, tg, 8000.0, 50.0, 7)
    assert np.array_equal(got[0], exp[0])
    assert np.array_equal(bits(got[1]), bits(exp[1]))
    assert np.array_equal(bits(got[2]), bits(exp[2]))


def test_orchestrator_rejects_non_parents_first(gpu_lib):
    with pytest.raises(kx.KxError):
        kx.orchestrator_dp([0, 2], [1, -1], [1, 1], [1, 1])


def test_record_remaining_matches_profiler(gpu_lib):
    d = kxf.read("remaining.kxf")
    fin, smp = kx.record_remaining(d["rec_offsets"], d["exec_start"], d["exec_end"])
    efin, esmp = O.record_remaining(d["rec_offsets"], d["exec_start"], d["exec_end"])
    assert np.array_equal(bits(fin), bits(efin))
    assert np.array_equal(bits(smp), bits(esmp))
    for a in np.unique(d["samples_agent"]):
        exp = d["samples_sorted"][d["samples_agent"] == a]
        assert np.array_equal(bits(np.sort(smp[d["agent"] == a])), bits(exp))
