"""§8(f)2: the priority table's W1 distance matrix (priority.cpp:15-65,
distribution.cpp:9-31). The oracle restatement is pinned to the reference's
matrices (w1_matrix.kxf, written by oracle/gen_golden.cpp from the
reference's build_distance_matrix_from_samples); the B200 kernel must match
them bit for bit, and the oracle on larger random sets."""
import numpy as np
import pytest

import kxf
import oracle_ffi as O
from helpers import bits


def golden_cases():
    d = kxf.read("w1_matrix.kxf")
    so, cs, mo = d["set_offsets"], d["case_sets"], d["matrix_offsets"]
    for c in range(len(cs) - 1):
        sets = [d["samples"][so[k]:so[k + 1]] for k in range(cs[c], cs[c + 1])]
        m = len(sets) + 1
        yield sets, d["matrix"][mo[c]:mo[c + 1]].reshape(m, m)


def oracle_matrix(sets):
    m = len(sets) + 1
    lab = list(sets) + [np.zeros(1)]
    out = np.zeros((m, m))
    for i in range(m):
        for j in range(i + 1, m):
            out[i, j] = out[j, i] = O.wasserstein(lab[i], lab[j])
    return out


def test_oracle_matches_reference_matrices():
    n = 0
    for sets, ref in golden_cases():
        assert np.array_equal(bits(oracle_matrix(sets)), bits(ref))
        n += 1
    assert n == 6


@pytest.mark.gpu
def test_w1_matrix_matches_reference(gpu_lib):
    import paper_2508_06948_b200 as kx
    for sets, ref in golden_cases():
        got = kx.w1_matrix(sets)
        assert np.array_equal(bits(got), bits(ref))


@pytest.mark.gpu
def test_w1_matrix_random_vs_oracle(gpu_lib):
    import paper_2508_06948_b200 as kx
    rng = np.random.default_rng(7)
    sets = [np.sort(np.where(rng.random(k) < 0.3, np.floor(rng.uniform(0, 9, k)), rng.uniform(0, 40, k)))
            for k in rng.integers(1, 700, 40)]
    assert np.array_equal(bits(kx.w1_matrix(sets)), bits(oracle_matrix(sets)))


@pytest.mark.gpu
def test_w1_matrix_errors(gpu_lib):
    import paper_2508_06948_b200 as kx
    with pytest.raises(kx.KxError) as e:
        kx.w1_matrix([])
    assert e.value.code == 1
    with pytest.raises(kx.KxError) as e:
        kx.w1_matrix([np.ones(3), np.zeros(0)])
    assert e.value.code == 1
