"""kx_expected_exec_times (ProfilerSnapshot::expected_exec_time,
profiler.cpp:11-16 -> mode_estimate, distribution.cpp:46-86) on the B200
against the oracle restatement, which tests/test_oracle_golden.py pins to
the reference's own distribution fixtures. Every sample count from 0 to
4200 (so every cbrt(n) the histogram width uses there), plus the edge
shapes: all-equal sets, zero IQR (64 bins), ties between modal bins (lowest
bin wins), below min_samples (median), heavy tails (4096-bin clamp)."""
import ctypes as C

import numpy as np
import pytest

import oracle_ffi as O
from helpers import bits

pytestmark = pytest.mark.gpu


def run(lib, sets, min_samples=16, fallback=1.25):
    off = np.zeros(len(sets) + 1, np.int64)
    off[1:] = np.cumsum([len(s) for s in sets])
    flat = np.ascontiguousarray(np.concatenate(sets) if off[-1] else np.zeros(1), np.float64)
    out = np.zeros(len(sets))
    rc = lib.kx_expected_exec_times(len(sets), off.ctypes.data, flat.ctypes.data, min_samples, fallback,
                                    out.ctypes.data)
    assert rc == 0
    return out


def expect(sets, min_samples=16, fallback=1.25):
    return np.array([fallback if len(s) == 0 else O.mode_estimate(s, min_samples)[0] for s in sets])


def test_every_sample_count(gpu_lib):
    rng = np.random.default_rng(11)
    sets = [np.sort(rng.gamma(2.0, 1.5, n)) for n in range(0, 4201)]
    assert np.array_equal(bits(run(gpu_lib, sets)), bits(expect(sets)))


def test_edge_shapes(gpu_lib):
    rng = np.random.default_rng(12)
    sets = [
        np.full(40, 3.5),                                          # degenerate: lo
        np.sort(np.r_[np.zeros(30), np.ones(30), [5.0]]),           # two equal modes
        np.sort(np.r_[np.full(50, 2.0), rng.uniform(0, 9, 3)]),     # iqr == 0 -> 64 bins
        np.sort(rng.uniform(0, 1, 15)),                            # median fallback
        np.sort(np.r_[rng.uniform(0, 1, 2000), [1e6]]),             # bins clamp to 4096
        np.sort(rng.integers(0, 7, 5000).astype(np.float64) * 0.25),  # many exact ties
        np.sort(rng.lognormal(0, 2, 100_000)),
        np.array([], np.float64),
    ]
    assert np.array_equal(bits(run(gpu_lib, sets)), bits(expect(sets)))
    assert np.array_equal(bits(run(gpu_lib, sets, min_samples=1)), bits(expect(sets, min_samples=1)))


def test_rejects_unsorted(gpu_lib):
    off = np.array([0, 3], np.int64)
    s = np.array([1.0, 0.5, 2.0])
    out = np.zeros(1)
    assert gpu_lib.kx_expected_exec_times(1, off.ctypes.data, s.ctypes.data, 16, 1.0, out.ctypes.data) != 0
