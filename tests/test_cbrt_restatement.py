"""The device's cbrt (kx_dist.cuh cbrt_glibc) replays glibc 2.39's
sysdeps/ieee754/dbl-64/s_cbrt.c: frexp, a degree-6 polynomial, one rational
correction, a 2^(k/3) factor and ldexp, every step one correctly rounded op.
glibc's cbrt is not correctly rounded, so the Freedman-Diaconis bin width of
mode_estimate (distribution.cpp:58) needs exactly this sequence.
Here the same op sequence in numpy (IEEE round-to-nearest, no contraction)
is checked against this host's libm, which is what the reference calls."""
import ctypes
import ctypes.util

import numpy as np

FACTOR = np.array([1.0 / 1.5874010519681994748, 1.0 / 1.2599210498948731648, 1.0,
                   1.2599210498948731648, 1.5874010519681994748])


def cbrt_restated(x):
    x = np.asarray(x, np.float64)
    xm, xe = np.frexp(np.abs(x))
    u = 0.784932344976639262 - 0.145263899385486377 * xm
    u = -1.83469277483613086 + u * xm
    u = 2.44693122563534430 + u * xm
    u = -2.11499494167371287 + u * xm
    u = 1.50819193781584896 + u * xm
    u = 0.354895765043919860 + u * xm
    t2 = (u * u) * u
    rem = np.fmod(xe, 3).astype(np.int64)          # C's % (truncating)
    quo = np.trunc(xe / 3.0).astype(np.int64)      # C's / (truncating)
    ym = ((u * (t2 + 2.0 * xm)) / (2.0 * t2 + xm)) * FACTOR[2 + rem]
    return np.ldexp(ym, quo)


def libm_cbrt():
    m = ctypes.CDLL(ctypes.util.find_library("m"))
    m.cbrt.restype = ctypes.c_double
    m.cbrt.argtypes = [ctypes.c_double]
    return m.cbrt


def test_restatement_matches_libm_on_sample_counts():
    # mode_estimate calls cbrt(n) for sample counts n >= 16
    cb = libm_cbrt()
    n = np.arange(1, 200_001, dtype=np.float64)
    ref = np.array([cb(float(v)) for v in n])
    assert np.array_equal(cbrt_restated(n).view(np.uint64), ref.view(np.uint64))


def test_restatement_matches_libm_on_random_doubles():
    cb = libm_cbrt()
    rng = np.random.default_rng(3)
    x = np.exp(rng.uniform(-300, 300, 50_000))
    ref = np.array([cb(float(v)) for v in x])
    assert np.array_equal(cbrt_restated(x).view(np.uint64), ref.view(np.uint64))


def test_libm_cbrt_is_not_correctly_rounded():
    # why the restatement is needed: a correctly rounded device cbrt would
    # disagree with the reference's libm on some sample counts
    cb = libm_cbrt()
    lib = ctypes.CDLL(ctypes.util.find_library("m"))
    lib.cbrtl.restype = ctypes.c_longdouble
    lib.cbrtl.argtypes = [ctypes.c_longdouble]
    diff = sum(cb(float(v)) != float(lib.cbrtl(float(v))) for v in range(16, 5000))
    assert diff > 0
