"""Pins for oracle O1-O4 (Philox4x32-10, uniform map, Box-Muller) -- CPU only."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest
from scipy import stats

from _golden import philox_kat

PIN_SRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pins", "curand_philox_pin.cpp")


@pytest.fixture(scope="module")
def curand_pin(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("pin") / "pin.so")
    subprocess.check_call(["g++", "-O2", "-fPIC", "-shared", "-D__host__=", "-D__device__=",
                           "-D__forceinline__=inline", "-I/usr/local/cuda/include", PIN_SRC,
                           "-o", out])
    lib = C.CDLL(out)
    u32 = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
    lib.pin_curand_philox.argtypes = [C.c_uint64, u32, C.c_int64, u32]

    def f(seed, ctr):
        ctr = np.ascontiguousarray(ctr, np.uint32)
        o = np.empty_like(ctr)
        lib.pin_curand_philox(C.c_uint64(seed), ctr, ctr.shape[0], o)
        return o
    return f


def test_philox_known_answer_vectors(orc):
    for ctr, key, expect in philox_kat():
        seed = key[0] | (key[1] << 32)
        got = orc.philox(seed, np.array([ctr], np.uint32))[0]
        assert [int(v) for v in got] == expect


def test_philox_matches_host_curand(orc, curand_pin):
    r = np.random.default_rng(123)
    for seed in [0, 1, 0xFFFFFFFFFFFFFFFF, int(r.integers(0, 2**63))]:
        ctr = r.integers(0, 2**32, (100_000, 4), dtype=np.uint64).astype(np.uint32)
        ctr[:4] = [[0, 0, 0, 0], [0xFFFFFFFF] * 4, [1, 0, 0, 0], [0, 0, 0, 1]]
        np.testing.assert_array_equal(orc.philox(seed, ctr), curand_pin(seed, ctr))


def test_uniform_exact_and_open_interval(orc):
    rs = [0, 1, 511, 512, 0xFFFFFFFF, 0x80000000, 123456789]
    for r in rs:
        u = orc.uniform_u32(r)
        k = u * 2**24
        assert k == int(k) and int(k) % 2 == 1          # odd multiple of 2^-24
        assert (int(k) - 1) // 2 == r >> 9              # reconstructs the top 23 bits
        assert 0.0 < u < 1.0
        assert np.float32(u) == u                        # exactly representable in fp32
    assert orc.uniform_u32(0) == 2.0**-24
    assert orc.uniform_u32(0xFFFFFFFF) == 1.0 - 2.0**-24


def test_box_muller_moments_and_ks(orc):
    n = 250_000
    ctr = np.zeros((n, 4), np.uint32)
    ctr[:, 0] = np.arange(n)
    ctr[:, 1] = 7
    z = orc.normals_batch(42, ctr).ravel()           # 1e6 normals
    assert abs(z.mean()) < 0.005
    assert abs(z.var() - 1.0) < 0.005
    assert abs(stats.kurtosis(z, fisher=False) - 3.0) < 0.05
    assert stats.kstest(z, "norm").pvalue > 1e-3
    # the two Box-Muller outputs of one pair are uncorrelated
    zz = z.reshape(-1, 4)
    assert abs(np.corrcoef(zz[:, 0], zz[:, 1])[0, 1]) < 0.01
    assert np.abs(z).max() <= np.sqrt(-2 * np.log(2.0**-24)) + 1e-12   # truncation bound 5.77


def test_streams_deterministic_and_distinct(orc):
    ctr = np.array([[5, 9, 3, 0]], np.uint32)
    a = orc.philox(77, ctr)
    np.testing.assert_array_equal(a, orc.philox(77, ctr))
    assert not np.array_equal(a, orc.philox(78, ctr))                    # seed change
    for pos in range(4):                                                 # any counter word
        c2 = ctr.copy()
        c2[0, pos] += 1
        assert not np.array_equal(a, orc.philox(77, c2))
    # empirical independence of neighbouring streams (particle p vs p+1)
    n = 100_000
    c = np.zeros((n, 4), np.uint32)
    c[:, 0] = np.arange(n)
    u = orc.philox(3, c).astype(np.float64)
    assert abs(np.corrcoef(u[:-1, 0], u[1:, 0])[0, 1]) < 0.01
