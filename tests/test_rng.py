"""The product's reference Rng (csrc/rng.hpp: parallel Box-Muller, parallel
canonical norm) is bit-identical to the oracle's sequential restatement of
rng.hpp:15-62 — the start vector of the power basis depends on it."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
import paper_2509_26475_b200 as P


def wl():
    L = P._wl()
    L.phx_wl_normals.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_double)]
    L.phx_wl_unit_vector.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_double)]
    return L


@pytest.mark.parametrize("n", [1, 2, 3, 1001, (1 << 18) + 3, 1 << 20])
def test_unit_vector_bitwise(n):
    seed = 0x9E3779B97F4A7C15
    out = np.empty(n)
    wl().phx_wl_unit_vector(C.c_uint64(seed), n, out.ctypes.data_as(C.POINTER(C.c_double)))
    assert np.array_equal(out, O.unit_vector(seed, n))


@pytest.mark.parametrize("n", [5, (1 << 17) + 1, 300001])
def test_normals_bitwise(n):
    out = np.empty(n)
    wl().phx_wl_normals(C.c_uint64(7), n, out.ctypes.data_as(C.POINTER(C.c_double)))
    assert np.array_equal(out, O.Rng(7).normals(n))
