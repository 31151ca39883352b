"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/fgt1d_b200.h declares (and nothing silently missing), and the
host-side logic that needs no device.  No compute call is made here when no
GPU is present -- except to check that compute entry points fail loudly
(there is no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1909_09825_b200 as fgt
from paper_1909_09825_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fgt1d_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(fgt_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_expected_entry_points():
    names = declared_functions()
    for must in ["fgt_plan_create", "fgt_apply_general", "fgt_apply_same", "fgt_direct",
                 "fgt_cf_soe", "fgt_gauss_transform", "fgt_plan_destroy", "fgt_mode_sums",
                 "fgt_plan_gap_table", "fgt_apply_chunk_aggregate", "fgt_apply_chunk_finish",
                 "fgt_chunk_carries", "fgt_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_capi.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_every_declared_symbol():
    assert set(declared_functions()) <= set(_capi.SIGNATURES)


def test_no_cpu_fallback_when_no_device():
    if _capi.lib().fgt_device_count() > 0:
        pytest.skip("device present: covered by the gpu tests")
    with pytest.raises(fgt.DeviceError):
        fgt.gauss_transform([0.1, 0.2], [0.3], [1.0], 0.5, ne=4)
    with pytest.raises(fgt.DeviceError):
        fgt.direct_transform([0.1], [0.3], [1.0], 0.5)


def test_validation_errors_raise_before_device_work():
    # test_transform.cpp:260-280: domain / invalid-argument -> ValueError in python
    soe = fgt.fold(fgt.cf_soe(8))
    base = dict(targets=[0.0, 0.5, 1.0], sources=[0.0, 0.1], strengths=[1.0, 2.0])
    for bad in [dict(delta=0.0), dict(delta=-2.0), dict(delta=float("nan")),
                dict(delta=1.0, targets=[0.0, float("nan")]),
                dict(delta=1.0, sources=[0.0, float("inf")]),
                dict(delta=1.0, strengths=[1.0])]:
        req = fgt.TransformRequest(**{**base, **bad})
        with pytest.raises(ValueError):
            fgt.plan(req, soe)


def test_chunk_carry_algebra_matches_sequential_recurrence():
    """fgt_chunk_carries: forward C_g = A_{g-1} C_{g-1} + F_{g-1};
    backward D_g = A_{g+1} D_{g+1} + G_{g+1}."""
    rng = np.random.default_rng(0)
    G, ne = 5, 4
    A = (rng.random((G, ne)) * 0.9) * np.exp(1j * rng.random((G, ne)))
    F = rng.standard_normal((G, ne)) + 1j * rng.standard_normal((G, ne))
    Gb = rng.standard_normal((G, ne)) + 1j * rng.standard_normal((G, ne))
    agg = np.concatenate([A, F, Gb], axis=1)  # [G][3ne] complex
    flat = np.empty(G * 6 * ne)
    flat[0::2] = agg.reshape(-1).real
    flat[1::2] = agg.reshape(-1).imag
    out = np.empty(G * 4 * ne)
    _capi.check(_capi.lib().fgt_chunk_carries(flat.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                              G, ne, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    car = (out[0::2] + 1j * out[1::2]).reshape(G, 2 * ne)
    f = np.zeros(ne, complex)
    for g in range(G):
        assert np.allclose(car[g, :ne], f, rtol=1e-15, atol=1e-15)
        f = A[g] * f + F[g]
    b = np.zeros(ne, complex)
    for g in reversed(range(G)):
        assert np.allclose(car[g, ne:], b, rtol=1e-15, atol=1e-15)
        b = A[g] * b + Gb[g]


def test_merge_split_tie_rule():
    import bench
    x = np.array([0.1, 0.3, 0.3, 0.7])
    y = np.array([0.3, 0.3, 0.5])
    # merged: 0.1(t) 0.3(s) 0.3(s) 0.3(t) 0.3(t) 0.5(s) 0.7(t)
    want = [0, 1, 1, 1, 2, 3, 3, 4]
    assert [bench.merge_split(x, y, d) for d in range(8)] == want
