"""Plan-time checks on inputs larger than a few plan tiles (GPU).

The reference's plan() rejects non-finite coordinates (check_points,
transform.cpp:21-25), detects same points by exact vector equality
(:214-216) and sorts each set stably (:27-39).  On the device a sorted input
is checked in the same pass that cuts the merged stream into tiles; an
unsorted one gets an element-wise pass over the arrays as given (its
merge-path tiles need not cover every element).  These cases use inputs of
many tiles, unsorted and sorted, through host and device pointers.
"""
import ctypes

import numpy as np
import pytest

import oracle
import paper_1909_09825_b200 as fgt
from paper_1909_09825_b200 import _capi
from paper_1909_09825_b200.transform import _soe_args
from paper_1909_09825_b200.transform import uniform_points_array as up

pytestmark = pytest.mark.gpu
PD = ctypes.POINTER(ctypes.c_double)
N_BIG = 200_003  # ~37 plan tiles of 5376 merged elements (21 segments)


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    return torch


def device_plan_rc(torch, x, y, delta=1e-3, ne=4):
    """fgt_plan_create on device pointers -> (rc, plan info dict or None)."""
    L = _capi.lib()
    xd = torch.as_tensor(np.asarray(x, dtype=np.float64), device="cuda")
    yd = torch.as_tensor(np.asarray(y, dtype=np.float64), device="cuda")
    keep, sargs = _soe_args(fgt.fold(fgt.cf_soe(2 * ne)))
    h = ctypes.c_void_p()
    rc = L.fgt_plan_create(ctypes.cast(xd.data_ptr(), PD), xd.numel(), ctypes.cast(yd.data_ptr(), PD),
                           yd.numel(), float(delta), *sargs, _capi.FGT_DEVICE_PTRS, 0, None,
                           ctypes.byref(h))
    info = None
    if rc == _capi.FGT_OK:
        same, ts, ss = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _capi.check(L.fgt_plan_info(h, None, None, None, ctypes.byref(same), ctypes.byref(ts),
                                    ctypes.byref(ss), None))
        info = dict(same=bool(same.value), tsorted=bool(ts.value), ssorted=bool(ss.value))
        L.fgt_plan_destroy(h)
    del keep
    return rc, info


@pytest.mark.parametrize("sort_it", [False, True])
def test_same_points_one_interior_change(torch_cuda, sort_it):
    x = up(N_BIG, 11, 3)
    if sort_it:
        x = np.sort(x)
    rc, info = device_plan_rc(torch_cuda, x, x.copy())
    assert rc == _capi.FGT_OK and info["same"]
    for pos in (N_BIG // 2, 7777, N_BIG - 2):
        y = x.copy()
        y[pos] = np.nextafter(y[pos], 2.0)  # keeps the order of a sorted input
        rc, info = device_plan_rc(torch_cuda, x, y)
        assert rc == _capi.FGT_OK and not info["same"], pos
    # the reference's equality: same values in the same order, -0.0 == 0.0
    z = x.copy()
    z[100] = 0.0
    w = z.copy()
    w[100] = -0.0
    rc, info = device_plan_rc(torch_cuda, z, w)
    assert rc == _capi.FGT_OK and info["same"]


@pytest.mark.parametrize("where", ["targets", "sources"])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
@pytest.mark.parametrize("sort_it", [False, True])
def test_non_finite_interior_rejected_through_device_pointers(torch_cuda, where, bad, sort_it):
    x = up(N_BIG, 12, 3)
    y = up(N_BIG + 5000, 12, 0)
    if sort_it:
        x, y = np.sort(x), np.sort(y)
    v = x if where == "targets" else y
    v[len(v) // 3 + 17] = bad
    rc, _ = device_plan_rc(torch_cuda, x, y)
    assert rc == _capi.FGT_ERR_DOMAIN
    msg = _capi.lib().fgt_last_error().decode()
    assert ("target" if where == "targets" else "source") in msg


def test_targets_checked_before_sources(torch_cuda):
    # transform.cpp:202-204: a bad target is reported even if sources are bad too
    x = up(N_BIG, 13, 3)
    y = up(N_BIG, 13, 0)
    x[N_BIG - 10] = np.nan
    y[5] = np.inf
    rc, _ = device_plan_rc(torch_cuda, x, y)
    assert rc == _capi.FGT_ERR_DOMAIN
    assert "target" in _capi.lib().fgt_last_error().decode()


@pytest.mark.parametrize("which", ["sources", "targets", "both_nearly"])
def test_partly_unsorted_input_is_detected_and_sorted(torch_cuda, which):
    # one set sorted, the other sorted except for a few swapped pairs deep
    # inside: the disorder can sit in a tile whose merge-path range is
    # inconsistent, so it must be found by the element-wise pass
    n = N_BIG
    x = np.sort(up(n, 14, 3))
    y = np.sort(up(n + 333, 14, 0))
    a = 2.0 * up(n + 333, 14, 1) - 1.0
    rng = np.random.default_rng(3)
    targets = [y] if which == "sources" else [x] if which == "targets" else [x, y]
    for v in targets:
        for i in rng.integers(1000, v.size - 1000, size=4):
            v[i], v[i + 500] = v[i + 500], v[i]
    rc, info = device_plan_rc(torch_cuda, x, y)
    assert rc == _capi.FGT_OK
    assert info["tsorted"] == (which == "sources")
    assert info["ssorted"] == (which == "targets")
    u = fgt.apply_general(fgt.plan(fgt.TransformRequest(x, y, a, 1e-3),
                                   fgt.fold(fgt.cf_soe(8))), a)
    ref = oracle.transform(x, y, a, 1e-3, ne=4, mode=0)
    assert np.max(np.abs(u - ref)) <= 1e-12 * np.sum(np.abs(a))


def test_device_array_transform_rejects_nan_in_unsorted_input(torch_cuda):
    torch = torch_cuda
    x = torch.as_tensor(up(N_BIG, 15, 3), device="cuda")
    y = torch.as_tensor(up(N_BIG, 15, 0), device="cuda")
    a = torch.as_tensor(up(N_BIG, 15, 1), device="cuda")
    y[N_BIG // 2] = float("nan")
    with pytest.raises(ValueError):
        fgt.gauss_transform(x, y, a, 1e-3, ne=4)
