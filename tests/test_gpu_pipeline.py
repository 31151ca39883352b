"""GPU tests of the pipelined host-buffer transform (fgt_transform_host).

The pipeline splits the merged stream into chunks on the host, computes each
chunk's aggregates from its sources alone, and plans / finishes each target
chunk as it uploads.  Its results must meet the same bar as plan + apply
(|u - oracle| <= 1e-12 sum|alpha|), whatever the chunking: the knobs
FGT_PIPE_MIN / FGT_PIPE_CHUNK force many small chunks here.  Inputs that are
not sorted, or not finite, must take the full path with the reference's
results and errors.
"""
import ctypes
import os

import numpy as np
import pytest

import oracle
import paper_1909_09825_b200 as fgt
from paper_1909_09825_b200 import _capi
from paper_1909_09825_b200.transform import uniform_points_array as up

pytestmark = pytest.mark.gpu
PARITY = 1e-12
PD = ctypes.POINTER(ctypes.c_double)


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if _capi.lib().fgt_device_count() < 1:
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")


@pytest.fixture
def small_chunks(monkeypatch):
    def set_(chunk, lo=1000):
        monkeypatch.setenv("FGT_PIPE_MIN", str(lo))
        monkeypatch.setenv("FGT_PIPE_CHUNK", str(chunk))
    return set_


def check(u, ref, a):
    err = np.max(np.abs(np.asarray(u) - ref)) / max(np.sum(np.abs(a)), 1e-300) if len(u) else 0.0
    assert err <= PARITY, err
    return err


def soe(ne):
    return fgt.fold(fgt.cf_soe(2 * ne))


@pytest.mark.parametrize("chunk", [997, 20000, 65536])
@pytest.mark.parametrize("delta,ne", [(1e-3, 6), (1e-6, 5), (1.0, 3)])
def test_pipelined_sorted_vs_oracle(small_chunks, chunk, delta, ne):
    small_chunks(chunk)
    M, N = 120000, 90000
    x = np.sort(up(M, 11, 3))
    y = np.sort(up(N, 11, 0))
    a = 2.0 * up(N, 11, 1) - 1.0
    u = fgt.transform_host(x, y, a, delta, soe(ne))
    check(u, oracle.transform(x, y, a, delta, ne=ne), a)


def test_pipelined_equals_plan_apply_and_one_shot(small_chunks):
    small_chunks(5000)
    M = N = 50000
    x = np.sort(up(M, 5, 3))
    y = np.sort(up(N, 5, 0))
    a = 2.0 * up(N, 5, 1) - 1.0
    s = soe(6)
    u = fgt.transform_host(x, y, a, 1e-4, s)
    p = fgt.plan(fgt.TransformRequest(x, y, a, 1e-4), s)
    check(u, np.asarray(fgt.apply_general(p, a)), a)
    # the python one-shot binding goes through the same entry point
    check(np.asarray(fgt.gauss_transform(x, y, a, 1e-4, ne=6)), np.asarray(u), a)


def test_pipelined_ties_same_points_and_grid(small_chunks):
    """Equal coordinates straddling chunk boundaries (sources before targets)."""
    small_chunks(777)
    g = np.round(up(40000, 3, 0) * 256) / 256.0  # 257 distinct values
    x = np.sort(g)
    a = 2.0 * up(40000, 3, 1) - 1.0
    u = fgt.transform_host(x, x, a, 1e-3, soe(4))
    check(u, oracle.transform(x, x, a, 1e-3, ne=4), a)
    y = np.sort(np.round(up(30000, 4, 0) * 64) / 64.0)
    b = 2.0 * up(30000, 4, 1) - 1.0
    u = fgt.transform_host(x, y, b, 1e-2, soe(6))
    check(u, oracle.transform(x, y, b, 1e-2, ne=6), b)


def test_pipelined_chunks_without_sources_or_targets(small_chunks):
    """Targets all left of the sources, then interleaved blocks: chunks with
    no sources and chunks with no targets."""
    small_chunks(3000)
    x = np.sort(up(20000, 8, 3)) * 0.5
    y = 0.5 + np.sort(up(20000, 8, 0)) * 0.5
    a = 2.0 * up(20000, 8, 1) - 1.0
    u = fgt.transform_host(x, y, a, 1e-2, soe(5))
    check(u, oracle.transform(x, y, a, 1e-2, ne=5), a)
    blocks = np.arange(40000) // 2500
    z = np.sort(up(40000, 9, 0))
    xt, ys = z[blocks % 2 == 0], z[blocks % 2 == 1]
    b = 2.0 * up(ys.size, 9, 1) - 1.0
    u = fgt.transform_host(xt, ys, b, 1e-5, soe(6))
    check(u, oracle.transform(xt, ys, b, 1e-5, ne=6), b)


def test_pipelined_clustered_wide_segments(small_chunks):
    small_chunks(10000)
    c = up(16, 0, 5)
    k = (up(60000, 0, 6) * 16).astype(int)
    x = np.sort(c[k] + 1e-3 * (up(60000, 0, 7) - 0.5))
    y = np.sort(c[(up(80000, 1, 6) * 16).astype(int)] + 1e-3 * (up(80000, 1, 7) - 0.5))
    a = up(80000, 1, 1)
    u = fgt.transform_host(x, y, a, 1e-6, soe(5))
    check(u, oracle.transform(x, y, a, 1e-6, ne=5), a)


def test_unsorted_input_falls_back_to_full_path(small_chunks):
    small_chunks(4000)
    x = up(30000, 2, 3)
    y = up(25000, 2, 0)
    a = 2.0 * up(25000, 2, 1) - 1.0
    u = fgt.transform_host(x, y, a, 1e-3, soe(6))  # original target order
    check(u, oracle.transform(x, y, a, 1e-3, ne=6), a)
    # sorted except one swap inside a single chunk (found by the device check)
    xs = np.sort(x)
    xs[20001], xs[20002] = xs[20002], xs[20001]
    u = fgt.transform_host(xs, np.sort(y), a, 1e-3, soe(6))
    check(u, oracle.transform(xs, np.sort(y), a, 1e-3, ne=6), a)
    # and one swap across a chunk boundary (found on the host)
    ys = np.sort(y)
    ys[0], ys[-1] = ys[-1], ys[0]
    u = fgt.transform_host(np.sort(x), ys, a, 1e-3, soe(6))
    check(u, oracle.transform(np.sort(x), ys, a, 1e-3, ne=6), a)


def _c_call(x, y, a, delta=1e-3, ne=6):
    s = soe(ne)
    tr, ti, wr, wi, sc = s.arrays()
    u = np.empty(x.size)
    rc = _capi.lib().fgt_transform_host(
        x.ctypes.data_as(PD), x.size, y.ctypes.data_as(PD), y.size, a.ctypes.data_as(PD), delta,
        tr.ctypes.data_as(PD), ti.ctypes.data_as(PD), wr.ctypes.data_as(PD), wi.ctypes.data_as(PD),
        sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), len(s), int(s.form),
        u.ctypes.data_as(PD), -1, None)
    return rc, u


def test_nonfinite_reports_targets_first_like_the_reference(small_chunks):
    """transform.cpp:202-204: targets are checked before sources, whichever
    chunk the bad values sit in."""
    small_chunks(2000)
    x = np.sort(up(20000, 1, 3))
    y = np.sort(up(20000, 1, 0))
    a = 2.0 * up(20000, 1, 1) - 1.0
    x2, y2 = x.copy(), y.copy()
    x2[-5] = np.inf
    y2[3] = np.nan
    rc, _ = _c_call(x2, y2, a)
    assert rc == _capi.FGT_ERR_DOMAIN
    assert b"target" in _capi.lib().fgt_last_error()
    rc, _ = _c_call(x, y2, a)
    assert rc == _capi.FGT_ERR_DOMAIN
    assert b"source" in _capi.lib().fgt_last_error()


def test_empty_and_small_sets(small_chunks):
    small_chunks(100, lo=10)
    x = np.sort(up(500, 1, 3))
    y = np.sort(up(400, 1, 0))
    a = 2.0 * up(400, 1, 1) - 1.0
    rc, u = _c_call(x, y[:0], a[:0])
    assert rc == 0 and np.all(u == 0.0)
    rc, u = _c_call(x[:0], y, a)
    assert rc == 0 and u.size == 0
    rc, u = _c_call(x, y, a)
    assert rc == 0
    check(u, oracle.transform(x, y, a, 1e-3, ne=6), a)
    rc, _ = _c_call(x, y, a, delta=-1.0)
    assert rc == _capi.FGT_ERR_DOMAIN


def test_large_default_chunking_vs_device_path():
    """Default knobs at a size that pipelines (2^23 merged points, G = 2..)."""
    n = 1 << 22
    x = np.sort(up(n, 4, 3))
    y = np.sort(up(n, 4, 0))
    a = 2.0 * up(n, 4, 1) - 1.0
    s = soe(6)
    u = fgt.transform_host(x, y, a, 1e-3, s)
    p = fgt.plan(fgt.TransformRequest(x, y, a, 1e-3), s)
    check(u, np.asarray(fgt.apply_general(p, a)), a)
