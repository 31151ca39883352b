"""Device helpers behind the plan and the benchmark inputs (GPU).

* the gap table of precompute_gap_table (transform.cpp:221-237, decay_factor
  :60-68) against the reference library's own table;
* the device counter RNG (fgt_uniform_points_device) against the pinned
  values of proj/tests/test_rng.cpp:10-25 and, bit for bit, the reference's
  rng::uniform_points (rng.cpp:7-29);
* the device stable sort (fgt_sort_device) against a stable argsort
  (sort_with_perm, transform.cpp:27-39).
"""
import ctypes

import numpy as np
import pytest

import oracle
import paper_1909_09825_b200 as fgt
from paper_1909_09825_b200 import _capi
from paper_1909_09825_b200.transform import uniform_points_array as up

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    return torch


def need_ref():
    if not oracle.ref_available():
        pytest.fail("oracle/_ref/libfgt1d_ref.so missing (built by __graft_entry__.build())")


# ----------------------------------------------------------------- gap table

GAP_CASES = [
    # name, targets, delta, ne
    ("uniform400", np.sort(up(400, 5, 0)), 0.8, 5),
    ("ties_and_dups", np.sort(np.concatenate([up(300, 6, 3), up(300, 6, 3)[:50],
                                              np.zeros(20), np.ones(7)])), 1e-2, 6),
    ("flush_to_zero", np.array([0.0, 1e-9, 0.3, 0.3, 0.9, 5.0, 5.0 + 1e-12, 80.0]), 1e-6, 6),
    ("small_delta", np.sort(up(5000, 7, 3)), 1e-7, 3),
    ("large_delta", np.sort(up(5000, 8, 3)), 1e3, 4),
    ("unsorted_input", up(3000, 9, 3), 1e-3, 6),
]


@pytest.mark.parametrize("name,x,delta,ne", GAP_CASES, ids=[c[0] for c in GAP_CASES])
def test_gap_table_matches_reference(name, x, delta, ne):
    need_ref()
    soe = fgt.fold(fgt.cf_soe(2 * ne))
    p = fgt.plan(fgt.TransformRequest(x, x, np.ones(x.size), delta), soe, True)
    got = np.asarray(p.gap_exponentials)
    ref = oracle.ref_gap_table(x, delta, ne)
    assert got.shape == ref.shape == (ne * (x.size - 1),)
    # exp and sincos on the device vs glibc cexp: a few ulp of |g| <= 1
    assert np.max(np.abs(got - ref)) <= 4.5e-16, np.max(np.abs(got - ref))
    assert np.all(np.abs(got) <= 1.0)
    # the exact values: 1 at a zero gap, 0 past the underflow exponent
    assert np.array_equal(got[ref == 1.0], ref[ref == 1.0])
    assert np.array_equal(got[ref == 0.0], ref[ref == 0.0])


# ----------------------------------------------------------------------- RNG

PINS = [  # proj/tests/test_rng.cpp:10-25
    (0, 0, 0, 0xa706dd2f4d197e6f, 0.65244848637403219),
    (0, 0, 1, 0xb382a305f4414f5e, 0.70121210952152524),
    (42, 1, 7, 0x8d3b7fd7abb430ae, 0.55168913855932611),
    (123456789, 3, 1000000, 0x2ca992c901c93ced, 0.17446248443028345),
]


def device_uniform(torch, count, seed, stream, offset=0):
    out = torch.empty(count, dtype=torch.float64, device="cuda")
    _capi.check(_capi.lib().fgt_uniform_points_device(ctypes.c_void_p(out.data_ptr()), count, seed,
                                                      stream, offset, None))
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("seed,stream,i,bits,value", PINS)
def test_device_rng_pins(torch_cuda, seed, stream, i, bits, value):
    v = device_uniform(torch_cuda, 1, seed, stream, offset=i)[0]
    assert v == (bits >> 11) * 2.0 ** -53
    assert abs(v - value) <= 1e-16 * value


@pytest.mark.parametrize("seed,stream", [(0, 0), (0, 1), (0, 3), (7, 9), (2 ** 40 + 3, 5)])
def test_device_rng_bit_identical_to_reference(torch_cuda, seed, stream):
    need_ref()
    n = 1_000_003
    got = device_uniform(torch_cuda, n, seed, stream)
    ref = oracle.ref_uniform_points(n, seed, stream)
    assert np.array_equal(got, ref)
    assert np.array_equal(got, up(n, seed, stream))  # host generator too
    tail = device_uniform(torch_cuda, 1000, seed, stream, offset=n - 1000)
    assert np.array_equal(tail, ref[-1000:])
    assert got.min() >= 0.0 and got.max() < 1.0


# ---------------------------------------------------------------------- sort

def device_sort(torch, v):
    d = torch.as_tensor(np.asarray(v, dtype=np.float64), device="cuda")
    out = torch.empty_like(d)
    perm = torch.empty(d.numel(), dtype=torch.int32, device="cuda")
    _capi.check(_capi.lib().fgt_sort_device(ctypes.c_void_p(d.data_ptr()), d.numel(),
                                            ctypes.c_void_p(out.data_ptr()),
                                            ctypes.c_void_p(perm.data_ptr()), None))
    torch.cuda.synchronize()
    return out.cpu().numpy(), perm.cpu().numpy().astype(np.int64)


SORT_CASES = {
    "one": np.array([0.25]),
    "ties": np.repeat(up(1000, 21, 0), 3),
    "signed_zero": np.array([0.0, -0.0, 1.0, -0.0, 0.0, -1.0, 0.0] * 50),
    "negative_and_huge": np.concatenate([-up(5000, 22, 0) * 1e300, up(5000, 22, 1), [-5e-324, 5e-324]]),
    "presorted": np.sort(up(200_000, 23, 0)),
    "reversed": np.sort(up(200_000, 24, 0))[::-1].copy(),
    "bench_size": up(3_000_000, 0, 3),
}


@pytest.mark.parametrize("name", list(SORT_CASES))
def test_device_sort_stable_permutation(torch_cuda, name):
    v = SORT_CASES[name]
    s, p = device_sort(torch_cuda, v)
    ref_p = np.argsort(v, kind="stable")
    assert np.array_equal(s, v[p])
    # -0.0 and +0.0 compare equal (std::sort on pair<double, int64>): the
    # permutation is the stable one of that order
    assert np.array_equal(p, ref_p)
    assert np.all(s[1:] >= s[:-1])


def test_device_sort_matches_reference_plan_order():
    need_ref()
    v = np.concatenate([up(50_000, 25, 3), up(50_000, 25, 3)[:7000]])
    sx, tp, sy, sp, same = oracle.ref_plan(v, v, np.ones(v.size), 1.0)
    torch = pytest.importorskip("torch")
    s, p = device_sort(torch, v)
    assert np.array_equal(p, tp) and np.array_equal(s, sx)
