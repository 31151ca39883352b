"""GPU parity tests: the CUDA path (through the C ABI) against the oracle.

Bar (BASELINE.json north_star): |u_gpu - u_ref| <= 1e-12 * sum|alpha| over all
targets, against the reference's own outputs (committed fixtures from the
reference library) and the C oracle (bit-identical restatement of the
reference) on seeded inputs; within the SOE tolerance of the direct sum.
"""
import ctypes
import json
import os

import numpy as np
import pytest

import oracle
import paper_1909_09825_b200 as fgt
from paper_1909_09825_b200 import _capi
from paper_1909_09825_b200.transform import uniform_points_array as up

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
PARITY = 1e-12  # x sum|alpha|
PD = ctypes.POINTER(ctypes.c_double)


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if _capi.lib().fgt_device_count() < 1:
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")


def cases():
    with open(os.path.join(HERE, "golden", "reference_cases.json")) as f:
        return json.load(f)["cases"]


def gpu_transform(x, y, a, delta, ne, mode=2, soe=None):
    soe = soe if soe is not None else fgt.fold(fgt.cf_soe(2 * ne))
    p = fgt.plan(fgt.TransformRequest(x, y, a, delta), soe)
    if mode == 1 or (mode == 2 and p.same_points):
        return fgt.apply_same(p, a)
    return fgt.apply_general(p, a)


def check(u, ref, a, bar=PARITY):
    scale = max(np.sum(np.abs(a)), 1e-300)
    err = np.max(np.abs(np.asarray(u) - np.asarray(ref))) / scale if len(u) else 0.0
    assert err <= bar, err
    return err


# ---------------------------------------------------------------- fixtures

@pytest.mark.parametrize("c", cases(), ids=lambda c: c["name"])
def test_reference_fixtures(c):
    u = gpu_transform(c["targets"], c["sources"], c["strengths"], c["delta"], c["ne"], c["mode"])
    check(u, c["potentials"], c["strengths"])
    if c["direct"] is not None:
        d = fgt.direct(fgt.TransformRequest(c["targets"], c["sources"], c["strengths"], c["delta"]))
        ref = np.asarray(c["direct"])
        assert np.max(np.abs(d - ref)) <= 1e-14 * max(1.0, np.max(np.abs(ref)))


def test_golden_potentials():
    # test_transform.cpp:60-76, test_smoke.py:88-96
    gold = [0.53026354628615822, 1.3078174711896560, 0.66552744606900788]
    ys = [0.0, 0.1, 0.35, 0.5, 0.75, 1.0]
    al = [0.5, -0.25, 1.0, 0.8, -0.6, 0.9]
    got = fgt.gauss_transform([0.0, 0.5, 1.0], ys, al, 0.02, ne=6)
    assert max(abs(g - w) for g, w in zip(got, gold)) < 5e-9
    exact = fgt.direct_transform([0.0, 0.5, 1.0], ys, al, 0.02)
    assert max(abs(g - w) / abs(w) for g, w in zip(exact, gold)) < 1e-15


# ------------------------------------------------------------ seeded sweeps

SWEEP = [
    # seed, M, N, delta, ne, sorted
    (1, 1000, 1000, 1e-2, 6, True),
    (2, 100000, 100000, 1e-2, 6, True),    # cfg1 shape
    (3, 200000, 300000, 1e-3, 6, False),
    (4, 50000, 80000, 1e-4, 4, False),     # cfg2 parameters, smaller
    (5, 30000, 30000, 1e-6, 6, True),      # large gaps relative to sqrt(delta)
    (6, 30000, 10000, 1.0, 3, False),
    (7, 7, 100000, 1e-1, 5, False),        # few targets
    (8, 100000, 3, 1e-1, 5, False),        # few sources
    (9, 1, 1, 0.3, 6, True),
    (10, 5000, 5000, 1e-8, 7, False),      # everything decoupled
    (11, 65536, 65536, 1e-6, 6, True),     # cfg5 transform shape
    (12, 65536, 65536, 1e-1, 3, True),
    # wide segments in the collapsed-form range (full-width degree 7-8):
    # smax * 2h between rmax[6] and rmax[8]
    (13, 200000, 200000, 3e-3, 6, True),
    (14, 200000, 200000, 1e-2, 6, False),
    (15, 150000, 250000, 2e-2, 4, True),
]


@pytest.mark.parametrize("seed,M,N,delta,ne,srt", SWEEP)
def test_seeded_vs_oracle(seed, M, N, delta, ne, srt):
    x, y = up(M, seed, 3), up(N, seed, 0)
    if srt:
        x, y = np.sort(x), np.sort(y)
    a = 2.0 * up(N, seed, 1) - 1.0
    u = gpu_transform(x, y, a, delta, ne, mode=0)
    ref = oracle.transform(x, y, a, delta, ne=ne, mode=0)
    check(u, ref, a)


def test_clustered_mixture_vs_oracle():
    # cfg4 recipe at small scale: 16 centres, sigma 1e-3, unsorted, alpha in [0,1)
    rng = np.random.default_rng(0)
    c = up(16, 0, 5)
    x = c[rng.integers(0, 16, 40000)] + 1e-3 * rng.standard_normal(40000)
    y = c[rng.integers(0, 16, 160000)] + 1e-3 * rng.standard_normal(160000)
    a = up(160000, 0, 1)
    u = gpu_transform(x, y, a, 1e-6, 5, mode=0)
    check(u, oracle.transform(x, y, a, 1e-6, ne=5, mode=0), a)


def test_duplicates_and_signed_zero():
    rng = np.random.default_rng(1)
    x = np.round(rng.standard_normal(20000), 2)
    y = np.round(rng.standard_normal(30000), 2)
    x[:50] = -0.0
    y[:50] = 0.0
    y[50:100] = -0.0
    a = rng.standard_normal(30000)
    u = gpu_transform(x, y, a, 0.05, 6, mode=0)
    check(u, oracle.transform(x, y, a, 0.05, ne=6, mode=0), a)


def test_negative_and_wide_coordinates():
    rng = np.random.default_rng(2)
    x = rng.uniform(-1e3, 1e3, 30000)
    y = rng.uniform(-1e3, 1e3, 30000)
    a = rng.standard_normal(30000)
    for delta in (1e2, 1.0, 1e-4):
        u = gpu_transform(x, y, a, delta, 6, mode=0)
        check(u, oracle.transform(x, y, a, delta, ne=6, mode=0), a)


# ------------------------------------------------------- API semantics

def test_same_points_and_apply_same():
    # test_transform.cpp:89-106
    y = up(500, 11, 0)
    a = 2.0 * up(500, 11, 1) - 1.0
    soe = fgt.fold(fgt.cf_soe(10))
    p = fgt.plan(fgt.TransformRequest(y, y, a, 0.37), soe)
    assert p.same_points
    fast = fgt.apply_same(p, a)
    gen = fgt.apply_general(p, a)
    assert np.max(np.abs(fast - gen)) < 1e-13
    check(fast, oracle.transform(y, y, a, 0.37, ne=5, mode=1), a)
    # same set, other order is not same_points (test_transform.cpp:282-295)
    p2 = fgt.plan(fgt.TransformRequest([0.1, 0.5, 0.9], [0.9, 0.1, 0.5], [1.0, 1.0, 1.0], 1.0),
                  fgt.fold(fgt.cf_soe(8)))
    assert not p2.same_points
    with pytest.raises(ValueError):
        fgt.apply_same(p2, [1.0, 1.0, 1.0])


def test_plan_reuse_and_determinism():
    # test_transform.cpp:142-162, 184-200
    x, y = up(2000, 3, 3), up(3000, 3, 0)
    a = 2.0 * up(3000, 3, 1) - 1.0
    p = fgt.plan(fgt.TransformRequest(x, y, a, 2.0), fgt.fold(fgt.cf_soe(12)), True)
    r1 = fgt.apply_general(p, a)
    b2 = np.sin(0.1 * np.arange(1, 3001))
    r2 = fgt.apply_general(p, b2)
    check(r2, oracle.transform(x, y, b2, 2.0, ne=6, mode=0), b2)
    r1b = fgt.apply_general(p, a, 8)
    assert np.array_equal(r1, r1b)  # bit identical, thread count irrelevant
    for _ in range(3):
        assert np.array_equal(fgt.apply_general(p, a), r1)


def test_linearity_in_strengths():
    x, y = up(50000, 4, 3), up(60000, 4, 0)
    a1 = 2.0 * up(60000, 4, 1) - 1.0
    a2 = up(60000, 4, 6)
    p = fgt.plan(fgt.TransformRequest(x, y, a1, 1e-3), fgt.soe_for_tolerance(1e-10))
    u1, u2, u12 = (fgt.apply_general(p, v) for v in (a1, a2, a1 + a2))
    assert np.max(np.abs(u12 - u1 - u2)) <= 1e-13 * np.sum(np.abs(a1) + np.abs(a2))


def test_gap_table_api_parity():
    # test_transform.cpp:164-182
    y = up(400, 5, 0)
    a = 2.0 * up(400, 5, 1) - 1.0
    soe = fgt.fold(fgt.cf_soe(10))
    lazy = fgt.plan(fgt.TransformRequest(y, y, a, 0.8), soe, False)
    eager = fgt.plan(fgt.TransformRequest(y, y, a, 0.8), soe, True)
    assert not lazy.precomputed and eager.precomputed
    assert len(eager.gap_exponentials) == len(soe) * (400 - 1)
    assert all(abs(g) <= 1.0 for g in eager.gap_exponentials)
    assert np.array_equal(fgt.apply_same(lazy, a), fgt.apply_same(eager, a))
    # the table itself matches the reference library's decay factors
    # (transform.cpp:60-68, 221-237) to a few ulp of |g| <= 1
    if oracle.ref_available():
        ref = oracle.ref_gap_table(y, 0.8, len(soe))
    else:
        ref = oracle.gap_table(np.sort(y), 0.8, len(soe))
    got = np.asarray(eager.gap_exponentials)
    assert np.max(np.abs(got - ref)) <= 4.5e-16


def test_mode_sums_vs_quadratic_definition():
    # test_transform.cpp:216-244, acceptance.cpp:312-353
    for seed in range(3):
        n = 10 + int(up(1, 2000 + seed, 10)[0] * 190)
        y = up(n, 2000 + seed, 0)
        a = 2.0 * up(n, 2000 + seed, 1) - 1.0
        delta = 0.1 + up(2, 2000 + seed, 10)[1]
        soe = fgt.fold(fgt.cf_soe(8))
        p = fgt.plan(fgt.TransformRequest(y, y, a, delta), soe)
        hp, hm = fgt.mode_sums(p, a)
        ys, sp = p.sorted_sources, p.source_perm
        xs = p.sorted_targets
        rs = 1.0 / np.sqrt(delta)
        bscale = np.sum(np.abs(a))
        for k in range(len(soe)):
            t = soe.nodes[k]
            gap = xs[:, None] - ys[None, :]
            beta = a[sp][None, :]
            left = ys[None, :] <= xs[:, None]
            ehp = np.sum(np.where(left, beta * np.exp(-t * gap * rs), 0), axis=1)
            ehm = np.sum(np.where(~left, beta * np.exp(t * gap * rs), 0), axis=1)
            assert np.max(np.abs(hp[k] - ehp)) <= 1e-12 * bscale
            assert np.max(np.abs(hm[k] - ehm)) <= 1e-12 * bscale


@pytest.mark.parametrize("delta", [10.0, 1e-4])
def test_mode_sums_vs_oracle_narrow_and_wide(delta):
    # delta = 10: every segment takes the moment (narrow) path of K1 and K3;
    # delta = 1e-4: every segment the per-element (wide) path
    x, y = up(30000, 77, 3), up(40000, 77, 0)
    a = 2.0 * up(40000, 77, 1) - 1.0
    soe = fgt.fold(fgt.cf_soe(12))
    p = fgt.plan(fgt.TransformRequest(x, y, a, delta), soe)
    hp, hm = fgt.mode_sums(p, a)
    rp, rm = oracle.mode_sums(x, y, a, delta, 6)
    bar = 1e-12 * np.sum(np.abs(a))
    assert np.max(np.abs(hp - rp)) <= bar
    assert np.max(np.abs(hm - rm)) <= bar


def test_sorted_fields_and_stable_permutation():
    # test_transform.cpp:297-310
    p = fgt.plan(fgt.TransformRequest([0.5, 0.2, 0.5, 0.2], [0.4], [1.0], 1.0),
                 fgt.fold(fgt.cf_soe(8)))
    assert p.target_perm.tolist() == [1, 3, 0, 2]
    assert p.sorted_targets.tolist() == [0.2, 0.2, 0.5, 0.5]


@pytest.mark.parametrize("n", [1, 2, 1000, 2049, 123457, 3000000])
def test_radix_sort_is_stable_and_matches_reference_order(n):
    rng = np.random.default_rng(n)
    v = np.round(rng.standard_normal(n), 3)  # many ties
    if n > 10:
        v[::7] = -0.0
        v[3::11] = 0.0
    p = fgt.plan(fgt.TransformRequest(v, [], [], 1.0), fgt.fold(fgt.cf_soe(6)))
    s_ref, p_ref = oracle.sort_with_perm(v)
    assert np.array_equal(p.target_perm, p_ref)
    assert np.array_equal(p.sorted_targets, s_ref)


def test_empty_inputs():
    # test_transform.cpp:121-140
    soe = fgt.fold(fgt.cf_soe(8))
    p = fgt.plan(fgt.TransformRequest([0.1, 0.9], [], [], 1.0), soe)
    assert fgt.apply_general(p, []).tolist() == [0.0, 0.0]
    p2 = fgt.plan(fgt.TransformRequest([], [0.5], [2.0], 1.0), soe)
    assert fgt.apply_general(p2, [2.0]).size == 0
    assert fgt.direct(fgt.TransformRequest([0.1, 0.9], [], [], 1.0)).tolist() == [0.0, 0.0]


def test_validation_errors():
    soe = fgt.fold(fgt.cf_soe(8))
    req = fgt.TransformRequest([0.0, 0.5, 1.0], [0.0, 0.1], [1.0, 2.0], 0.02)
    p = fgt.plan(req, soe)
    with pytest.raises(ValueError):
        fgt.apply_general(p, [1.0])
    with pytest.raises(ValueError):
        fgt.apply_same(p, [1.0, 2.0])
    with pytest.raises(ValueError):
        fgt.direct(req, [3])
    with pytest.raises(ValueError):
        fgt.direct(req, [-1])
    # device-pointer plans check finiteness on the device
    import torch
    xd = torch.tensor([0.1, float("nan")], dtype=torch.float64, device="cuda")
    yd = torch.tensor([0.2], dtype=torch.float64, device="cuda")
    tr, ti, wr, wi, sc = soe.arrays()
    h = ctypes.c_void_p()
    rc = _capi.lib().fgt_plan_create(ctypes.cast(xd.data_ptr(), PD), 2, ctypes.cast(yd.data_ptr(), PD),
                                     1, 1.0, tr.ctypes.data_as(PD), ti.ctypes.data_as(PD),
                                     wr.ctypes.data_as(PD), wi.ctypes.data_as(PD),
                                     sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), len(soe), 1,
                                     _capi.FGT_DEVICE_PTRS, 0, None, ctypes.byref(h))
    assert rc == _capi.FGT_ERR_DOMAIN


def test_direct_subset_and_vs_oracle():
    # test_transform.cpp:78-87
    x, y = up(300, 1, 3), up(20000, 1, 0)
    a = 2.0 * up(20000, 1, 1) - 1.0
    req = fgt.TransformRequest(x, y, a, 1e-3)
    full = fgt.direct(req)
    sub = fgt.direct(req, [2, 0])
    assert sub[0] == full[2] and sub[1] == full[0]
    ref = oracle.direct(x, y, a, 1e-3)
    assert np.max(np.abs(full - ref)) <= 1e-15 * np.sum(np.abs(a))


@pytest.mark.parametrize("ne,bar", [(3, 4e-6 * 10), (4, 6e-8 * 10), (5, 6.4e-10 * 10),
                                    (6, 7.9e-12 * 10)])
def test_acceptance_window_vs_direct(ne, bar):
    # acceptance.cpp:185-267 criterion 7 (distinct points, delta = 1, bench_error)
    n = 100000
    y = up(n, 0, 0)
    x = up(n, 0, 3)
    a = up(n, 0, 1)
    u = gpu_transform(x, y, a, 1.0, ne, mode=0)
    idx = np.minimum(n - 1, (up(100, 0, 2) * n).astype(np.int64))
    d = fgt.direct(fgt.TransformRequest(x, y, a, 1.0), idx)
    umax = np.max(np.abs(d))
    keep = np.abs(d) >= 1e-3 * umax
    err = np.max(np.abs(u[idx][keep] - d[keep]) / np.abs(d[keep]))
    assert err <= bar


def test_chunked_two_phase_equals_single_plan():
    """Multi-GPU carry algebra on one GPU: split the merged stream into chunks,
    run each chunk's phase 1, exchange aggregates through fgt_chunk_carries,
    run phase 2; must match the single-plan result (no ranks waiting on each
    other: chunks run one after another)."""
    import bench
    M, N, delta, ne = 200000, 150000, 1e-3, 6
    x, y = np.sort(up(M, 9, 3)), np.sort(up(N, 9, 0))
    a = 2.0 * up(N, 9, 1) - 1.0
    soe = fgt.soe_for_tolerance(1e-10)
    tr, ti, wr, wi, sc = soe.arrays()
    sp = (tr.ctypes.data_as(PD), ti.ctypes.data_as(PD), wr.ctypes.data_as(PD),
          wi.ctypes.data_as(PD), sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), ne, 1)
    L = _capi.lib()
    full = gpu_transform(x, y, a, delta, ne, mode=0, soe=soe)
    for G in (2, 3, 8):
        tot = M + N
        bounds = [(bench.merge_split(x, y, tot * g // G), tot * g // G) for g in range(G + 1)]
        plans, aggs = [], []
        for g in range(G):
            (i0, d0), (i1, d1) = bounds[g], bounds[g + 1]
            j0, j1 = d0 - i0, d1 - i1
            xc, yc, ac = x[i0:i1].copy(), y[j0:j1].copy(), a[j0:j1].copy()
            zp = max(x[i0 - 1] if i0 > 0 else -np.inf, y[j0 - 1] if j0 > 0 else -np.inf)
            h = ctypes.c_void_p()
            _capi.check(L.fgt_plan_create_chunk(xc.ctypes.data_as(PD), xc.size, yc.ctypes.data_as(PD),
                                                yc.size, float(zp) if d0 > 0 else 0.0, int(d0 > 0),
                                                delta, *sp, 0, -1, None, ctypes.byref(h)))
            agg = np.empty(6 * ne)
            _capi.check(L.fgt_apply_chunk_aggregate(h, ac.ctypes.data_as(PD), agg.ctypes.data_as(PD),
                                                    0, None))
            plans.append((h, xc, ac, i0))
            aggs.append(agg)
        allagg = np.concatenate(aggs)
        car = np.empty(G * 4 * ne)
        _capi.check(L.fgt_chunk_carries(allagg.ctypes.data_as(PD), G, ne, car.ctypes.data_as(PD)))
        u = np.empty(M)
        for g, (h, xc, ac, i0) in enumerate(plans):
            mine = np.ascontiguousarray(car[g * 4 * ne:(g + 1) * 4 * ne])
            out = np.empty(max(xc.size, 1))
            _capi.check(L.fgt_apply_chunk_finish(h, ac.ctypes.data_as(PD), mine.ctypes.data_as(PD),
                                                 out.ctypes.data_as(PD), 0, None))
            u[i0:i0 + xc.size] = out[:xc.size]
            L.fgt_plan_destroy(h)
        check(u, full, a, 1e-13)


def test_chunked_device_exchange_equals_single_plan():
    """The multi-GPU path with no host round trip (FGT_DEVICE_AGGS): chunk
    aggregates land in one device array (the all_gather's output), each
    chunk's carries come from fgt_chunk_carries_device, phase 2 reads them on
    the device; same bar as the host exchange, and the device carries equal
    the host algebra's."""
    import torch
    import bench
    M, N, delta, ne = 180000, 220000, 1e-4, 6
    x, y = np.sort(up(M, 12, 3)), np.sort(up(N, 12, 0))
    a = 2.0 * up(N, 12, 1) - 1.0
    soe = fgt.soe_for_tolerance(1e-10)
    tr, ti, wr, wi, sc = soe.arrays()
    sp = (tr.ctypes.data_as(PD), ti.ctypes.data_as(PD), wr.ctypes.data_as(PD),
          wi.ctypes.data_as(PD), sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), ne, 1)
    L = _capi.lib()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    sh = ctypes.c_void_p(st.cuda_stream)
    full = gpu_transform(x, y, a, delta, ne, mode=0, soe=soe)
    dx, dy, da = (torch.from_numpy(v).to(dev) for v in (x, y, a))
    fl = _capi.FGT_DEVICE_PTRS | _capi.FGT_BORROW | _capi.FGT_DEVICE_AGGS
    for G in (1, 2, 5, 8):
        tot = M + N
        bounds = [(bench.merge_split(x, y, tot * g // G), tot * g // G) for g in range(G + 1)]
        aggs = torch.empty(G * 6 * ne, dtype=torch.float64, device=dev)
        u = torch.zeros(M, dtype=torch.float64, device=dev)
        plans = []
        for g in range(G):
            (i0, d0), (i1, d1) = bounds[g], bounds[g + 1]
            j0, j1 = d0 - i0, d1 - i1
            zp = max(x[i0 - 1] if i0 > 0 else -np.inf, y[j0 - 1] if j0 > 0 else -np.inf)
            h = ctypes.c_void_p()
            _capi.check(L.fgt_plan_create_chunk(ctypes.cast(dx[i0:].data_ptr(), PD), i1 - i0,
                                                ctypes.cast(dy[j0:].data_ptr(), PD), j1 - j0,
                                                float(zp) if d0 > 0 else 0.0, int(d0 > 0), delta,
                                                *sp, fl, 0, sh, ctypes.byref(h)))
            _capi.check(L.fgt_apply_chunk_aggregate(
                h, ctypes.cast(da[j0:].data_ptr(), PD),
                ctypes.cast(aggs[g * 6 * ne:].data_ptr(), PD), fl, sh))
            plans.append((h, i0, j0))
        host_car = np.empty(G * 4 * ne)
        agg_h = aggs.cpu().numpy()
        _capi.check(L.fgt_chunk_carries(agg_h.ctypes.data_as(PD), G, ne,
                                        host_car.ctypes.data_as(PD)))
        car = torch.empty(4 * ne, dtype=torch.float64, device=dev)
        for g, (h, i0, j0) in enumerate(plans):
            _capi.check(L.fgt_chunk_carries_device(ctypes.c_void_p(aggs.data_ptr()), G, ne, g,
                                                   ctypes.c_void_p(car.data_ptr()), sh))
            assert np.allclose(car.cpu().numpy(), host_car[g * 4 * ne:(g + 1) * 4 * ne],
                               rtol=1e-15, atol=1e-300)
            _capi.check(L.fgt_apply_chunk_finish(h, ctypes.cast(da[j0:].data_ptr(), PD),
                                                 ctypes.cast(car.data_ptr(), PD),
                                                 ctypes.cast(u[i0:].data_ptr(), PD), fl, sh))
        torch.cuda.synchronize()
        for h, _, _ in plans:
            L.fgt_plan_destroy(h)
        check(u.cpu().numpy(), full, a, 1e-13)


def test_device_pointer_path_matches_host_path():
    import torch
    M, N = 300000, 250000
    x, y = np.sort(up(M, 12, 3)), np.sort(up(N, 12, 0))
    a = 2.0 * up(N, 12, 1) - 1.0
    host = gpu_transform(x, y, a, 1e-3, 6, mode=0)
    soe = fgt.fold(fgt.cf_soe(12))
    tr, ti, wr, wi, sc = soe.arrays()
    xd, yd, ad = (torch.from_numpy(v).cuda() for v in (x, y, a))
    ud = torch.empty(M, dtype=torch.float64, device="cuda")
    L = _capi.lib()
    h = ctypes.c_void_p()
    fl = _capi.FGT_DEVICE_PTRS | _capi.FGT_BORROW
    _capi.check(L.fgt_plan_create(ctypes.cast(xd.data_ptr(), PD), M, ctypes.cast(yd.data_ptr(), PD), N,
                                  1e-3, tr.ctypes.data_as(PD), ti.ctypes.data_as(PD),
                                  wr.ctypes.data_as(PD), wi.ctypes.data_as(PD),
                                  sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), 6, 1, fl, 0,
                                  None, ctypes.byref(h)))
    _capi.check(L.fgt_apply_general(h, ctypes.cast(ad.data_ptr(), PD), N,
                                    ctypes.cast(ud.data_ptr(), PD), 1, fl, None))
    torch.cuda.synchronize()
    L.fgt_plan_destroy(h)
    assert np.array_equal(ud.cpu().numpy(), host)


@pytest.mark.parametrize("ox,oy", [(1, 0), (0, 1), (1, 1), (3, 2)])
def test_device_pointers_not_16_byte_aligned(ox, oy):
    # borrowed device arrays at odd element offsets: the plan's bulk staging
    # must handle 8-byte aligned starts and ends (head / tail elements)
    import torch
    M, N = 70001, 50003
    x, y = np.sort(up(M, 13, 3)), np.sort(up(N, 13, 0))
    a = 2.0 * up(N, 13, 1) - 1.0
    host = gpu_transform(x, y, a, 1e-3, 6, mode=0)
    soe = fgt.fold(fgt.cf_soe(12))
    tr, ti, wr, wi, sc = soe.arrays()
    xb = torch.zeros(M + 8, dtype=torch.float64, device="cuda")
    yb = torch.zeros(N + 8, dtype=torch.float64, device="cuda")
    xb[ox:ox + M] = torch.from_numpy(x).cuda()
    yb[oy:oy + N] = torch.from_numpy(y).cuda()
    xd, yd = xb[ox:ox + M], yb[oy:oy + N]
    ad = torch.from_numpy(a).cuda()
    ud = torch.empty(M, dtype=torch.float64, device="cuda")
    L = _capi.lib()
    h = ctypes.c_void_p()
    fl = _capi.FGT_DEVICE_PTRS | _capi.FGT_BORROW
    _capi.check(L.fgt_plan_create(ctypes.cast(xd.data_ptr(), PD), M, ctypes.cast(yd.data_ptr(), PD), N,
                                  1e-3, tr.ctypes.data_as(PD), ti.ctypes.data_as(PD),
                                  wr.ctypes.data_as(PD), wi.ctypes.data_as(PD),
                                  sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), 6, 1, fl, 0,
                                  None, ctypes.byref(h)))
    _capi.check(L.fgt_apply_general(h, ctypes.cast(ad.data_ptr(), PD), N,
                                    ctypes.cast(ud.data_ptr(), PD), 1, fl, None))
    torch.cuda.synchronize()
    L.fgt_plan_destroy(h)
    assert np.array_equal(ud.cpu().numpy(), host)


def test_gauss_transform_accepts_device_arrays():
    # pymodule.cpp:37-60 entry with CUDA tensors in and out
    import torch
    x, y = up(40000, 31, 3), up(30000, 31, 0)
    a = 2.0 * up(30000, 31, 1) - 1.0
    host = np.array(fgt.gauss_transform(x, y, a, 1e-3, ne=6))
    ud = fgt.gauss_transform(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(),
                             torch.from_numpy(a).cuda(), 1e-3, ne=6)
    assert ud.is_cuda and ud.dtype == torch.float64
    assert np.array_equal(ud.cpu().numpy(), host)
    # same points on the device take apply_same, like the host entry
    yd = torch.from_numpy(y).cuda()
    us = fgt.gauss_transform(yd, yd, torch.from_numpy(a).cuda(), 1e-3, ne=6)
    assert np.array_equal(us.cpu().numpy(), np.array(fgt.gauss_transform(y, y, a, 1e-3, ne=6)))
    with pytest.raises(ValueError):
        fgt.gauss_transform(yd, yd, yd[:5], 1e-3)


def test_gpu_kernels_actually_launch():
    L = _capi.lib()
    before = L.fgt_launch_counter()
    fgt.gauss_transform(up(1000, 1, 3), up(1000, 1, 0), up(1000, 1, 1), 0.1, ne=4)
    assert L.fgt_launch_counter() - before >= 3


# ------------------------------------------------------- batched transforms

def test_batched_transforms_vs_oracle():
    """BASELINE cfg 5 shape (scaled down): independent presorted transforms
    with per-transform delta (log-uniform in [1e-6, 1e-1]) in one plan;
    ragged sizes including empty sets."""
    rng = np.random.default_rng(5)
    B = 48
    sizes = [(int(m), int(n)) for m, n in rng.integers(0, 3000, size=(B, 2))]
    sizes[3] = (0, 500)
    sizes[7] = (400, 0)
    sizes[11] = (1, 1)
    sizes[19] = (5000, 4100)
    xs = [np.sort(up(m, 100 + b, 3)) for b, (m, n) in enumerate(sizes)]
    ys = [np.sort(up(n, 100 + b, 0)) for b, (m, n) in enumerate(sizes)]
    al = [2.0 * up(n, 100 + b, 1) - 1.0 for b, (m, n) in enumerate(sizes)]
    deltas = 10.0 ** (-6.0 + 5.0 * up(B, 0, 9))
    for ne in (3, 4, 6):
        soe = fgt.fold(fgt.cf_soe(2 * ne))
        out = fgt.batch_transform(xs, ys, al, deltas, soe)
        for b in range(B):
            ref = oracle.transform(xs[b], ys[b], al[b], deltas[b], ne=ne, mode=0)
            assert out[b].size == ref.size
            if ref.size:
                check(out[b], ref, al[b] if al[b].size else [1.0])


def test_batched_mixed_segment_classes():
    # transforms large enough that narrow (moment) and wide (per-element)
    # segments of K1 and K3 meet in one batched plan
    deltas = [10.0, 1.0, 0.1, 1e-3, 1e-5, 1e-7]
    n = 60000
    xs = [np.sort(up(n, 300 + b, 3)) for b in range(len(deltas))]
    ys = [np.sort(up(n, 300 + b, 0)) for b in range(len(deltas))]
    al = [2.0 * up(n, 300 + b, 1) - 1.0 for b in range(len(deltas))]
    soe = fgt.soe_for_tolerance(1e-10)
    out = fgt.batch_transform(xs, ys, al, deltas, soe)
    for b, d in enumerate(deltas):
        check(out[b], oracle.transform(xs[b], ys[b], al[b], d, ne=len(soe), mode=0), al[b])


@pytest.mark.parametrize("nmodes", [1, 2, 5, 7, 8])
def test_custom_mode_counts_all_segment_classes(nmodes):
    """Folded SOEs with 1..8 modes (kMaxModes = 8; the presets have 3..7): every
    instantiated mode count of the lane-collapsed wide kernels, on deltas that
    put segments in the narrow (moment), lane-collapsed and per-mode classes,
    as single plans and as one batched plan.  The modes are the folded modes of
    the n = 14 and n = 12 tables (no longer a Gaussian approximation: parity
    with the oracle on the same modes is the bar)."""
    t7, w7 = oracle.folded_table(14)
    t6, w6 = oracle.folded_table(12)
    t = np.concatenate([t7, t6[:1]])[:nmodes]
    mw = np.concatenate([w7, w6[:1]])[:nmodes]
    # mw carries the fold multiplier 2 of a conjugate pair (halving is exact)
    soe = fgt.SoeApprox(list(t), list(0.5 * mw), fgt.SoeForm.FOLDED, [0] * nmodes)
    n = 20000
    deltas = [1.0, 1e-3, 1e-5, 3e-7, 1e-9, 1e-12]
    xs = [np.sort(up(n, 700 + b, 3)) for b in range(len(deltas))]
    ys = [np.sort(up(n + 37, 700 + b, 0)) for b in range(len(deltas))]
    al = [2.0 * up(n + 37, 700 + b, 1) - 1.0 for b in range(len(deltas))]
    refs = [oracle.transform(xs[b], ys[b], al[b], d, mode=0, soe=(t, mw))
            for b, d in enumerate(deltas)]
    for b, d in enumerate(deltas):
        check(gpu_transform(xs[b], ys[b], al[b], d, None, mode=0, soe=soe), refs[b], al[b])
    out = fgt.batch_transform(xs, ys, al, deltas, soe)
    for b in range(len(deltas)):
        check(out[b], refs[b], al[b])


def test_batched_rejects_unsorted_and_reuses_plan():
    soe = fgt.fold(fgt.cf_soe(8))
    with pytest.raises(ValueError):
        fgt.batch_transform([np.array([0.5, 0.1])], [np.array([0.2])], [np.array([1.0])], [0.1], soe)
    xs = [np.sort(up(1000, 7, 3)), np.sort(up(700, 8, 3))]
    ys = [np.sort(up(900, 7, 0)), np.sort(up(1200, 8, 0))]
    bp = fgt.BatchPlan(xs, ys, [1e-3, 1e-5], soe)
    for seed in (1, 2):
        al = [up(900, seed, 1), up(1200, seed, 6)]
        out = bp.apply(al)
        for b, d in enumerate([1e-3, 1e-5]):
            check(out[b], oracle.transform(xs[b], ys[b], al[b], d, ne=4, mode=0), al[b])


# ---------------------------------------------- error harness (§8f item 3)

def test_delta_sweep_acceptance_criterion10():
    # acceptance.cpp:394-423: N=1e5 same points, n_e=4, delta=1e-7..1e4; the
    # sampled error is nondecreasing within x3 and saturates near E_n
    rows = fgt.delta_sweep(100000, 4, [10.0 ** p for p in range(-7, 5)], seed=0)
    errs = [r["error"] for r in rows]
    en = fgt.max_error(fgt.fold(fgt.cf_soe(8))).max_abs_error
    for i in range(1, len(errs)):
        assert errs[i] >= errs[i - 1] / 3.0, errs
    sat = errs[-1]
    assert en / 10.0 <= sat <= 10.0 * en, (sat, en)
    assert sat >= max(errs) / 3.0


def test_measure_error_matches_reference_on_its_own_result():
    # fgt1d_cli.cpp:198-218 on the same request: our sampled error vs the one
    # the reference library's transform has (same SOE, same 100 targets)
    if not oracle.ref_available():
        pytest.skip("reference library not built")
    n = 20000
    y = up(n, 0, 0)
    a = up(n, 0, 1)
    for delta in (1e-6, 1e-4, 1e-2, 1.0):
        req = fgt.TransformRequest(y, y, a, delta)
        ours = fgt.measure_error(req, np.array(fgt.gauss_transform(y, y, a, delta, ne=6)), 0)
        ref_u, _ = oracle.ref_transform(y, y, a, delta, ne=6, mode=1)
        theirs = fgt.measure_error(req, ref_u, 0)
        assert ours <= max(1.1 * theirs, 1e-13), (delta, ours, theirs)


# --------------------------- plan tile checks: non-finite / nearly-sorted

def _plan_rc(x, y):
    import torch
    soe = fgt.fold(fgt.cf_soe(8))
    tr, ti, wr, wi, sc = soe.arrays()
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    yd = torch.from_numpy(np.ascontiguousarray(y)).cuda()
    h = ctypes.c_void_p()
    rc = _capi.lib().fgt_plan_create(ctypes.cast(xd.data_ptr(), PD), x.size,
                                     ctypes.cast(yd.data_ptr(), PD), y.size, 1e-3,
                                     tr.ctypes.data_as(PD), ti.ctypes.data_as(PD),
                                     wr.ctypes.data_as(PD), wi.ctypes.data_as(PD),
                                     sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), len(soe), 1,
                                     _capi.FGT_DEVICE_PTRS, 0, None, ctypes.byref(h))
    msg = _capi.lib().fgt_last_error().decode() if rc else ""
    if rc == 0:
        _capi.lib().fgt_plan_destroy(h)
    return rc, msg


@pytest.mark.parametrize("srt", [True, False])
def test_nonfinite_detected_anywhere(srt):
    # transform.cpp:21-25 check_points: every coordinate, targets before sources
    rng = np.random.default_rng(31)
    for trial in range(12):
        n, m = int(rng.integers(1, 20000)), int(rng.integers(1, 20000))
        x, y = up(n, trial, 3), up(m, trial, 0)
        if srt:
            x, y = np.sort(x), np.sort(y)
        bad = [np.nan, np.inf, -np.inf][trial % 3]
        which = trial % 2
        arr = x if which == 0 else y
        pos = [0, arr.size - 1, int(rng.integers(0, arr.size))][trial % 3]
        arr[pos] = bad
        rc, msg = _plan_rc(x, y)
        assert rc == _capi.FGT_ERR_DOMAIN, (trial, srt, which, pos, bad)
        assert ("target" if which == 0 else "source") in msg, msg


def test_nearly_sorted_inputs_are_sorted_first():
    # one adjacent swap at tile / segment boundaries must be detected
    n = 3 * 4096 + 77
    for pos in (0, 127, 255, 256, 2047, 2048, 4095, 4096, 8191, n - 2):
        x, y = np.sort(up(n, 40, 3)), np.sort(up(n, 40, 0))
        for arr in (x, y):
            a2 = arr.copy()
            a2[pos], a2[pos + 1] = a2[pos + 1], a2[pos]
            xx, yy = (a2, y) if arr is x else (x, a2)
            a = 2.0 * up(n, 40, 1) - 1.0
            u = gpu_transform(xx, yy, a, 1e-3, 6, mode=0)
            check(u, oracle.transform(xx, yy, a, 1e-3, ne=6, mode=0), a)
