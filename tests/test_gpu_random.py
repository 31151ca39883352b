"""Randomised parity sweep of the device path against the oracle.

Seeded cases; each draws a point layout (uniform, clustered, integer grid,
heavy duplicates, wide range), ragged sizes (including empty sets and single
points), sorted or unsorted input, delta across twelve decades and n_e in 3..7.
Every case is small enough for the C oracle; the bar is the parity bar
|u_gpu - u_oracle| <= 1e-12 sum|alpha|.
"""
import numpy as np
import pytest

import oracle
import paper_1909_09825_b200 as fgt

pytestmark = pytest.mark.gpu

PARITY = 1e-12


def draw_points(rng, n, kind):
    if n == 0:
        return np.empty(0)
    if kind == "uniform":
        return rng.uniform(0.0, 1.0, n)
    if kind == "cluster":
        c = rng.uniform(-1.0, 1.0, 4)
        return c[rng.integers(0, 4, n)] + 10.0 ** rng.uniform(-6, -2) * rng.standard_normal(n)
    if kind == "grid":
        return rng.integers(-50, 50, n).astype(np.float64) * 0.01
    if kind == "dups":
        base = rng.uniform(0.0, 1.0, max(1, n // 20))
        return base[rng.integers(0, base.size, n)]
    if kind == "wide":
        return rng.uniform(-1e4, 1e4, n)
    raise ValueError(kind)


def one_case(seed):
    rng = np.random.default_rng(10_000 + seed)
    kinds = ["uniform", "cluster", "grid", "dups", "wide"]
    M = int(rng.choice([0, 1, 2, 7, 255, 256, 257, int(rng.integers(1, 6000))]))
    N = int(rng.choice([0, 1, 3, 255, 256, 513, int(rng.integers(1, 6000))]))
    x = draw_points(rng, M, kinds[rng.integers(0, len(kinds))])
    y = draw_points(rng, N, kinds[rng.integers(0, len(kinds))])
    if rng.random() < 0.5:
        x, y = np.sort(x), np.sort(y)
    a = rng.standard_normal(N)
    delta = float(10.0 ** rng.uniform(-8, 4))
    ne = int(rng.integers(3, 8))
    return x, y, a, delta, ne


@pytest.mark.parametrize("block", range(16))
def test_random_cases_vs_oracle(block):
    worst = 0.0
    for seed in range(block * 40, block * 40 + 40):
        x, y, a, delta, ne = one_case(seed)
        u = np.asarray(fgt.gauss_transform(x, y, a, delta, ne=ne))
        ref = oracle.transform(x, y, a, delta, ne=ne, mode=0)
        assert u.shape == ref.shape, seed
        if u.size == 0:
            continue
        scale = max(np.sum(np.abs(a)), 1e-300)
        err = np.max(np.abs(u - ref)) / scale
        worst = max(worst, err)
        assert err <= PARITY, (seed, err, x.size, y.size, delta, ne)


@pytest.mark.parametrize("seed", range(6))
def test_random_same_points_vs_oracle(seed):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(1, 5000))
    y = draw_points(rng, n, ["uniform", "cluster", "grid", "dups", "wide"][seed % 5])
    a = rng.standard_normal(n)
    delta = float(10.0 ** rng.uniform(-8, 3))
    ne = int(rng.integers(3, 8))
    soe = fgt.fold(fgt.cf_soe(2 * ne))
    p = fgt.plan(fgt.TransformRequest(y, y, a, delta), soe)
    assert p.same_points
    u = fgt.apply_same(p, a)
    ref = oracle.transform(y, y, a, delta, ne=ne, mode=1)
    assert np.max(np.abs(u - ref)) <= PARITY * np.sum(np.abs(a))


def test_random_batches_vs_oracle():
    rng = np.random.default_rng(77)
    B = 40
    xs, ys, al, deltas = [], [], [], []
    for b in range(B):
        m, n = int(rng.integers(0, 3000)), int(rng.integers(0, 3000))
        kind = ["uniform", "cluster", "grid", "dups", "wide"][b % 5]
        xs.append(np.sort(draw_points(rng, m, kind)))
        ys.append(np.sort(draw_points(rng, n, kind)))
        al.append(rng.standard_normal(n))
        deltas.append(float(10.0 ** rng.uniform(-8, 2)))
    soe = fgt.soe_for_tolerance(1e-10)
    out = fgt.batch_transform(xs, ys, al, deltas, soe)
    for b in range(B):
        if xs[b].size == 0:
            assert out[b].size == 0
            continue
        ref = oracle.transform(xs[b], ys[b], al[b], deltas[b], ne=len(soe), mode=0)
        scale = max(np.sum(np.abs(al[b])), 1e-300)
        assert np.max(np.abs(out[b] - ref)) <= PARITY * scale, b
