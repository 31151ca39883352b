"""CPU tests: pin the oracle (C restatement) before trusting it.

- against the reference's own golden potentials (proj/tests/test_transform.cpp:19-26),
- against the committed fixtures generated from the reference library
  (tests/golden/reference_cases.json, tests/golden/make_golden.py),
- bit-for-bit against the reference library itself when oracle/_ref was built.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1909_09825_b200.transform import counter_rand, uniform_points_array as up

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD_X = [0.0, 0.5, 1.0]
GOLD_Y = [0.0, 0.1, 0.35, 0.5, 0.75, 1.0]
GOLD_A = [0.5, -0.25, 1.0, 0.8, -0.6, 0.9]
GOLD_U = [0.53026354628615822, 1.3078174711896560, 0.66552744606900788]


def cases():
    with open(os.path.join(HERE, "golden", "reference_cases.json")) as f:
        return json.load(f)["cases"]


def test_direct_matches_50_digit_reference():
    # test_transform.cpp:60-66: epsilon 1e-15 relative
    u = oracle.direct(GOLD_X, GOLD_Y, GOLD_A, 0.02)
    assert np.allclose(u, GOLD_U, rtol=1e-15, atol=0)


def test_fast_transform_within_soe_accuracy():
    # test_transform.cpp:68-76: folded cf12, |u - gold| < 5e-9
    u = oracle.transform(GOLD_X, GOLD_Y, GOLD_A, 0.02, ne=6)
    assert np.max(np.abs(u - GOLD_U)) < 5e-9


@pytest.mark.parametrize("c", cases(), ids=lambda c: c["name"])
def test_oracle_reproduces_reference_fixtures(c):
    u = oracle.transform(c["targets"], c["sources"], c["strengths"], c["delta"], ne=c["ne"],
                         mode=c["mode"])
    # the restatement is operation-for-operation: bit identical
    assert np.array_equal(u, np.asarray(c["potentials"]))
    if c["direct"] is not None:
        d = oracle.direct(c["targets"], c["sources"], c["strengths"], c["delta"])
        assert np.array_equal(d, np.asarray(c["direct"]))


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed,n,m,delta,ne,sort", [
    (1, 5000, 7000, 1e-2, 6, True), (2, 20000, 20000, 1e-4, 4, False),
    (3, 3000, 100, 1.0, 3, False), (4, 100, 3000, 1e-6, 7, True)])
def test_oracle_bit_identical_to_reference_library(seed, n, m, delta, ne, sort):
    x, y = up(n, seed, 3), up(m, seed, 0)
    if sort:
        x, y = np.sort(x), np.sort(y)
    a = 2.0 * up(m, seed, 1) - 1.0
    u_ref, _ = oracle.ref_transform(x, y, a, delta, ne=ne, mode=0, threads=3)
    u = oracle.transform(x, y, a, delta, ne=ne, mode=0, threads=2)
    assert np.array_equal(u, u_ref)


def test_stable_sort_permutation():
    # test_transform.cpp:297-310
    _, p = oracle.sort_with_perm([0.5, 0.2, 0.5, 0.2])
    assert p.tolist() == [1, 3, 0, 2]


def test_mode_sums_match_quadratic_definition():
    # test_transform.cpp:216-244 (cf8, same points, delta 0.6)
    y = up(120, 21, 0)
    a = 2.0 * up(120, 21, 1) - 1.0
    hp, hm = oracle.mode_sums(y, y, a, 0.6, 4)
    t, _ = oracle.folded_table(8)
    ys, sp = oracle.sort_with_perm(y)
    rs = 1.0 / np.sqrt(0.6)
    bscale = np.sum(np.abs(a))
    for k in range(4):
        gap = ys[:, None] - ys[None, :]
        beta = a[sp][None, :]
        left = ys[None, :] <= ys[:, None]
        e = np.exp(-t[k] * gap * rs)
        ehp = np.sum(np.where(left, beta * e, 0), axis=1)
        ehm = np.sum(np.where(~left, beta * np.exp(t[k] * gap * rs), 0), axis=1)
        assert np.max(np.abs(hp[k] - ehp)) <= 1e-12 * bscale
        assert np.max(np.abs(hm[k] - ehm)) <= 1e-12 * bscale


def test_empty_inputs():
    # test_transform.cpp:121-140
    assert np.all(oracle.transform([0.1, 0.9], [], [], 1.0, ne=4) == 0.0)
    assert oracle.transform([], [0.5], [2.0], 1.0, ne=4).size == 0


def test_rng_pins():
    # proj/tests/test_rng.cpp:10-25
    assert int(counter_rand(0, 0, 0)) == 0xa706dd2f4d197e6f
    assert int(counter_rand(0, 0, 1)) == 0xb382a305f4414f5e
    assert int(counter_rand(42, 1, 7)) == 0x8d3b7fd7abb430ae
    assert int(counter_rand(123456789, 3, 1000000)) == 0x2ca992c901c93ced
    L = oracle.oracle_lib()
    assert L.oracle_counter_rand(42, 1, 7) == 0x8d3b7fd7abb430ae
    assert up(1, 0, 0)[0] == 0.65244848637403219
    assert abs(up(1, 123456789, 3, offset=1000000)[0] - 0.17446248443028345) < 1e-16


def test_gap_table_and_rng_restatements_match_reference():
    # precompute_gap_table (transform.cpp:221-237) and rng::uniform_points
    # (rng.cpp:7-29) of the C restatement, bit for bit against the reference
    if not oracle.ref_available():
        pytest.skip("reference library not built")
    from paper_1909_09825_b200.transform import uniform_points_array as up
    x = np.sort(np.concatenate([up(700, 31, 3), up(700, 31, 3)[:40], [5.0, 90.0]]))
    for delta, ne in ((0.8, 5), (1e-6, 6), (1e3, 3)):
        assert np.array_equal(oracle.gap_table(x, delta, ne), oracle.ref_gap_table(x, delta, ne))
    for seed, stream in ((0, 0), (42, 1), (123456789, 3)):
        assert np.array_equal(oracle.ref_uniform_points(10_000, seed, stream), up(10_000, seed, stream))
    assert oracle.ref_lib().fgt_ref_counter_rand(123456789, 3, 1000000) == 0x2ca992c901c93ced
