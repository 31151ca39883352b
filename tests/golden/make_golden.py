#!/usr/bin/env python3
"""Generates tests/golden/*.json from the REFERENCE library itself
(oracle/_ref/libfgt1d_ref.so = /root/reference/proj/src/{transform,soe,rng}.cpp
compiled in place by oracle/build_ref.sh).  Run in the build container, where
/root/reference exists; the fixtures travel to the GPU box, the reference does
not.  Inputs are small and seeded (counter RNG) so the files stay small.

Each case: targets, sources, strengths, delta, n_e, the reference's
apply_general (or apply_same) potentials, and direct() potentials.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1909_09825_b200.transform import uniform_points_array as up  # noqa: E402


def case(name, x, y, a, delta, ne, mode=0):
    x, y, a = (np.asarray(v, dtype=np.float64) for v in (x, y, a))
    u, _ = oracle.ref_transform(x, y, a, delta, ne=ne, mode=mode, threads=1, precompute=True)
    d = oracle.ref_direct(x, y, a, delta) if x.size * max(y.size, 1) <= 4e7 else None
    return {"name": name, "targets": x.tolist(), "sources": y.tolist(), "strengths": a.tolist(),
            "delta": delta, "ne": ne, "mode": mode, "potentials": u.tolist(),
            "direct": None if d is None else d.tolist()}


def main():
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref/libfgt1d_ref.so missing: run oracle/build_ref.sh first")
    cases = []
    # proj/tests/test_transform.cpp:19-35 golden 6-source / 3-target case
    cases.append(case("golden_test_transform", [0.0, 0.5, 1.0],
                      [0.0, 0.1, 0.35, 0.5, 0.75, 1.0], [0.5, -0.25, 1.0, 0.8, -0.6, 0.9],
                      0.02, 6))
    # ties (test_transform.cpp:108-119)
    cases.append(case("ties", [0.3, 0.5, 0.7, 0.9, 0.3], [0.3, 0.3, 0.7, 0.7, 0.7],
                      [1.0, -2.0, 0.5, 0.5, 0.25], 0.05, 6))
    # widely separated clusters (test_transform.cpp:202-214)
    cases.append(case("underflow_clusters", [5e-4, 100.0005], [0.0, 1e-3, 100.0, 100.001],
                      [1.0, 2.0, -3.0, 4.0], 1e-8, 6))
    # same set, different order (test_transform.cpp:282-295)
    cases.append(case("same_set_other_order", [0.1, 0.5, 0.9], [0.9, 0.1, 0.5],
                      [1.0, 1.0, 1.0], 1.0, 4))
    # random_request(seed, n, m, delta) style (test_transform.cpp:37-48)
    for seed, n, m, delta, ne in [(3, 200, 300, 2.0, 6), (8, 700, 900, 0.25, 6),
                                  (11, 500, 500, 0.37, 5), (21, 120, 120, 0.6, 4),
                                  (5, 2000, 1500, 1e-3, 6), (9, 3000, 3000, 1e-5, 3),
                                  (13, 1000, 4000, 1e-2, 7)]:
        x = up(n, seed, 3)
        y = up(m, seed, 0)
        a = 2.0 * up(m, seed, 1) - 1.0
        cases.append(case(f"random_s{seed}_n{n}_m{m}_d{delta:g}_ne{ne}", x, y, a, delta, ne))
    # same points through apply_same (test_transform.cpp:89-106)
    y = up(500, 11, 0)
    a = 2.0 * up(500, 11, 1) - 1.0
    cases.append(case("same_points_apply_same", y, y, a, 0.37, 5, mode=1))
    # clustered (cfg4-like) small: 4-component mixture, sigma 1e-3
    rng = np.random.default_rng(4)
    cen = up(4, 0, 5)
    xs = cen[rng.integers(0, 4, 800)] + 1e-3 * rng.standard_normal(800)
    ys = cen[rng.integers(0, 4, 2400)] + 1e-3 * rng.standard_normal(2400)
    cases.append(case("clustered_mixture", xs, ys, rng.random(2400), 1e-6, 5))
    with open(os.path.join(HERE, "reference_cases.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py via oracle/_ref (reference library)",
                   "cases": cases}, f)
    # counter RNG pins straight from the reference's own test (test_rng.cpp:10-25)
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    main()
