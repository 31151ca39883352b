"""CPU tests of the SOE table data and host-side SOE logic.

The compiled-in CF tables (tools/gen_soe_tables.py, a numpy restatement of
proj/src/cf.cpp) are pinned against the reference's frozen grid errors
(proj/tests/test_cf.cpp:20-23, 5% window), the argmax-at-origin property
(:33-36), the cf8 window of the Python smoke test (test_smoke.py:23), and the
printed n=5 row of proj/README.md:141.
"""
import io
import math
import os

import numpy as np
import pytest

import oracle
import paper_1909_09825_b200 as fgt
from paper_1909_09825_b200 import soe as S

PINS = {2: 1.2476e-1, 4: 3.5683e-3, 6: 7.2279e-5, 8: 1.2570e-6, 10: 2.0042e-8,
        12: 3.0208e-10, 14: 4.4564e-12}


def grid_error(soe):
    i = np.arange(1, 100001)
    xs = np.concatenate([[0.0], 10.0 ** (-5.0 + 7.0 * (i - 1) / 99999.0)])
    acc = np.zeros(xs.shape, complex)
    for k in range(len(soe)):
        t, w = soe.nodes[k], soe.weights[k]
        m = t.real * xs <= 745.0
        acc[m] += soe.multiplier(k) * w * np.exp(-t * xs[m])
    err = np.abs(np.exp(-xs * xs / 4.0) - acc.real)
    j = int(np.argmax(err))
    return err[j], xs[j]


@pytest.mark.parametrize("n", sorted(PINS))
def test_cf_table_errors_match_frozen_values(n):
    e, x = grid_error(fgt.cf_soe(n))
    assert abs(e - PINS[n]) <= 0.05 * PINS[n]
    if n <= 12:
        assert x == 0.0
    else:
        assert x <= 2e-5


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("n", [6, 8, 10, 12])
def test_cf_table_error_through_reference_max_error(n):
    # the reference's own max_error (soe.cpp:242-248) on our table
    e, x = oracle.ref_max_error(n)
    assert abs(e - PINS[n]) <= 0.05 * PINS[n] and x == 0.0


def test_cf8_window_of_python_smoke():
    e, x = grid_error(fgt.cf_soe(8))
    assert 1.19e-6 <= e <= 1.33e-6 and x == 0.0


def test_readme_n5_row():
    s = fgt.cf_soe(5)
    want = (1.4125273859597052, -1.7420506859336538, 5.5174094028788465e-02, 1.9821811587250646e-01)
    got = (s.nodes[0].real, s.nodes[0].imag, s.weights[0].real, s.weights[0].imag)
    for g, w in zip(got, want):
        assert abs(g - w) <= 1e-11 * abs(w)


def test_table_text_files_match_compiled_tables():
    data = os.path.join(os.path.dirname(fgt.__file__), "data")
    for n in range(2, 15):
        t = S.load_coefficient_table(os.path.join(data, f"cf_n{n}.soe"))
        c = fgt.cf_soe(n)
        assert t.nodes == c.nodes and t.weights == c.weights


def test_fold_matches_capi_fold_and_reference_structure():
    for n in range(2, 15):
        full = fgt.cf_soe(n)
        py = fgt.fold(full)
        capi = S._from_capi(n, True)
        assert py.nodes == capi.nodes and py.weights == capi.weights
        assert py.self_conjugate == capi.self_conjugate
        assert len(py) == (n + 1) // 2
        # odd n: exactly one self-conjugate node (test_cf.cpp:56-80)
        assert sum(py.self_conjugate) == n % 2
        back = fgt.unfold(py)
        assert len(back) == n
        for x in (0.0, 0.37, 2.5):
            assert math.isclose(fgt.evaluate(full, x, 1.0), fgt.evaluate(py, x, 1.0),
                                rel_tol=1e-12, abs_tol=1e-15)


def test_presets_and_tolerance_lookup():
    assert [fgt.preset_mode_count(p) for p in range(4)] == [3, 4, 5, 6]
    for p in range(4):
        s = fgt.preset_soe(p)
        assert s.form == fgt.SoeForm.FOLDED and len(s) == fgt.preset_mode_count(p)
    assert fgt.mode_count_for_tolerance(1e-3) == 3
    assert fgt.mode_count_for_tolerance(1e-6) == 4
    assert fgt.mode_count_for_tolerance(1e-8) == 5
    assert fgt.mode_count_for_tolerance(1e-10) == 6
    assert fgt.mode_count_for_tolerance(1e-11) == 7
    with pytest.raises(ValueError):
        fgt.mode_count_for_tolerance(1e-14)
    with pytest.raises(ValueError):
        fgt.preset_mode_count(9)
    with pytest.raises(ValueError):
        fgt.cf_soe(1)
    with pytest.raises(ValueError):
        fgt.cf_soe(15)


def test_coefficient_table_roundtrip_bit_exact(tmp_path):
    # test_smoke.py:99-107 / soe.hpp:98
    s = fgt.fold(fgt.cf_soe(7))
    p = str(tmp_path / "cf7.soe")
    fgt.save_coefficient_table(p, s)
    back = fgt.load_coefficient_table(p)
    assert back.form == s.form and back.nodes == s.nodes and back.weights == s.weights
    assert back.self_conjugate == s.self_conjugate


def test_table_reader_errors():
    for bad in ["", "xx n=1 form=full\n", "soe form=full\n", "soe n=1 form=weird\n",
                "soe n=2 form=full\n1 0 1 0\n", "soe n=1 form=folded\n1 -1 1 0\n",
                "soe n=1 form=full\n1 0 abc 0\n", "soe n=1 bogus\n1 0 1 0\n"]:
        with pytest.raises(ValueError):
            S.read_coefficient_table(io.StringIO(bad))


def test_validate_and_fold_errors():
    with pytest.raises(ValueError):
        S.validate(S.SoeApprox([1 + 1j], [1.0, 2.0]))
    with pytest.raises(ValueError):
        S.validate(S.SoeApprox([-1 + 0j], [1.0]))
    with pytest.raises(ValueError):
        fgt.fold(S.SoeApprox([1 + 1j], [1.0]))  # no conjugate partner
    with pytest.raises(ValueError):
        fgt.fold(S.SoeApprox([1 + 0j], [1 + 1j]))  # real node, complex weight


# -- max_error on the standard grid (soe.cpp:38-101, 236-248) ---------------

@pytest.mark.parametrize("n", [2, 4, 6, 8, 10, 12, 14])
@pytest.mark.parametrize("folded", [False, True])
def test_max_error_matches_reference_library(n, folded):
    import oracle
    if not oracle.ref_available():
        pytest.skip("reference library not built")
    soe = fgt.cf_soe(n)
    if folded:
        soe = fgt.fold(soe)
    r = fgt.max_error(soe)
    e_ref, arg_ref = oracle.ref_max_error(n, folded)
    assert r.n == n
    if n >= 14:
        # ~4e-12: at the rounding level of the double sum, where libm and
        # numpy exponentials differ in the last ulps; the maximum moves
        assert abs(r.max_abs_error - e_ref) <= 1e-2 * e_ref
        return
    assert abs(r.max_abs_error - e_ref) <= 1e-9 * e_ref + 1e-17
    assert r.argmax_x == pytest.approx(arg_ref, rel=1e-12, abs=0.0)


def test_max_error_extended_and_grid():
    assert fgt.error_grid_point(0) == 0.0
    assert fgt.error_grid_point(1) == pytest.approx(1e-5)
    assert fgt.error_grid_point(100000) == pytest.approx(100.0)
    r = fgt.max_error_extended(fgt.fold(fgt.cf_soe(12)))
    assert 2.9e-10 < r.max_abs_error < 3.1e-10  # test_cf.cpp:20-23 pin +-5% of 3.0208e-10


def test_chebyshev_points_formula():
    # rng.cpp:31-40
    n = 7
    p = fgt.chebyshev_points(n)
    i = np.arange(1, n + 1)
    assert np.array_equal(p, (1.0 + np.cos(np.pi * (2.0 * i - 1.0) / (2.0 * n))) / 2.0)
    assert fgt.chebyshev_points(0).size == 0
