"""CLI front end (reference proj/tools/fgt1d_cli.cpp schema): host-side parts
on CPU; the device subcommands are in the GPU suite (test_gpu_cli below)."""
import json
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_1909_09825_b200 as fgt
from paper_1909_09825_b200 import cli


def run_cli(*args):
    p = subprocess.run([sys.executable, "-m", "paper_1909_09825_b200.cli", *args],
                       capture_output=True, text=True)
    return p.returncode, p.stdout, p.stderr


def test_soe_subcommand_prints_grid_error_and_saves_table(tmp_path):
    out = tmp_path / "cf8.txt"
    rc, so, _ = run_cli("soe", "--n", "8", "--out", str(out))
    assert rc == 0
    line = so.strip()
    assert line.startswith("n=8 max_error=")
    err = float(line.split("max_error=")[1].split()[0])
    assert 1.19e-6 <= err <= 1.33e-6  # cli_checks.py:51-52 window
    t = fgt.load_coefficient_table(str(out))
    assert len(t) == 8 and t.form == fgt.SoeForm.FULL


def test_exit_codes_follow_the_reference():
    # fgt1d_cli.cpp:577-590: invalid input -> 2
    assert run_cli("soe", "--method", "talbot")[0] == 2
    assert run_cli("bench", "--N", "0")[0] == 2
    assert run_cli("bench", "--scenario", "sideways")[0] == 2
    assert run_cli("delta-sweep", "--delta", "-1")[0] == 2
    assert run_cli("transform", "/nonexistent/file.csv")[0] == 2
    assert run_cli("nonsense")[0] == 2
    assert run_cli("--help")[0] == 0


def test_point_file_parsing(tmp_path):
    # fgt1d_cli.cpp:360-400: header tolerated once, comments, separators
    f = tmp_path / "pts.csv"
    f.write_text("x,alpha\n0.5, 2.0\n# comment\n0.25;1\n\n0.75\t-3 # trailing\n")
    c, a = cli.read_point_file(str(f))
    assert c == [0.5, 0.25, 0.75] and a == [2.0, 1.0, -3.0]
    g = tmp_path / "bad.csv"
    g.write_text("0.1,1\nnot-a-number,2\n")
    with pytest.raises(ValueError):
        cli.read_point_file(str(g))
    h = tmp_path / "ragged.csv"
    h.write_text("0.1,1\n0.2\n")
    with pytest.raises(ValueError):
        cli.read_point_file(str(h))


@pytest.mark.gpu
def test_gpu_cli_bench_transform_and_sweep(tmp_path):
    rc, so, se = run_cli("bench", "--N", "20000", "--ne", "4", "--delta", "1e-3", "--json",
                         "--repeat", "2")
    assert rc == 0, se
    rows = json.loads(so)
    assert len(rows) == 2 and rows[0]["scenario"] == "SamePoints"
    for k in ("t_sort", "t_pre", "t_rem", "t_total", "max_rel_error", "throughput_full",
              "throughput_amortized"):
        assert k in rows[0]
    assert rows[0]["max_rel_error"] < 1e-5
    rc, so, se = run_cli("bench", "--scenario", "distinct", "--N", "5000", "--M", "7000")
    assert rc == 0, se
    hdr, row = so.strip().splitlines()
    assert hdr == cli.BENCH_HEADER and row.startswith("DistinctPoints,5000,7000,4,")
    # transform on files: same numbers as the library call
    x = fgt.uniform_points_array(500, 3, 3)
    y = fgt.uniform_points_array(400, 3, 0)
    a = 2.0 * fgt.uniform_points_array(400, 3, 1) - 1.0
    sf, tf = tmp_path / "s.csv", tmp_path / "t.csv"
    sf.write_text("\n".join(f"{float(v)!r},{float(w)!r}" for v, w in zip(y, a)) + "\n")
    tf.write_text("\n".join(repr(float(v)) for v in x) + "\n")
    rc, so, se = run_cli("transform", str(sf), str(tf), "--delta", "0.01", "--ne", "6")
    assert rc == 0, se
    lines = so.strip().splitlines()
    assert lines[0] == "index,potential"
    got = np.array([float(l.split(",")[1]) for l in lines[1:]])
    assert np.max(np.abs(got - oracle.transform(x, y, a, 0.01, ne=6, mode=0))) <= 1e-12 * np.abs(a).sum()
    rc, so, se = run_cli("delta-sweep", "--N", "5000", "--delta", "1e-4", "--delta", "1")
    assert rc == 0, se
    assert so.splitlines()[0] == "delta,error" and len(so.splitlines()) == 3
