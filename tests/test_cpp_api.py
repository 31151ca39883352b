"""Runs the C++ API test binary (tests/cpp/test_fgt1d_api.cpp) against the
drop-in host library include/fgt1d/*.hpp -> libfgt1d.so -> libfgt1d_b200.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1909_09825_b200", "lib", "test_fgt1d_api")


def run(mode):
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} missing: run __graft_entry__.build()")
    r = subprocess.run([BIN, mode], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout


def test_cpp_api_host_side():
    run("cpu")


@pytest.mark.gpu
def test_cpp_api_transforms():
    run("gpu")
