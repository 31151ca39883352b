"""bench.py --impl reference (the reference arm: the reference's own CPU
transform path on our arm's workload), single process and under torchrun
(rank 0 alone prints; the other ranks exit 0).  CPU only; a small --n keeps
it quick (the driver runs the default N = M = 1e8)."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--impl", "reference", "--steps", "2", "--warmup", "1", "--size", "20000"]


def _lines(out):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


def test_reference_arm_line():
    out = subprocess.run([sys.executable, "bench.py"] + ARGS, cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    (d,) = _lines(out.stdout)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 2
    assert d["value"] > 0 and d["unit"] == "points/s" and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["cores"] >= 1
    assert cb["kind"] in ("reference", "port")
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    # same workload dict as our arm reports
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.workload_config(20000, 1e-3, 1e-10)


def test_reference_arm_loads_no_product_code():
    # the reference arm runs the reference's own transform (oracle/_ref) and
    # nothing of the product: no package import, no libfgt1d_b200.so mapped
    code = ("import sys, bench; sys.argv = ['bench.py'] + %r; bench.main(); "
            "import sys; maps = open('/proc/self/maps').read(); "
            "assert 'libfgt1d_b200' not in maps, 'product library mapped'; "
            "assert not any(m.startswith('paper_1909_09825_b200') for m in sys.modules); "
            "print('CLEAN')" % (ARGS,))
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "CLEAN" in out.stdout


def test_reference_arm_under_torchrun_prints_once():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", "bench.py", "--gpus", "2"] + ARGS
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    (d,) = _lines(out.stdout)
    assert d["impl"] == "reference" and d["n_gpus"] == 2
