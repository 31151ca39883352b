"""bench.py's multi-rank path end to end (N > 1 ranks under torchrun).

The box has one GPU, so the ranks share it and exchange over gloo
(FGT_BENCH_BACKEND=gloo, the bench's test hook); the device-side aggregate
exchange (FGT_DEVICE_AGGS, fgt_chunk_carries_device) and the host-buffer e2e
chunk path run as they would over NCCL.  --check makes rank 0 compare the
ranks' potentials with one plan over the whole stream.  Timings here mean
nothing (ranks share a GPU)."""
import json
import os
import socket
import subprocess
import sys

import pytest

from paper_1909_09825_b200 import _capi

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_bench_multirank_device_exchange(world):
    if _capi.lib().fgt_device_count() < 1:
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    env = dict(os.environ, FGT_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
           "bench.py", "--gpus", str(world), "--steps", "2", "--warmup", "1", "--size", "300000",
           "--no-cpu-baseline", "--no-sweep", "--e2e-steps", "1", "--check"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == world
    assert d["multi_rank_check"]["pass"], d["multi_rank_check"]
    assert d["e2e"]["matches_device_path"], d["e2e"]


def test_bench_chunk_path_single_rank():
    """--chunk-path on one GPU: the per-rank step of the multi-GPU path, checked
    against one plan."""
    if _capi.lib().fgt_device_count() < 1:
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    cmd = [sys.executable, "bench.py", "--steps", "2", "--warmup", "1", "--size", "400000",
           "--no-cpu-baseline", "--no-sweep", "--no-e2e", "--chunk-path", "--check"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["parallelism"] == "1 GPU (chunk path)"
    assert d["multi_rank_check"]["pass"], d["multi_rank_check"]


def test_bench_chunk_path_over_nccl_world_one():
    """The multi-rank step with its collectives over the real backend: torchrun
    with one rank, a forced NCCL process group (FGT_BENCH_FORCE_PG), so the
    aggregate all_gather_into_tensor, the device-id barrier, the max-over-ranks
    all_reduce and the check's all_gather run through NCCL on the box's GPU."""
    if _capi.lib().fgt_device_count() < 1:
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    env = dict(os.environ, FGT_BENCH_FORCE_PG="1")
    env.pop("FGT_BENCH_BACKEND", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", "bench.py", "--gpus", "1",
           "--steps", "2", "--warmup", "1", "--size", "400000", "--no-cpu-baseline",
           "--no-sweep", "--no-e2e", "--chunk-path", "--check"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["multi_rank_check"]["pass"], d["multi_rank_check"]


@pytest.mark.parametrize("world", [1, 2])
def test_bench_cfg5_transforms_split_over_ranks(world):
    """--config 5 under torchrun: the batched transforms split over the ranks
    (no exchange), every rank's potentials checked against one batched plan
    over all transforms on rank 0."""
    if _capi.lib().fgt_device_count() < 1:
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    env = dict(os.environ, FGT_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
           "bench.py", "--config", "5", "--gpus", str(world), "--steps", "2", "--warmup", "1",
           "--cfg5-transforms", "12", "--cfg5-size", "5000", "--tols", "1e-6", "--check"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == world
    assert d["config"]["transforms"] == 12
    assert d["multi_rank_check"]["pass"], d["multi_rank_check"]
