"""Multi-GPU sharded path on >= 2 GPUs (torchrun + NCCL): tests/dist_sharded_check.py."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
def test_sharded_forward_bit_identical_to_single_gpu():
    n = min(_gpus(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29517",
           os.path.join(ROOT, "tests", "dist_sharded_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "bit-identical to the single-GPU path on every rank: True" in r.stdout


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
def test_cpp_sharded_network_bit_identical():
    """lattice::ShardedNetwork (C++ host over the C ABI, CUDA IPC + peer barriers) across
    processes: tests/cpp/test_sharded.cpp."""
    n = min(_gpus(), 4)
    r = subprocess.run([os.path.join(ROOT, "tests", "cpp", "test_sharded"), str(n)], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("bit-identical to") == n


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
def test_data_parallel_tower_training():
    """gradient all-reduce over NCCL keeps the replicas bit-identical."""
    n = min(_gpus(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29518", os.path.join(ROOT, "tests", "dist_train_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for red in ("nccl", "peer"):  # NCCL all-reduce + SGD, and the fused peer-memory reduce + SGD kernel
        assert f"[{red}] replicas bit-identical after every step: True" in r.stdout, r.stdout
        assert f"[{red}] loss falls: True" in r.stdout, r.stdout
    assert "peer-memory step matches the NCCL step: True" in r.stdout, r.stdout
