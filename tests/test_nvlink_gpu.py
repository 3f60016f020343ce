"""Multi-process NVLink engine: parity run under torchrun on 2..N GPUs.

Skipped on single-GPU boxes (fused peer kernels must never be emulated as
waiting launches on one GPU); run with `gpurun --gpus 2/4`.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch

    return torch.cuda.device_count()


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
def test_nvlink_parity_all_gpus():
    n = min(_ngpus(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", "29617", os.path.join(ROOT, "tests", "nvlink_parity.py")]
    env = dict(os.environ, HCCX_TIMEOUT_MS="20000")
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0 and "NVLINK PARITY OK" in r.stdout


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
def test_trainer_across_processes_matches_reference():
    """trainer_dist.DistTrainer3D, one process per GPU over the NVLink
    engine, against the reference trainer's golden runs of this world size."""
    n = 4 if _ngpus() >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", "29618", os.path.join(ROOT, "tests", "trainer_dist_parity.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=dict(os.environ, HCCX_TIMEOUT_MS="20000"), capture_output=True, text=True,
                       timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0 and "TRAINER DIST PARITY OK" in r.stdout


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
def test_nvlink_randomized_soak():
    """Random ops / sizes / codecs back to back (tests/nvlink_soak.py)."""
    n = min(_ngpus(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", "29619", os.path.join(ROOT, "tests", "nvlink_soak.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=dict(os.environ, SOAK_ITERS="80", HCCX_TIMEOUT_MS="20000"),
                       capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0 and "NVLINK SOAK OK" in r.stdout
