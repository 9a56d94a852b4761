"""Multi-GPU parity through the NCCL path (torchrun, one process per GPU);
skipped on single-GPU boxes."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT, cuda_available


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available() or _ngpu() < 2, reason="needs >= 2 GPUs")
def test_two_gpu_nccl_parity():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(ROOT, "tests", "mgpu_check.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "mgpu ok" in p.stdout
