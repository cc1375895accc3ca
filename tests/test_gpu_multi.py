"""Multi-GPU parity (needs >= 2 GPUs): branch sharding + NCCL reduction vs the oracle."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
def test_two_gpu_sharded_reduction():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "tools", "mgpu_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
def test_distributed_halves():
    """Every half sharded over the GPUs (QSIM_OPT_DISTRIBUTE), fused local/global swaps over peer memory,
    against the oracle (2 GPUs; 4 GPUs when present)."""
    for n in (2, 4):
        if _ngpus() < n:
            continue
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(29533 + n),
               os.path.join(ROOT, "tools", "mgpu_check.py"), "--dist"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
        print(r.stdout[-4000:], r.stderr[-3000:])
        assert r.returncode == 0, n
