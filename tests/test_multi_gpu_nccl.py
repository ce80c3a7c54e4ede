"""Element-partitioned multi-GPU run over NCCL (one process per GPU, torchrun) against the single-GPU
run.  Needs >= 2 visible GPUs; the round-end GPU box has one, so this skips there and runs on any
multi-GPU node (the same check the bench's N > 1 launch depends on)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("N,M,n", [(4, 2, 6), (7, 4, 4)])
def test_two_rank_nccl_matches_single_gpu(N, M, n):
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29641", os.path.join(ROOT, "scripts", "nccl_parity.py"),
           str(N), str(M), str(n)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert '"ok": true' in r.stdout
