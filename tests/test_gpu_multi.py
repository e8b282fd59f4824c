"""Multi-GPU parity: the column-slab path on 2..8 real GPUs (one process per
GPU, NCCL process group; the candidate-column exchange over peer memory and over NCCL), bit for
bit against the oracle.  Runs only on a box with >= 2 GPUs (skipped on the 1-GPU round-end box;
the same data flow is covered on one GPU by the virtual-slab tests of test_gpu_lookahead.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


def test_column_slabs_on_real_gpus():
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for world in sorted({2, min(n, 8)}):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1",
               f"--nproc-per-node={world}", os.path.join(root, "tests", "mgpu_worker.py")]
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root,
                             env=dict(os.environ, MASTER_ADDR="127.0.0.1"))
        assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
