"""The per-process multi-GPU leg (bench.py under torchrun)
on a real NCCL process group: tests/workers/nccl_gather.py launched by
torch.distributed.run with one process per visible GPU (gpurun grants one,
so world size 1 here: NCCL init, the record all-gather and the max-over-ranks
all-reduce all run through NCCL; the gather/combine logic at world size 2 is
tests/test_distributed.py over gloo). theta_combined must equal one process
fitting every block, bit for bit."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_torchrun_nccl_gather_combine():
    import torch
    ngpu = torch.cuda.device_count()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(ngpu),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "workers", "nccl_gather.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    ok = [l for l in r.stdout.splitlines() if l.startswith("NCCL_OK")]
    assert len(ok) == 3 * ngpu, r.stdout
