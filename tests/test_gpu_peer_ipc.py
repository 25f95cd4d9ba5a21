"""Peer-memory transport across PROCESSES (N1): two ranks as two processes, windows opened
from CUDA IPC handles (moe_peer_export / moe_peer_import) all-gathered over a gloo group.
Each process takes its own GPU.  With fewer GPUs than ranks the test is skipped: kernels that
spin on flags another process writes must not share one GPU (B200_PROFILING.md: two such
processes on one B200 raised Xid 109, a context-switch timeout); MOE_TEST_SHARED_GPU_PROCS=1
forces the shared-GPU run for manual checks.  The multi-rank protocol is covered on one GPU by
the in-process virtual-rank tests (test_gpu_ep.py) and on the CPU by test_ep_cpu.py."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(
    torch.cuda.device_count() < 2 and os.environ.get("MOE_TEST_SHARED_GPU_PROCS") != "1",
    reason="needs one GPU per process (spinning cross-process kernels must not share a GPU)")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("shape", ["", "ret"])
def test_peer_transport_two_processes_ipc(shape):
    """shape "ret": d = 128, top-1 -- the owners' GEMM epilogues store O and dx rows into
    the other PROCESS's window (return rows + fused dispatch backward)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "workers", "peer_ipc_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=ROOT,
                       env=dict(os.environ, IPC_SHAPE=shape))
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-3000:]
    assert out.count(": OK") == 2, out[-3000:]
