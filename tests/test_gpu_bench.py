"""bench.py contract on the GPU: one JSON line with the keys the driver reads, at N = 1 and
through the multi-process (torchrun) path with two ranks, one GPU each (skipped on a one-GPU box)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
        "clocks")


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def test_bench_one_gpu_small():
    r = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--steps", "3", "--warmup",
                        "3", "--cpu-sample", "64"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    j = _line(r.stdout)
    for k in KEYS:
        assert k in j, k
    assert j["n_gpus"] == 1 and j["value"] > 0 and j["gpu_launches"] > 0
    assert j["roofline"]["frac"] is not None and j["cpu_baseline"]["kind"] == "oracle"
    assert j["e2e"]["h2d_bytes_per_step"] > 0 and j["device_flags"] == 0


@pytest.mark.skipif(
    __import__("torch").cuda.device_count() < 2 and os.environ.get("MOE_TEST_SHARED_GPU_PROCS") != "1",
    reason="needs one GPU per rank: ranks whose kernels spin on each other's flags must not share "
           "a GPU as separate processes (B200_PROFILING.md, Xid 109)")
def test_bench_two_ranks():
    """Two ranks, one GPU each (the driver's N = 2 launch).  With MOE_TEST_SHARED_GPU_PROCS=1 on
    a one-GPU box both ranks share cuda:0 through the MOE_BENCH_SHARE_GPU hook (manual only)."""
    import torch
    env = dict(os.environ)
    if torch.cuda.device_count() < 2:
        env["MOE_BENCH_SHARE_GPU"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2",
           "--config", "c1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    j = _line(r.stdout)
    assert j["n_gpus"] == 2 and j["value"] > 0 and j["device_flags"] == 0
    assert "ep2" in j["config"]["parallelism"] and "peer" in j["config"]["parallelism"]
