"""a11 on real GPUs: N ranks (torchrun, NCCL over NVLink) must return the
single-GPU frontier bit for bit on every rank.  Skipped with < 2 GPUs."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("workload,ykey", [(1, 0), (1, 1), (2, 0)])
def test_nccl_merge_equals_single_gpu(workload, ykey):
    n = _ngpu()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_2503_19050_b200 import build
    build.build()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={min(n, 8)}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + 10 * workload + ykey),
           os.path.join(ROOT, "tools", "mgpu_check.py"), "--workload", str(workload), "--ykey", str(ykey)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0
    assert "merged==single: True" in r.stdout and "identical on all ranks: True" in r.stdout
