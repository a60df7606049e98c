"""Multi-GPU parity under torchrun + NCCL (tests/mp_parity.py), one rank per GPU.

Skips the topologies that need more GPUs than the box has; the single-GPU
LocalCluster tests in test_gpu_parity.py cover the same goldens in one process.
"""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("grouping", ["1x2", "2x1", "2x2", "1x4", "4x1", "2x4", "4x2"])
def test_torchrun_nccl_parity(grouping):
    m, p = (int(x) for x in grouping.split("x"))
    n = m * p
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n * 7 + m),
           os.path.join(ROOT, "tests", "mp_parity.py"), grouping]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ok" in r.stdout


VARIANTS = [("1x2", {"HSX_K1_SPLIT": "1"}), ("2x2", {"HSX_K1_SPLIT": "1"}), ("2x2", {"HSX_FUSED_UNION": "0"}),
            ("2x2", {"HSX_ONESIDED": "1"})]


@pytest.mark.parametrize("idx", range(len(VARIANTS)))
def test_torchrun_parity_variants(idx):
    """The opt-in / fallback step variants (split two-rank K1, K4 before K5, one-sided
    leader hand-offs) against the same goldens and full-size agreement checks."""
    grouping, env = VARIANTS[idx]
    m, p = (int(x) for x in grouping.split("x"))
    n = m * p
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29650 + idx),
           os.path.join(ROOT, "tests", "mp_parity.py"), grouping]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env={**os.environ, "HSX_BARRIER_TIMEOUT_S": "60", **env})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ok" in r.stdout
