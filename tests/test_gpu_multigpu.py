"""Cross-rank averaging over NCCL/NVLink (2+ GPUs): bit-exact with the
reference's in-process K-worker mean.  Skips on single-GPU boxes."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world", [2, 4])
def test_multirank_sync_bit_exact(world):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world),
           os.path.join(REPO, "tests", "multigpu_parity.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert '"pass": true' in out.stdout


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
def test_multirank_fused_update_average_bit_exact():
    """The opt-in fused update + cross-rank average (DSX_FUSED=1: one kernel,
    per-tile peer-memory handshake) is bit-identical too."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29517",
           os.path.join(REPO, "tests", "multigpu_parity.py")]
    env = dict(os.environ, DSX_FUSED="1")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert '"pass": true' in out.stdout
