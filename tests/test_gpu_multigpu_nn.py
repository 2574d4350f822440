"""The MLP's cross-rank scheduled averaging (NCCL, side stream) at 2 and 4
GPUs matches the single-GPU K-worker run and the float64 restatement
(tests/multigpu_mlp.py).  Skips on boxes with fewer GPUs."""
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


@pytest.mark.parametrize("graphs", [False, True])  # graphs: compute-only step graphs, NCCL averages eager behind external events (several ranks)
@pytest.mark.parametrize("world", [2, 4])
def test_mlp_multirank_matches_single_gpu(world, graphs):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world + 10 * graphs),
           os.path.join(REPO, "tests", "multigpu_mlp.py")]
    env = dict(os.environ, DSX_TEST_GRAPHS="1" if graphs else "0")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert '"pass": true' in out.stdout


def test_mlp_multirank_graphs_without_overlap():
    """Hybrid graphs with every average after the whole local step (the
    ssgd / flsgd modes): the external event sits at the end of the BP."""
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29637",
           os.path.join(REPO, "tests", "multigpu_mlp.py")]
    env = dict(os.environ, DSX_TEST_GRAPHS="1", DSX_TEST_OVERLAP="0")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert '"pass": true' in out.stdout


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("world", [2, 4])
def test_cnn_multirank_matches_single_gpu(world, dtype):
    """The conv stack (BASELINE configs[1] shape) across ranks: fp32 within
    1e-5 of one GPU and of float64; bf16 (implicit-GEMM convs) within bf16
    tolerance; averaged layers identical on every worker."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29640 + world + 10 * (dtype == "bf16")),
           os.path.join(REPO, "tests", "multigpu_cnn.py")]
    env = dict(os.environ, DSX_TEST_DTYPE=dtype)
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert '"pass": true' in out.stdout
