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


# ---- the drop-in C++ API on several GPUs in one process (DREAMSCHED_GPUS) ----
# plsgd_step / run_training split the K workers over N labs (one per GPU,
# one host thread each, dsx_lab_comm_init_local): the reference's goldens
# must still match (trainer.hpp:94,112; trainer.cpp:237-307).

@pytest.mark.parametrize("gpus", [2, 4])
def test_cpp_api_plsgd_step_on_several_gpus(gpus, monkeypatch):
    if _gpus() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    from tests import test_gpu_parity as P
    monkeypatch.setenv("DREAMSCHED_GPUS", str(gpus))
    for fname in P.STEP_FILES:
        P.test_cpp_api_steps_match_reference(fname)


@pytest.mark.parametrize("gpus", [2, 4])
@pytest.mark.parametrize("cfg", ["lab_partial", "lab_full"])
def test_cpp_api_run_training_on_several_gpus(gpus, cfg, monkeypatch):
    if _gpus() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    from tests import test_gpu_parity as P
    monkeypatch.setenv("DREAMSCHED_GPUS", str(gpus))
    P.test_cpp_api_run_training_matches_reference(cfg)


def test_reference_unit_suite_trainer_cases_on_two_gpus(monkeypatch):
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs")
    from tests import test_unit_suite as U
    monkeypatch.setenv("DREAMSCHED_GPUS", "2")
    U.test_reference_unit_suite_trainer_cases_on_gpu()


@pytest.mark.parametrize("nranks", [2, 3, 4, 6, 8])
def test_p2p_average_kernel_ranks_bit_exact(nranks):
    """The cross-rank averaging kernel for up to 8 ranks (the 8-GPU
    instantiation included), ranks spread round-robin over this box's GPUs
    in one process: bit-identical to the reference's pairwise tree / K."""
    if _gpus() < 2:
        pytest.skip("needs >= 2 GPUs (peer access)")
    import ctypes as C
    from paper_2502_11058_b200 import native as N
    err = C.c_double()
    N.call("dsx_p2p_average_selftest", nranks, 100003, C.byref(err))
    assert err.value == 0.0, err.value
