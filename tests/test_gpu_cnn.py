"""Conv-stack local step on the GPU (BASELINE configs[1] as a network):
dsx_cnn_* against the float64 restatement oracle/cnn_oracle.py.

* fp32 (SIMT GEMMs): after one step every worker within 1e-6 (relative L2)
  of float64; after 2H steps of scheduled partial sync at a small lr within
  1e-5 (north_star: fp32 parameters within 1e-5); synced layers identical on
  every worker, unsynced ones different;
* bf16 (tcgen05/TMA GEMMs): the full ResNet-18 shape trains (loss falls) and
  a reduced-width net tracks the float64 restatement's loss step by step.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle.cnn_oracle import CnnOracle  # noqa: E402  (checker only)
from paper_2502_11058_b200.cnn import Cnn, batch, init_params, teacher  # noqa: E402
from paper_2502_11058_b200.lab import enp, sync_mask  # noqa: E402


def _init(m, seed):
    roles = []
    from oracle.cnn_oracle import topology
    convs, _, _ = topology(m.width, m.image, 8, m.classes)
    roles = [c["role"] for c in convs] + ["head"]
    return init_params(seed, m.layer_sizes(), m.fan_in, roles)


def _run(width, image, K, H, steps, optimizer, lr, dtype="f32", bsz=4, seed=2, classes=10, oracle=True):
    m = Cnn(bsz, K, width=width, image=image, classes=classes, dtype=dtype, optimizer=optimizer,
            eps=1e-6 if optimizer == "adam" else 1e-8)
    init = _init(m, seed)
    for k in range(K):
        m.set_params(k, init)
    orc = CnnOracle(width, image, 3, classes, init, K, optimizer=optimizer,
                    eps=1e-6 if optimizer == "adam" else 1e-8) if oracle else None
    t = teacher(seed, image, 3, classes)
    sets = enp(m.L, H)
    losses, masks = [], []
    for r in range(steps):
        bs = [batch(seed, k, r, bsz, image, 3, t) for k in range(K)]
        mask = sync_mask("partial", H, r, m.L, sets)
        m.set_batch(np.stack([b[0] for b in bs]), np.stack([b[1] for b in bs]))
        m.step(lr, r, mask)
        if orc is not None:
            orc.step(bs, lr, r, mask)
        losses.append((m.last_loss().copy(), orc.loss.copy() if orc is not None else None))
        masks.append(mask)
    got = [m.get_params(k) for k in range(K)]
    offsets = m.offsets
    m.close()
    return got, orc, losses, masks, offsets


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("optimizer,lr", [("momentum", 0.01), ("adam", 1e-3), ("sgd", 0.05)])
def test_cnn_fp32_one_step_matches_cpu_restatement(optimizer, lr):
    got, orc, losses, _, _ = _run(16, 16, 4, 2, 1, optimizer, lr)
    for k in range(4):
        assert _rel(got[k], orc.w[k]) <= 1e-6, (optimizer, k, _rel(got[k], orc.w[k]))
    np.testing.assert_allclose(losses[0][0], losses[0][1], rtol=1e-5)


@pytest.mark.parametrize("optimizer", ["momentum", "adam"])
def test_cnn_fp32_trajectory_within_1e5(optimizer):
    K, H = 4, 2
    got, orc, losses, masks, offs = _run(8, 16, K, H, 2 * H, optimizer, 1e-3 if optimizer == "momentum" else 1e-4)
    for k in range(K):
        assert _rel(got[k], orc.w[k]) <= 1e-5, (optimizer, k, _rel(got[k], orc.w[k]))
    for gl, ol in losses:
        np.testing.assert_allclose(gl, ol, rtol=1e-4)
    last = masks[-1]
    for l in range(1, len(offs)):
        lo, hi = offs[l - 1], offs[l]
        same = all(np.array_equal(got[0][lo:hi], g[lo:hi]) for g in got)
        if last[l]:
            assert same, l


def test_cnn_bf16_tracks_float64_loss():
    K, H = 2, 2
    got, orc, losses, _, _ = _run(16, 16, K, H, 6, "momentum", 0.02, dtype="bf16", bsz=8)
    for gl, ol in losses:
        np.testing.assert_allclose(gl, ol, rtol=3e-2)
    for k in range(K):
        assert _rel(got[k], orc.w[k]) < 2e-2


@pytest.mark.parametrize("image", [16, 32])
def test_cnn_implicit_gemm_convs_track_float64(image):
    """Width 64: every 3x3 stride-1 conv runs as an implicit GEMM (shifted
    5-D TMA boxes, no im2col); 3 steps at K = 2 track float64 (images 16:
    stage grids 16/8/4/2; 32: 32/16/8/4)."""
    # lr 0.005: at 0.02 this batch-4 run diverges (loss 2.3 -> 5) and bf16
    # rounding differences grow with it
    got, orc, losses, _, _ = _run(64, image, 2, 2, 3, "momentum", 0.005, dtype="bf16", bsz=4)
    for gl, ol in losses:
        np.testing.assert_allclose(gl, ol, rtol=3e-2)
    for k in range(2):
        assert _rel(got[k], orc.w[k]) < 2e-2, (k, _rel(got[k], orc.w[k]))


def test_cnn_resnet18_bf16_first_step_loss():
    """Full ResNet-18 geometry, K = 2, batch 8: the tensor-core forward's loss
    within bf16 rounding of float64's, per worker."""
    got, orc, losses, _, _ = _run(64, 32, 2, 2, 1, "momentum", 0.02, dtype="bf16", bsz=8)
    np.testing.assert_allclose(losses[0][0], losses[0][1], rtol=3e-3)
    for k in range(2):
        assert _rel(got[k], orc.w[k]) < 1e-2


def test_cnn_resnet18_bf16_trains():
    """The full ResNet-18 shape (width 64, 32x32x3, 10 classes), K = 2, batch
    32 per worker, H = 2: the tensor-core path runs and the loss falls over
    repeated passes over one pool of batches."""
    K, H, bsz, seed = 2, 2, 32, 5
    m = Cnn(bsz, K, dtype="bf16", optimizer="momentum")
    init = _init(m, seed)
    for k in range(K):
        m.set_params(k, init)
    t = teacher(seed, 32, 3, 10)
    pool = [[batch(seed, k, p, bsz, 32, 3, t) for k in range(K)] for p in range(2)]
    sets = enp(m.L, H)
    losses = []
    for r in range(40):
        bs = pool[r % 2]
        m.set_batch(np.stack([b[0] for b in bs]), np.stack([b[1] for b in bs]))
        m.step(0.02, r, sync_mask("partial", H, r, m.L, sets))
        losses.append(float(np.mean(m.last_loss())))
    m.close()
    assert np.all(np.isfinite(losses))
    assert np.mean(losses[-4:]) < 0.9 * np.mean(losses[:2]), losses
