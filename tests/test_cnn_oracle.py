"""CPU checks of the conv-stack restatement (oracle/cnn_oracle.py, test
infrastructure) — the reference has no network to pin it against, so its
math is pinned here: im2col/col2im adjointness, the backward pass against
central finite differences of its own loss, the topology against ResNet-18's
layer inventory, and the average against pairwise_coord_sum's tree."""
import numpy as np
import pytest

from oracle.cnn_oracle import CnnOracle, col2im, im2col, layer_sizes, topology
from paper_2502_11058_b200.cnn import batch, init_params, teacher


def _small(seed=3, width=8, image=8, cin=3, classes=5):
    convs, _, head = topology(width, image, 8, classes)
    sizes = layer_sizes(width, image, 8, classes)
    fan = [c["k"] * c["k"] * c["cin"] for c in convs] + [head["cin"]]
    roles = [c["role"] for c in convs] + ["head"]
    return init_params(seed, sizes, fan, roles).astype(np.float64), sizes


def test_resnet18_inventory():
    convs, blocks, head = topology(64, 32, 8, 10)
    assert len(convs) + 1 == 21  # stem + 16 block convs + 3 projections + head
    assert [c["cout"] for c in convs if c["role"] == "sc"] == [128, 256, 512]
    assert head["cin"] == 512
    # conv biases instead of BatchNorm: 11.17M parameters with the 3-channel
    # stem, as CIFAR ResNet-18 (11.17M with BN affine, no conv biases)
    assert sum(layer_sizes(64, 32, 3, 10)) == 11_169_162


@pytest.mark.parametrize("k,stride", [(3, 1), (3, 2), (1, 2)])
def test_im2col_col2im_adjoint(k, stride):
    rng = np.random.default_rng(0)
    c = dict(k=k, stride=stride, cin=8)
    x = rng.standard_normal((2, 8, 8, 8))
    col = im2col(x, c)
    d = rng.standard_normal(col.shape)
    assert np.vdot(col, d) == pytest.approx(np.vdot(x, col2im(d, c, 8)), rel=1e-12)


def test_backward_matches_finite_differences():
    seed, width, image, cin, classes = 3, 8, 8, 3, 5
    init, sizes = _small(seed, width, image, cin, classes)
    t = teacher(seed, image, cin, classes)
    x, y = batch(seed, 0, 0, 3, image, cin, t)
    orc = CnnOracle(width, image, cin, classes, init, 1, optimizer="sgd")
    orc.local_step(0, x.astype(np.float64), y, 1.0, 0)
    grad = init - orc.w[0]  # plain SGD, lr = 1: w1 = w0 - g (input grads use pre-update weights)

    def loss(w):
        o = CnnOracle(width, image, cin, classes, w, 1, optimizer="sgd")
        o.local_step(0, x.astype(np.float64), y, 0.0, 0)
        return o.loss[0]

    rng = np.random.default_rng(1)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    # a few coordinates of every registered layer (weights and biases), skipping
    # the stem's zero-padded input channels (their gradient is exactly 0)
    picks = []
    for l in range(len(sizes)):
        picks += list(rng.integers(offs[l], offs[l + 1], 3))
    for i in picks:
        e = np.zeros_like(init)
        e[i] = 1e-6
        fd = (loss(init + e) - loss(init - e)) / 2e-6
        assert fd == pytest.approx(grad[i], rel=2e-5, abs=1e-9), i


def test_step_averages_masked_layers_pairwise():
    seed, width, image, cin, classes = 4, 8, 8, 3, 5
    init, sizes = _small(seed, width, image, cin, classes)
    t = teacher(seed, image, cin, classes)
    K = 4
    orc = CnnOracle(width, image, cin, classes, init, K, optimizer="momentum")
    mask = np.zeros(len(sizes) + 1, dtype=np.uint8)
    mask[[1, 5, len(sizes)]] = 1
    orc.step([batch(seed, k, 0, 2, image, cin, t) for k in range(K)], 0.05, 0, mask)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    for l in range(1, len(sizes) + 1):
        lo, hi = offs[l - 1], offs[l]
        same = all(np.array_equal(orc.w[0][lo:hi], w[lo:hi]) for w in orc.w)
        assert same == bool(mask[l]), l
