"""CPU checks of the NN restatement (oracle/mlp_oracle.py, test
infrastructure) — the reference has no NN to pin it against, so its math is
pinned here: the backward pass against central finite differences of its own
loss, the optimizers against their closed forms, and the average against
pairwise_coord_sum's tree (trainer.cpp:31-38)."""
import numpy as np
import pytest

from oracle.mlp_oracle import MlpOracle, pairwise_sum, split
from paper_2502_11058_b200.nn import batch, init_params, teacher


def _loss(orc, w, x, y):
    L = len(orc.widths) - 1
    a = x.astype(np.float64)
    for l, (W, b) in enumerate(split(w, orc.widths)):
        z = a @ W.T + b
        a = np.maximum(z, 0.0) if l < L - 1 else z
    zmax = a.max(axis=1, keepdims=True)
    lse = zmax[:, 0] + np.log(np.exp(a - zmax).sum(axis=1))
    return float(np.mean(lse - a[np.arange(len(y)), y]))


def test_backward_matches_finite_differences():
    widths, seed = [12, 9, 7, 5], 4
    t = teacher(seed, widths[0], widths[-1])
    x, y = batch(seed, 0, 0, 16, widths[0], t)
    init = init_params(seed, widths).astype(np.float64)
    orc = MlpOracle(widths, init, 1, optimizer="sgd")
    lr = 1.0
    orc.local_step(0, x, y, lr, 0)
    grad = (init - orc.w[0]) / lr  # plain SGD: w1 = w0 - lr * g
    rng = np.random.default_rng(0)
    for i in rng.choice(len(init), 40, replace=False):
        e = np.zeros_like(init)
        e[i] = 1e-6
        fd = (_loss(orc, init + e, x, y) - _loss(orc, init - e, x, y)) / 2e-6
        assert fd == pytest.approx(grad[i], rel=1e-5, abs=1e-8), i


def test_optimizers_closed_form():
    widths = [4, 3, 2]
    init = init_params(1, widths).astype(np.float64)
    g = np.linspace(-1, 1, len(init))
    for opt in ("sgd", "momentum", "adam"):
        orc = MlpOracle(widths, init, 1, optimizer=opt, momentum=0.9, beta1=0.9, beta2=0.999, eps=1e-8)
        orc._update(0, 0, len(init), g.copy(), 0.1, 0)
        orc._update(0, 0, len(init), g.copy(), 0.1, 1)
        if opt == "sgd":
            want = init - 0.2 * g
        elif opt == "momentum":
            want = init - 0.1 * g - 0.1 * (0.9 * g + g)
        else:  # Adam with a constant gradient: both bias-corrected steps are lr * g/(|g| + eps)
            step = g / (np.abs(g) + 1e-8)
            want = init - 0.1 * step - 0.1 * step
        np.testing.assert_allclose(orc.w[0], want, rtol=1e-12, atol=1e-12)


def test_average_is_the_pairwise_tree():
    rows = [np.array([1e16, 1.0, 3.0]), np.array([1.0, 2.0, 5.0]), np.array([-1e16, 4.0, 7.0]),
            np.array([1.0, 8.0, 11.0])]
    got = pairwise_sum(rows, 0, 4)
    want = (rows[0] + rows[1]) + (rows[2] + rows[3])
    assert np.array_equal(got, want)
