"""BASELINE.json configs[0] as a parity case: the 8-layer, width-1024 MLP
shape registered as quadratic-lab blocks ("the reference
CPU run is run_training on Problem{block_sizes = per-layer param counts}"),
K = 4 workers, H = 4, sigma = 1, seed 1, with the ENP schedule and with the
searched schedule (schedule_dfs + bubble_fill of tests/golden/data/
mlp8_w1024.profile, pinned byte-identical to the reference in
test_native_cpu.py).  Full size (7,357,450 parameters per worker): the GPU
path against the C oracle step by step — max ||g||^2 and parameters at
1e-12 relative, every worker's mt19937_64 state exactly.
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from tests import golden_io as G

pytestmark = pytest.mark.gpu

PROFILE = os.path.join(G.DATA, "mlp8_w1024.profile")


def rel_err(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


@pytest.mark.parametrize("schedule", ["dfs", "enp"])
def test_config1_mlp_shaped_lab_matches_oracle(schedule):
    from paper_2502_11058_b200 import Lab, LabDesc
    from paper_2502_11058_b200.lab import lab_problem, schedule_from_profile, sync_mask
    K, H, sigma, seed = 4, 4, 1.0, 1
    sizes, dim = lab_problem(PROFILE)
    L = len(sizes)
    assert (L, dim) == (8, 7 * (1024 * 1024 + 1024) + 1024 * 10 + 10)
    if schedule == "dfs":
        sets, fills, _, _ = schedule_from_profile(PROFILE, H, fill=True)
    else:
        sets, fills = O.enp(L, H), None
    curv, _ = O.make_quadratic(dim, L)
    lab = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, sigma=sigma))
    lab.seed(seed)
    lab.fill(0.0)
    w = np.zeros((K, dim))
    rngs = [O.worker_rng(seed, k) for k in range(K)]
    bsz = np.asarray(sizes, dtype=np.uint64)
    for r in range(2 * H):
        eta = O.learning_rate(r, 1.0, 2.0, H)
        mask = sync_mask("partial", H, r, L, sets, fills)
        lab.step(eta, mask)
        g2 = O.plsgd_step(w, rngs, curv, np.ones(dim), sigma, bsz, eta, mask)
        assert rel_err(lab.max_grad_norm_sq(), g2) <= 1e-12, r
    assert rel_err(lab.get_params(), w) <= 1e-12
    for k in range(K):
        assert lab.rng_text(k) == O.mt_state_text(rngs[k])
    lab.close()
