"""Per-layer, per-worker error of dsx_cnn after a few steps against the
float64 restatement (debug aid)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle.cnn_oracle import CnnOracle, topology  # noqa: E402
from paper_2502_11058_b200.cnn import Cnn, batch, init_params, teacher  # noqa: E402
from paper_2502_11058_b200.lab import enp, sync_mask  # noqa: E402


def run(width, image, K, H, steps, dtype, bsz, lr=0.02, seed=2, opt="momentum"):
    m = Cnn(bsz, K, width=width, image=image, dtype=dtype, optimizer=opt)
    convs, _, _ = topology(width, image, 8, 10)
    roles = [c["role"] for c in convs] + ["head"]
    init = init_params(seed, m.layer_sizes(), m.fan_in, roles)
    for k in range(K):
        m.set_params(k, init)
    orc = CnnOracle(width, image, 3, 10, init, K, optimizer=opt)
    t = teacher(seed, image, 3, 10)
    sets = enp(m.L, H)
    for r in range(steps):
        bs = [batch(seed, k, r, bsz, image, 3, t) for k in range(K)]
        mask = sync_mask("partial", H, r, m.L, sets)
        m.set_batch(np.stack([b[0] for b in bs]), np.stack([b[1] for b in bs]))
        m.step(lr, r, mask)
        orc.step(bs, lr, r, mask)
        print(f"{dtype} w{width} K{K} step {r}: loss gpu {m.last_loss()} f64 {orc.loss}")
    for k in range(K):
        g = m.get_params(k)
        errs = []
        for l in range(m.L):
            lo, hi = m.offsets[l], m.offsets[l + 1]
            d = init[lo:hi] - orc.w[k][lo:hi]
            e = np.linalg.norm((init[lo:hi] - g[lo:hi]) - d) / max(np.linalg.norm(d), 1e-30)
            errs.append(f"{e:.1e}")
        print(f"  worker {k} per-layer update error: {' '.join(errs)}")
    m.close()


if __name__ == "__main__":
    run(16, 16, 2, 2, 1, "f32", 8)
    run(16, 16, 2, 2, 1, "bf16", 8)
    run(16, 16, 1, 2, 1, "bf16", 8)
    run(16, 16, 4, 2, 1, "bf16", 8)
    run(64, 32, 2, 2, 1, "bf16", 8)
