"""A few training steps of a llama-shaped MLP slice (3 up/down blocks + the
32000-class head, batch 4096/worker, 4 workers, local Adam) for an ncu
launch list: which kernels the step's time goes to."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2502_11058_b200.lab import enp, sync_mask  # noqa: E402
from paper_2502_11058_b200.nn import Mlp, batch_pool, init_params  # noqa: E402

widths = [2048] + [5632, 2048] * 3 + [32000]
K, B, H = 4, 4096, 4
m = Mlp(widths, B, K, dtype="bf16", optimizer="adam", eps=1e-6)
init = init_params(1, widths)
for k in range(K):
    m.set_params(k, init)
xs, ys = batch_pool(1, list(range(K)), 1, B, widths[0], widths[-1], 0)
dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
m.set_batch_ptr(dx[0].data_ptr(), dy[0].data_ptr(), True)
L = len(widths) - 1
masks = [sync_mask("partial", H, r, L, enp(L, H)) for r in range(H)]
for r in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    m.step(1e-3, r, masks[r % H])
m.sync()
print("ok")
