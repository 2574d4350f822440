"""One warm-up + one timed ResNet-18 conv-stack step (bench config
resnet18_cnn) for ncu launch lists; prints the CUDA-event step time."""
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from bench import cnn_init_host  # noqa: E402
from paper_2502_11058_b200.cnn import Cnn, batch, teacher  # noqa: E402
from paper_2502_11058_b200.lab import enp, sync_mask  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
m = Cnn(B, K, dtype="bf16")
init = cnn_init_host(1)
for k in range(K):
    m.set_params(k, init)
t = teacher(1, 32, 3, 10)
bs = [batch(1, k, 0, B, 32, 3, t) for k in range(K)]
x = torch.from_numpy(np.stack([b[0] for b in bs])).cuda()
y = torch.from_numpy(np.stack([b[1] for b in bs])).cuda()
m.set_batch_ptr(x.data_ptr(), y.data_ptr(), True)
sets = enp(m.L, 5)
m.step(0.01, 0, sync_mask("partial", 5, 0, m.L, sets))
m.sync()
m.record(0)
for r in range(steps):
    m.step(0.01, 1 + r, sync_mask("partial", 5, 1 + r, m.L, sets))
m.record(1)
print(f"ms/step {m.elapsed_ms(0, 1) / steps:.3f}  loss {m.last_loss()}")
