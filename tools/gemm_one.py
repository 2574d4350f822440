"""One tcgen05 GEMM shape, a few launches (for ncu): the wide MLP's forward
layer GEMM (M=2048 batch, N=K=4096, 4 workers batched), bf16 -> fp32."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_11058_b200.nn import gemm  # noqa: E402

dev = torch.device("cuda:0")
M, N, K, b = 2048, 4096, 4096, 4
A = torch.randn(b, M, K, device=dev).bfloat16()
B = torch.randn(b, N, K, device=dev).bfloat16()
C = torch.empty(b, M, N, device=dev)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    gemm(A, B, C, M=M, N_=N, K=K, batch=b, lda=K, sA=M * K, ldb=K, sB=N * K, ldc=N, sC=M * N, bn=256)
torch.cuda.synchronize()
print("ok")
