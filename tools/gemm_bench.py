"""tcgen05 GEMM throughput (dsx_gemm, bf16 in / fp32 accumulate) against
cuBLAS (torch.matmul) on the same shapes; CUDA events, after warm-up.
Shapes: the MLP layer GEMMs (configs[0], 4 workers batched) and large
square ones for the tensor-pipe roofline.  One JSON line per shape."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_11058_b200 import native as N  # noqa: E402
from paper_2502_11058_b200.nn import gemm  # noqa: E402


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dev = torch.device("cuda:0")
    shapes = [  # (name, M, N, K, batch, a_mn, b_mn)
        ("mlp_fwd", 256, 1024, 1024, 4, False, False),
        ("mlp_dgrad", 256, 1024, 1024, 4, False, True),
        ("mlp_wgrad", 1024, 1024, 256, 4, True, True),
        ("sq4096", 4096, 4096, 4096, 1, False, False),
        ("sq8192", 8192, 8192, 8192, 1, False, False),
        ("wide_fwd", 2048, 4096, 4096, 4, False, False),
        ("wide_dgrad", 2048, 4096, 4096, 4, False, True),
        ("wide_wgrad", 4096, 4096, 2048, 4, True, True),
    ]
    for name, M, Nn, K, b, am, bm in shapes:
        A = (torch.randn(b, K, M, device=dev) if am else torch.randn(b, M, K, device=dev)).bfloat16()
        B = (torch.randn(b, K, Nn, device=dev) if bm else torch.randn(b, Nn, K, device=dev)).bfloat16()
        C = torch.empty(b, M, Nn, device=dev)
        flops = 2.0 * M * Nn * K * b
        res = {"shape": name, "M": M, "N": Nn, "K": K, "batch": b, "a_mn": am, "b_mn": bm}
        for bn in (64, 128, 256):
            ms = timeit(lambda: gemm(A, B, C, M=M, N_=Nn, K=K, batch=b, a_mn=am, b_mn=bm, lda=M if am else K,
                                     sA=M * K, ldb=Nn if bm else K, sB=Nn * K, ldc=Nn, sC=M * Nn, bn=bn), 20)
            res[f"tc_bn{bn}_ms"] = round(ms, 4)
            res[f"tc_bn{bn}_tflops"] = round(flops / ms / 1e9, 1)
        Af = A.transpose(1, 2) if am else A
        Bf = B if bm else B.transpose(1, 2)
        ms = timeit(lambda: torch.bmm(Af, Bf, out=None), 20)
        res["cublas_ms"] = round(ms, 4)
        res["cublas_tflops"] = round(flops / ms / 1e9, 1)
        ref = torch.bmm(Af.float(), Bf.float())
        gemm(A, B, C, M=M, N_=Nn, K=K, batch=b, a_mn=am, b_mn=bm, lda=M if am else K, sA=M * K,
             ldb=Nn if bm else K, sB=Nn * K, ldc=Nn, sC=M * Nn)
        torch.cuda.synchronize()
        res["rel_err"] = float((C - ref).norm() / ref.norm())
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
