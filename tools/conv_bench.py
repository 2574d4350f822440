"""Time the implicit-GEMM conv kernels against a plain GEMM of the same
M x N x K (explicit im2col operand) and epilogue variants (CUDA events)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_11058_b200 import native as N  # noqa: E402
from paper_2502_11058_b200.nn import gemm  # noqa: E402

dev = torch.device("cuda:0")


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(H, B, cin, cout, nb=8):
    P = B * H * H
    x = torch.randn(nb, P, cin, device=dev).bfloat16()
    w = torch.randn(nb, cout, 9 * cin, device=dev).bfloat16()
    col = torch.randn(nb, P, 9 * cin, device=dev).bfloat16()
    dy = torch.randn(nb, P, cout, device=dev).bfloat16()
    bias = torch.randn(nb, cout, device=dev)
    y = torch.empty(nb, P, cout, device=dev, dtype=torch.bfloat16)
    yf = torch.empty(nb, P, cout, device=dev)
    dx = torch.empty(nb, P, cin, device=dev, dtype=torch.bfloat16)
    mask = torch.randn(nb, P, cin, device=dev).bfloat16()
    dw = torch.empty(nb, cout, 9 * cin, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    flops = 2.0 * P * cout * 9 * cin * nb
    geo = (H, H, B, cin, cout)
    res = {"shape": [H, B, cin, cout, nb], "gflop": flops / 1e9}
    kw = dict(batch=nb, stream=s)
    variants = {
        "fwd_bias_relu": lambda: gemm(x, w, y, M=0, N_=0, K=0, lda=cin, sA=P * cin, ldb=9 * cin, sB=cout * 9 * cin,
                                      ldc=cout, sC=P * cout, epi=1, relu=True, bias=bias, s_bias=cout,
                                      conv=(1,) + geo, **kw),
        "fwd_nobias": lambda: gemm(x, w, y, M=0, N_=0, K=0, lda=cin, sA=P * cin, ldb=9 * cin, sB=cout * 9 * cin,
                                   ldc=cout, sC=P * cout, epi=1, conv=(1,) + geo, **kw),
        "fwd_f32out": lambda: gemm(x, w, yf, M=0, N_=0, K=0, lda=cin, sA=P * cin, ldb=9 * cin, sB=cout * 9 * cin,
                                   ldc=cout, sC=P * cout, epi=0, conv=(1,) + geo, **kw),
        "plain_gemm_same_shape": lambda: gemm(col, w, y, M=P, N_=cout, K=9 * cin, lda=9 * cin, sA=P * 9 * cin,
                                              ldb=9 * cin, sB=cout * 9 * cin, ldc=cout, sC=P * cout, epi=1,
                                              relu=True, bias=bias, s_bias=cout, **kw),
        "dgrad_drelu": lambda: gemm(dy, w, dx, M=0, N_=0, K=0, b_mn=True, lda=cout, sA=P * cout, ldb=9 * cin,
                                    sB=cout * 9 * cin, ldc=cin, sC=P * cin, epi=2, mask=mask, ldmask=cin,
                                    s_mask=P * cin, conv=(3,) + geo, **kw),
        "dgrad_plain_epi": lambda: gemm(dy, w, dx, M=0, N_=0, K=0, b_mn=True, lda=cout, sA=P * cout, ldb=9 * cin,
                                        sB=cout * 9 * cin, ldc=cin, sC=P * cin, epi=1, conv=(3,) + geo, **kw),
        "wgrad": lambda: gemm(dy, x, dw, M=0, N_=0, K=0, a_mn=True, b_mn=True, lda=cout, sA=P * cout, ldb=cin,
                              sB=P * cin, ldc=9 * cin, sC=cout * 9 * cin, conv=(2,) + geo, **kw),
    }
    dwt = torch.empty(4, nb, 9 * cin, cout, device=dev)
    variants["wgradT_ks4"] = lambda: gemm(x, dy, dwt, M=0, N_=0, K=0, a_mn=True, b_mn=True, lda=cin, sA=P * cin,
                                          ldb=cout, sB=P * cout, ldc=cout, sC=9 * cin * cout, ksplit=4,
                                          s_split=nb * 9 * cin * cout, bn=64, conv=(4,) + geo, **kw)
    for bn in (64, 128, 256):
        if bn <= cout or bn == 64:
            variants[f"fwd_bn{bn}"] = (lambda bn=bn: gemm(
                x, w, y, M=0, N_=0, K=0, lda=cin, sA=P * cin, ldb=9 * cin, sB=cout * 9 * cin, ldc=cout,
                sC=P * cout, epi=1, relu=True, bias=bias, s_bias=cout, conv=(1,) + geo, bn=bn, **kw))
    for k, f in variants.items():
        ms = timeit(f)
        res[k] = {"ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 1)}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    run(32, 128, 64, 64)
    run(16, 128, 128, 128)
    run(8, 128, 256, 256)
    run(4, 128, 512, 512)
