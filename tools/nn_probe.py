import sys, numpy as np
sys.path.insert(0, '.')
from tests.test_gpu_nn import _run_pair
widths = [256]*8+[10]
for opt, lr, eps in [("adam", 1e-3, 1e-6), ("momentum", 0.01, 1e-8)]:
    for steps in (1, 2, 8):
        got, orc, losses = _run_pair(widths, 4, 4, steps, opt, lr, eps=eps)
        o = orc.offsets
        row = []
        for l in range(8):
            i, n = widths[l], widths[l+1]
            W = slice(o[l], o[l]+i*n); B = slice(o[l]+i*n, o[l+1])
            eW = np.linalg.norm(got[0][W]-orc.w[0][W])/np.linalg.norm(orc.w[0][W])
            db = np.abs(got[0][B]-orc.w[0][B]).max()
            row.append(f"L{l+1}:W{eW:.1e} bmax{db:.1e}")
        print(opt, steps, " ".join(row), flush=True)
