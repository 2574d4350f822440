import sys, numpy as np
sys.path.insert(0,'.')
from tests.test_gpu_nn import _run_pair
for eps in (1e-8, 1e-6):
    got, orc, _ = _run_pair([256]*8+[10], 4, 4, 8, "adam", 1e-3, eps=eps)
    for k in range(4):
        d = np.abs(got[k]-orc.w[k]); print(eps, k, np.linalg.norm(got[k]-orc.w[k])/np.linalg.norm(orc.w[k]), d.max(), (d>1e-4).sum())
