"""Host-link probe: concurrent bidirectional pinned copies (748 MB each way,
the headline e2e step's bytes) on 1, 2 and 4 GPUs at once, one host thread
per GPU.  Prints per-direction GB/s aggregated over the GPUs — the bound of
bench.py's e2e (host state in, host state out every step)."""
import json
import threading
import time

import torch

B = 748_150_080
n = B // 8


def setup(dev):
    torch.cuda.set_device(dev)
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    h2 = torch.empty(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device=f"cuda:{dev}")
    d2 = torch.empty(n, dtype=torch.float64, device=f"cuda:{dev}")
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    return h, h2, d, d2, s1, s2


def run(bufs, reps, res, i, barrier, mode):
    h, h2, d, d2, s1, s2 = bufs
    torch.cuda.set_device(d.device)
    barrier.wait()
    t0 = time.perf_counter()
    for _ in range(reps):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    s1.synchronize()
    s2.synchronize()
    res[i] = time.perf_counter() - t0


out = {}
ng = torch.cuda.device_count()
allbufs = [setup(g) for g in range(ng)]
for k in [g for g in (1, 2, 4, 8) if g <= ng]:
    for mode in ("h2d", "d2h", "both"):
        reps = 4
        for warm in (True, False):
            res = [0.0] * k
            bar = threading.Barrier(k)
            th = [threading.Thread(target=run, args=(allbufs[g], 1 if warm else reps, res, g, bar, mode)) for g in range(k)]
            [t.start() for t in th]
            [t.join() for t in th]
        out[f"{k}gpu_{mode}_GBps_per_direction"] = round(k * reps * B / max(res) / 1e9, 1)
print(json.dumps(out))
