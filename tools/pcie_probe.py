"""PCIe probe: H2D, D2H and concurrent bidirectional pinned copies (GB/s)."""
import torch, time
n = 748_150_080 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
b = n * 8
th = t(lambda: d.copy_(h, non_blocking=True))
td = t(lambda: h.copy_(d, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
tb = t(both)
print(f"h2d {b/th/1e9:.1f} GB/s  d2h {b/td/1e9:.1f} GB/s  both {b/tb/1e9:.1f} GB/s per direction ({tb*1e3:.2f} ms)")
