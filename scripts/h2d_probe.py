"""Pinned host<->device copy bandwidth on this box (context for bench.py's e2e)."""
import time
import torch

n = 1_649_184_128 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"{name} {n * 4 / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms for {n * 4 / 1e9:.2f} GB)")
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print(f"h2d+d2h concurrent {2 * n * 4 / dt / 1e9:.1f} GB/s total")

# does a kernel on another stream wait for a bulk H2D copy in flight?
cs = torch.cuda.Stream()
x = torch.randn(4096, 4096, device="cuda")
torch.cuda.synchronize()
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
c0, c1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
c0.record(cs)
with torch.cuda.stream(cs):
    d.copy_(h, non_blocking=True)
c1.record(cs)
e0.record()
for _ in range(20):
    x = x @ x.T * 1e-3
e1.record()
torch.cuda.synchronize()
print(f"copy stream: copy {c0.elapsed_time(c1):.1f} ms; main stream: matmuls start +{c0.elapsed_time(e0):.2f} ms, "
      f"take {e0.elapsed_time(e1):.2f} ms")
