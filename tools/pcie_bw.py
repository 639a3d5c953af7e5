import torch, time
n = 2 << 30
d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
h = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
for _ in range(2): h.copy_(d, non_blocking=True); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): h.copy_(d, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("D2H single stream GB/s", 5 * n / e0.elapsed_time(e1) / 1e6)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
half = n // 16
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): h[:half].copy_(d[:half], non_blocking=True)
    with torch.cuda.stream(s2): h[half:].copy_(d[half:], non_blocking=True)
torch.cuda.synchronize()
print("D2H two streams GB/s", 5 * n / (time.perf_counter() - t) / 1e9)
x = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
e0.record()
for _ in range(5): d.copy_(x, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("H2D GB/s", 5 * n / e0.elapsed_time(e1) / 1e6)
