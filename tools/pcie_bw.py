import torch, time
n = 200_000_000
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
d = torch.empty(n, dtype=torch.int32, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter() - t
t = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter() - t
print(f"H2D {0.8/t1:.1f} GB/s  D2H {0.8/t2:.1f} GB/s")
s = torch.cuda.Stream()
t = time.perf_counter()
with torch.cuda.stream(s): d.copy_(h, non_blocking=True)
h2 = torch.empty(n, dtype=torch.int32, pin_memory=True); d2 = torch.zeros(n, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s): d.copy_(h, non_blocking=True)
h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); t3 = time.perf_counter() - t
print(f"bidirectional 1.6 GB in {t3*1e3:.1f} ms = {1.6/t3:.1f} GB/s")
