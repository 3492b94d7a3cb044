import torch, time
n = 2_784_704_044
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
o = torch.empty(740_000_000, dtype=torch.uint8, pin_memory=True)
do = torch.empty(740_000_000, dtype=torch.uint8, device="cuda")
for it in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"H2D {n/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms)")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for it in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): o.copy_(do, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"H2D+D2H concurrent {dt*1e3:.1f} ms")
