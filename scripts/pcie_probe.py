import torch, time
n = 128 * 2**20 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
for mode in ("h2d", "d2h", "both"):
    t = time.perf_counter()
    for _ in range(10):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 10
    print(mode, "%.3f ms per 128 MiB" % (dt * 1e3), "%.1f GB/s" % (128 * 2**20 / dt / 1e9))
