import torch, time
n = 3623878656 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - t0
for _ in range(2):
    a = t(lambda: d.copy_(h, non_blocking=True))
    b = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    c = t(both)
print("H2D %.1f GB/s  D2H %.1f GB/s  both %.1f ms (%.1f GB/s each)" % (n*8/a/1e9, n*8/b/1e9, c*1e3, n*8/c/1e9))
