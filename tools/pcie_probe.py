import torch, time
n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for it in range(3):
    torch.cuda.synchronize(); t = time.time()
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    torch.cuda.synchronize(); h2d = n / (time.time() - t) / 1e9
    t = time.time()
    with torch.cuda.stream(s1): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); d2h = n / (time.time() - t) / 1e9
    t = time.time()
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); both = 2 * n / (time.time() - t) / 1e9
    print("H2D %.1f GB/s  D2H %.1f GB/s  concurrent total %.1f GB/s" % (h2d, d2h, both))
