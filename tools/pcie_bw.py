import torch, time
n = 717 * 1024 * 1024 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory(); h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, device="cuda"); d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def t(f, k=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
b = n * 4
print("H2D GB/s", b / t(lambda: d.copy_(h, non_blocking=True)) / 1e9)
print("D2H GB/s", b / t(lambda: h2.copy_(d2, non_blocking=True)) / 1e9)
print("both GB/s each", b / t(both) / 1e9)
