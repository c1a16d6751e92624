import torch, time
n = 839 * 2**20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device='cuda'); d2 = torch.empty(n, dtype=torch.uint8, device='cuda')
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
def t(f, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - a)
    return best
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both(): h2d(); d2h()
for name, f in [("h2d", h2d), ("d2h", d2h), ("both", both)]:
    s = t(f); print(name, f"{s*1e3:.2f} ms", f"{n/s/1e9:.1f} GB/s per direction")
