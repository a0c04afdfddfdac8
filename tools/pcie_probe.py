import torch, time
n = 7_500_000_000 // 8 // 4   # 1.9 GB chunks
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def bw(f, reps=3):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
b = n * 8
t = bw(lambda: d.copy_(h, non_blocking=True)); print("H2D GB/s", b / t / 1e9)
t = bw(lambda: h2.copy_(d2, non_blocking=True)); print("D2H GB/s", b / t / 1e9)
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
t = bw(both); print("H2D+D2H concurrent GB/s each", b / t / 1e9)
