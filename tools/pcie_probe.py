import torch, time
d = torch.device("cuda:0")
h_in = torch.empty(217_000_000 // 8, dtype=torch.float64).pin_memory()
h_out = torch.empty(254_000_000 // 8, dtype=torch.float64).pin_memory()
d_in = torch.empty_like(h_in, device=d); d_out = torch.empty_like(h_out, device=d)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, n=5):
    f(); torch.cuda.synchronize()
    w = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - w) / n * 1e3
def h2d():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
def both(): h2d(); d2h()
print("h2d 217MB ms", t(h2d), "d2h 254MB ms", t(d2h), "both ms", t(both))
