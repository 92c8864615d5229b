import torch, time
n = 604 * 1024 * 1024 // 2
h_in = torch.empty(n, dtype=torch.bfloat16).pin_memory(); h_out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d_in = torch.empty(n, dtype=torch.bfloat16, device="cuda"); d_out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
def h2d():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
def both(): h2d(); d2h()
a, b, c = t(h2d), t(d2h), t(both)
gb = n * 2 / 1e9
print(f"H2D {a:.2f} ms ({gb/a*1e3:.1f} GB/s)  D2H {b:.2f} ms ({gb/b*1e3:.1f} GB/s)  both concurrently {c:.2f} ms")
