import torch, time
h = torch.empty(41_000_000 // 4, dtype=torch.float32).pin_memory()
d = torch.empty_like(h, device="cuda")
g = torch.empty(28_000_000 // 4, dtype=torch.float32, device="cuda")
hg = torch.empty_like(g, device="cpu").pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, n=20):
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/n
def h2d():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
def d2h():
    with torch.cuda.stream(s2): hg.copy_(g, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): hg.copy_(g, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for f in (h2d, d2h, both): t(f, 3)
a, b, c = t(h2d), t(d2h), t(both)
print(f"H2D 41MB {a:.3f} ms ({41/a:.1f} GB/s); D2H 28MB {b:.3f} ms ({28/b:.1f} GB/s); both {c:.3f} ms")
