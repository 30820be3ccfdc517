import torch, time
n = 1 << 28  # 268M floats = 1.07 GB
h_in = torch.empty(n, dtype=torch.float32).pin_memory(); h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, dtype=torch.float32, device='cuda'); d_out = torch.empty(n, dtype=torch.float32, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); return (time.perf_counter()-a)*1e3
for _ in range(2):
    h2d = t(lambda: d_in.copy_(h_in, non_blocking=True))
    d2h = t(lambda: h_out.copy_(d_out, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    bi = t(both)
print(f"H2D {h2d:.1f} ms ({4*n/h2d/1e6:.1f} GB/s)  D2H {d2h:.1f} ms ({4*n/d2h/1e6:.1f} GB/s)  both {bi:.1f} ms")
