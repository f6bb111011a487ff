import torch, time
n = 201326592 // 8
d = torch.empty(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64).pin_memory()
hu = torch.empty(134217728 // 8, dtype=torch.float64).pin_memory()
du = torch.empty(134217728 // 8, dtype=torch.float64, device="cuda")
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
def t(f, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3
print("d2h 1D 201MB ms", t(lambda: h.copy_(d, non_blocking=True)))
print("h2d 1D 134MB ms", t(lambda: du.copy_(hu, non_blocking=True)))
def both():
    with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2): du.copy_(hu, non_blocking=True)
print("both concurrent ms", t(both))
# 2-D strided D2H: 16 chunks each 512 rows x 16KB at pitch 32KB (like the pipeline)
dv = d[: 16777216]
hv = h[: 16777216]
def d2h_2d():
    for p in range(16):
        o = p * (16777216 // 16)
        # emulate with a strided view copy: rows of 2048 doubles at pitch 4096
        src = dv[o:o + 16777216 // 16].view(512, 2048)
        hv[o:o + 16777216 // 16].view(512, 2048).copy_(src, non_blocking=True)
print("d2h 16 pieces 134MB ms", t(d2h_2d))
