"""D2H of 134 MB (a b/m3/exp1 V) into pageable vs pinned host memory."""
import time

import numpy as np
import torch

n = 16777216
d = torch.randn(n, dtype=torch.float64, device="cuda")
pin = torch.empty(n, dtype=torch.float64).pin_memory()
pg = torch.from_numpy(np.zeros(n))  # touched pageable
for name, h in [("pinned", pin), ("pageable", pg)]:
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        t = time.perf_counter()
        h.copy_(d)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"{name}: {best * 1e3:.2f} ms, {n * 8 / best / 1e9:.1f} GB/s")
# host memcpy pinned -> pageable, 1 and 8 threads
import threading
src = pin.numpy(); dst = pg.numpy()
for nt in (1, 4, 8, 16):
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        ths = []
        ch = n // nt
        for k in range(nt):
            th = threading.Thread(target=lambda k=k: np.copyto(dst[k * ch:(k + 1) * ch], src[k * ch:(k + 1) * ch]))
            th.start(); ths.append(th)
        for th in ths:
            th.join()
        best = min(best, time.perf_counter() - t)
    print(f"host memcpy {nt} threads: {best * 1e3:.2f} ms, {n * 8 / best / 1e9:.1f} GB/s")
