import torch, time, ctypes
n = 16777216
d = torch.empty(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64).pin_memory()
cud = ctypes.CDLL("libcudart.so")
s = torch.cuda.current_stream().cuda_stream
def run(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return best * 1e3
# 16 pieces of 1M doubles: 1-D contiguous vs 2-D (512 rows x 2048 doubles at pitch 4096)
per = n // 16
def one_d():
    for p in range(16):
        cud.cudaMemcpyAsync(ctypes.c_void_p(h.data_ptr() + p * per * 8), ctypes.c_void_p(d.data_ptr() + p * per * 8), ctypes.c_size_t(per * 8), 2, ctypes.c_void_p(s))
def two_d():
    for p in range(16):
        base = (p // 2) * 2 * per + (p % 2) * 2048
        cud.cudaMemcpy2DAsync(ctypes.c_void_p(h.data_ptr() + base * 8), ctypes.c_size_t(4096 * 8), ctypes.c_void_p(d.data_ptr() + base * 8), ctypes.c_size_t(4096 * 8), ctypes.c_size_t(2048 * 8), ctypes.c_size_t(512), 2, ctypes.c_void_p(s))
print("1-D 16 pieces ms", run(one_d), "GB/s", n * 8 / run(one_d) / 1e6)
print("2-D 16 pieces ms", run(two_d), "GB/s", n * 8 / run(two_d) / 1e6)
