"""H2D rate of a 1.2 MB pinned payload measured by a tiny C library from inside Python:
before torch is imported, after torch initialises CUDA, and with torch's own copy_."""
import ctypes, os, sys, time
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "h2dlib.so"))
lib.h2d_us.restype = ctypes.c_float
print("C lib, before torch:", lib.h2d_us(0))
import torch
torch.cuda.init(); x = torch.ones(1, device="cuda")
print("C lib, after torch CUDA init:", lib.h2d_us(0))
print("torch threads", torch.get_num_threads())
hp = torch.ones(1228800 // 4).pin_memory(); d = torch.empty_like(hp, device="cuda")
def t(fn, n=200):
    for _ in range(5): fn()
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / n * 1e3
print("torch copy_ pinned:", t(lambda: d.copy_(hp, non_blocking=True)))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    print("torch copy_ pinned, side stream:", t(lambda: d.copy_(hp, non_blocking=True)))
torch.set_num_threads(1)
print("torch copy_ pinned, 1 thread:", t(lambda: d.copy_(hp, non_blocking=True)))
print("C lib again:", lib.h2d_us(0))
