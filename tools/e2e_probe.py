#!/usr/bin/env python
"""Diagnose the e2e (host-buffer) leg: raw pinned copy rates, host time per call, device time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_00876_b200 as tsb  # noqa: E402
import tsgen  # noqa: E402

dev = torch.device("cuda:0")
if len(sys.argv) > 2 and sys.argv[2] == "numa":
    bus = torch.cuda.get_device_properties(dev).pci_bus_id.lower()
    base = f"/sys/bus/pci/devices/{bus}"
    if not os.path.exists(base):
        base = f"/sys/bus/pci/devices/0000:{bus.split(':', 1)[-1]}"
    print("pci", bus, "numa_node", open(base + "/numa_node").read().strip(),
          "local_cpulist", open(base + "/local_cpulist").read().strip())
    cpus = set()
    for part in open(base + "/local_cpulist").read().strip().split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    cpus &= os.sched_getaffinity(0)
    if cpus:
        os.sched_setaffinity(0, cpus)
        print("bound to", len(cpus), "cpus")
cfg = tsgen.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
B, N, C, E = cfg.B, cfg.N, cfg.C, cfg.E
nbytes = B * E * C * C * 4
hp = torch.from_numpy(tsgen.config_potentials(cfg)).pin_memory()
hm = torch.empty_like(hp).pin_memory()
d = torch.empty_like(hp, device=dev)
s = torch.cuda.current_stream()


def ev_time(fn, n=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    th = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3, th


print(f"bytes {nbytes}")
us, th = ev_time(lambda: d.copy_(hp, non_blocking=True))
print(f"H2D {us:.1f} us ({nbytes / us / 1e3:.1f} GB/s), host {th:.1f} us")
us, th = ev_time(lambda: hm.copy_(d, non_blocking=True))
print(f"D2H {us:.1f} us ({nbytes / us / 1e3:.1f} GB/s), host {th:.1f} us")
s2 = torch.cuda.Stream()


def both():
    d.copy_(hp, non_blocking=True)
    with torch.cuda.stream(s2):
        hm.copy_(d, non_blocking=True)


us, th = ev_time(both)
print(f"H2D||D2H (2 streams) {us:.1f} us, host {th:.1f} us")
hl = torch.empty(B, dtype=torch.float32).pin_memory()
hf = torch.empty(B, dtype=torch.int32).pin_memory()
ws = tsb.Workspace(dev)
hp2 = tsb.host_empty(tuple(hp.shape))
hp2.copy_(hp)
hm2 = tsb.host_empty(tuple(hp.shape))
us, th = ev_time(lambda: d.copy_(hp2, non_blocking=True))
print(f"H2D from ts_host_alloc buffer {us:.1f} us ({nbytes / us / 1e3:.1f} GB/s)")
for g in (True, False):
    tsb.set_host_graphs(g)
    us, th = ev_time(lambda: tsb.marginals_host(hp2, hm2, hl, hf, device=dev, ws=ws))
    print(f"host_empty buffers: marginals_host graphs={g}: device {us:.1f} us/call, "
          f"host enqueue {th:.1f} us/call")
for g in (True, False):
    tsb.set_host_graphs(g)
    us, th = ev_time(lambda: tsb.marginals_host(hp, hm, hl, hf, device=dev, ws=ws))
    print(f"marginals_host graphs={g}: device {us:.1f} us/call, host enqueue {th:.1f} us/call")
tsb.set_host_graphs(True)

# --- H2D rate vs host allocation strategy -------------------------------------------------
import ctypes  # noqa: E402
import mmap  # noqa: E402

libc = ctypes.CDLL("libc.so.6", use_errno=True)
cr = torch.cuda.cudart()


def h2d_rate(ptr, label):
    src = (ctypes.c_uint8 * nbytes).from_address(ptr)
    t = torch.frombuffer(src, dtype=torch.uint8, count=nbytes)
    t.fill_(1)
    dd = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    us, _ = ev_time(lambda: dd.copy_(t, non_blocking=True))
    print(f"{label}: H2D {us:.1f} us ({nbytes / us / 1e3:.1f} GB/s)")


big = tsb._lib.load().ts_host_alloc(256 << 20)
h2d_rate(big, "slice of a 256 MB ts_host_alloc block")
h2d_rate(big + (128 << 20), "slice at +128 MB of that block")
for adv in (14, None):  # MADV_HUGEPAGE = 14
    sz = 64 << 20
    libc.mmap.restype = ctypes.c_void_p
    libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                          ctypes.c_long]
    p = libc.mmap(None, sz + (2 << 20), 3, 0x22, -1, 0)  # PROT_RW, MAP_PRIVATE|ANON
    p = (p + (2 << 20) - 1) & ~((2 << 20) - 1)
    if adv is not None:
        print("madvise", libc.madvise(ctypes.c_void_p(p), ctypes.c_size_t(sz), adv))
    ctypes.memset(p, 1, sz)
    r = cr.cudaHostRegister(p, sz, 0)
    print("cudaHostRegister", r)
    h2d_rate(p, f"mmap 64 MB madvise={adv} + cudaHostRegister")
try:
    print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
    print(open("/proc/meminfo").read().split("HugePages_Total")[1][:60])
except Exception as e:  # noqa: BLE001
    print(e)
