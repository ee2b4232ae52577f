"""D2H rate into torch-pinned memory vs an mmap'd, THP-advised,
cudaHostRegister'ed buffer (fewer, larger pages for the DMA mappings)."""
import mmap
import time

import numpy as np
import torch

print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
nb = 3_500_000_000
d = torch.empty(nb // 4, dtype=torch.int32, device="cuda")


def thp_registered(nbytes):
    al = 2 << 20
    size = (nbytes + al - 1) // al * al
    m = mmap.mmap(-1, size + al, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    try:
        m.madvise(mmap.MADV_HUGEPAGE)
    except Exception as e:  # noqa: BLE001
        print("madvise failed", e)
    a = np.frombuffer(m, dtype=np.uint8)
    off = (-a.ctypes.data) % al
    a = a[off:off + size]
    a[::4096] = 0
    rc = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, size, 0)
    print("register rc", rc)
    return m, torch.from_numpy(a[:nbytes].view(np.int32))


def rate(h, tag):
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        h.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"{tag}: {dt * 1e3:.1f} ms {nb / dt / 1e9:.1f} GB/s", flush=True)


t0 = time.perf_counter()
hp = torch.empty(nb // 4, dtype=torch.int32).pin_memory()
print(f"pin_memory alloc {time.perf_counter() - t0:.2f} s")
rate(hp, "torch pinned")
t0 = time.perf_counter()
keep, ht = thp_registered(nb)
print(f"thp+register alloc {time.perf_counter() - t0:.2f} s")
rate(ht, "thp registered")
with open("/proc/meminfo") as f:
    print([l.strip() for l in f if "Huge" in l or "MemFree" in l])
