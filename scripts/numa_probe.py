"""Host<->device copy rate vs the process's CPU affinity (GPU-local NUMA node
or not): pinned buffers are first-touched on the node the process runs on."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
import pynvml  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
local = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
print("gpu-local cpus", len(local), local[:4], "...")
mode = sys.argv[1] if len(sys.argv) > 1 else "default"
if mode == "local":
    os.sched_setaffinity(0, local)
elif mode == "remote":
    other = sorted(set(range(os.cpu_count())) - set(local))
    if other:
        os.sched_setaffinity(0, other)
import torch  # noqa: E402

n = 3_500_000_000 // 4
d = torch.empty(n, dtype=torch.int32, device="cuda")
hbuf = torch.empty(n, dtype=torch.int32).pin_memory()
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    hbuf.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"[{mode}] D2H 3.5 GB {dt * 1e3:.1f} ms {3.5 / dt:.1f} GB/s", flush=True)
