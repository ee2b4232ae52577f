"""Raw pinned host<->device copy bandwidth (the e2e path's ceiling)."""
import torch

for nbytes in (256 << 20, 1 << 30, 3300 << 20):
    d = torch.empty(nbytes // 4, dtype=torch.int32, device="cuda")
    h = torch.empty(nbytes // 4, dtype=torch.int32).pin_memory()
    for direction in ("d2h", "h2d"):
        for _ in range(2):
            (h.copy_(d, non_blocking=True) if direction == "d2h" else d.copy_(h, non_blocking=True))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            (h.copy_(d, non_blocking=True) if direction == "d2h" else d.copy_(h, non_blocking=True))
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{direction} {nbytes / 1e9:.2f} GB: {ms:.2f} ms = {nbytes / ms / 1e6:.1f} GB/s", flush=True)
    # both directions at once on two streams
    d2 = torch.empty_like(d)
    h2 = torch.empty_like(h).pin_memory()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    with torch.cuda.stream(s1):
        h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2):
        d2.copy_(h2, non_blocking=True)
    torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    print(f"duplex {nbytes / 1e9:.2f} GB each way: {e0.elapsed_time(e1):.2f} ms", flush=True)
