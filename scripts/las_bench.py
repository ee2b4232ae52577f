"""LAS ingestion throughput: device decode of a
20M-point image, device-resident (kernel roofline) and host -> host (e2e),
beside the CPU restatement and the reference's read_las. Prints one JSON
line; evidence for DESIGN.md / profiles/, not the driver's bench."""
import ctypes
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle as orc  # noqa: E402
from paper_2502_11602_b200 import _native  # noqa: E402
from paper_2502_11602_b200 import cheesemap as cm  # noqa: E402
from test_las import make_las, rand_raw  # noqa: E402


def main():
    n, fmt = 20_000_000, 1
    raw = rand_raw(n, 7, lo=-(10 ** 8), hi=10 ** 8)
    img = make_las(raw, (0.001, 0.001, 0.0005), (4.5e5, 5.2e6, 10.0), fmt=fmt)
    rl = 28
    L = _native.lib()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    peak = float(peaks.get("hbm_gbs", 6542.1))
    dimg = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
    out = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    h = _native.LasHeaderC()

    def dev_run():
        cm._check(L.cm_las_decode(ctypes.c_void_p(dimg.data_ptr()), dimg.numel(),
                                  ctypes.c_void_p(out.data_ptr()), n, ctypes.byref(h), 0, None))

    for _ in range(3):
        dev_run()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(10):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev_run()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    alg = n * (rl + 24)
    # host -> host (pinned image in, pinned points out)
    himg = torch.frombuffer(bytearray(img), dtype=torch.uint8).pin_memory()
    hout = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    e2e = []
    for _ in range(3):
        t = time.perf_counter()
        cm._check(L.cm_las_decode(ctypes.c_void_p(himg.data_ptr()), himg.numel(),
                                  ctypes.c_void_p(hout.data_ptr()), n, ctypes.byref(h), 0, None))
        e2e.append((time.perf_counter() - t) * 1e3)
    # parity on the full image vs the restatement
    rc, _, _, oxyz = orc.las_read(img)
    exact = bool(rc == 0 and np.array_equal(out.cpu().numpy().view(np.uint64), oxyz.view(np.uint64)))
    # CPU: the restatement (in memory) and the reference read_las (file)
    t = time.perf_counter()
    orc.las_read(img)
    cpu_ms = (time.perf_counter() - t) * 1e3
    ref_ms = None
    if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libcheesemap_ref.so")):
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "b.las")
            with open(p, "wb") as f:
                f.write(img)
            t = time.perf_counter()
            orc.las_read(path=p, which="reference")
            ref_ms = (time.perf_counter() - t) * 1e3
    print(json.dumps({
        "workload": f"LAS 1.2 format {fmt}, {n} points ({len(img) / 1e9:.2f} GB image)",
        "device_ms": round(ms, 3), "points_per_s": n / (ms * 1e-3),
        "roofline": {"bound": "hbm", "achieved": round(alg / (ms * 1e-3) / 1e9, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(alg / (ms * 1e-3) / 1e9 / peak, 3),
                     "basis": f"{rl} B record read + 24 B point written per point"},
        "e2e_host_to_host_ms": round(float(np.median(e2e)), 2),
        "e2e_points_per_s": n / (float(np.median(e2e)) * 1e-3),
        "cpu_restatement_ms": round(cpu_ms, 1), "cpu_reference_read_las_ms":
            None if ref_ms is None else round(ref_ms, 1),
        "bit_exact_vs_restatement": exact}))


if __name__ == "__main__":
    main()
