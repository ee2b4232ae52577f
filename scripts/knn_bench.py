"""Config-3 kNN timing + parity sample (A/B: run with CMGPU_KNN_LEGACY=1 for
the round-1 path). 20M-point config-1 cloud, mixed index, 5M centres from the
CenterStream, k in {8, 16, 32, 64}. Roofline: 24 B x
points_tested of kernel_search at the exact k-th distance, estimated from
the oracle on a sample."""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import CpuIndex  # noqa: E402
from paper_2502_11602_b200 import _native, synth  # noqa: E402
from paper_2502_11602_b200 import cheesemap as cm  # noqa: E402


def main():
    ks = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8,16,32,64").split(",")]
    sample = int(os.environ.get("KNN_SAMPLE", "200000"))
    total = torch.cuda.get_device_properties(0).total_memory
    cm.pool_configure(0, int(total * 0.75), 0)
    cloud = synth.config_cloud(3)
    q = synth.config_queries(3, cloud)
    dc = torch.from_numpy(cloud).cuda()
    qd = torch.from_numpy(q).cuda()
    m = cm.Cheesemap.build(dc, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    L = _native.lib()
    o = CpuIndex(cloud, flavor=1)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6546.0
    out = []
    nq = q.shape[0]
    for k in ks:
        idx = torch.empty((nq, k), dtype=torch.int32, device="cuda")
        d2 = torch.empty((nq, k), dtype=torch.float64, device="cuda")

        def run():
            cm._check(L.cm_knn(m.handle, ctypes.c_void_p(qd.data_ptr()), nq, k,
                               ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(d2.data_ptr()), None))
        run()
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        qs = np.ascontiguousarray(q[:sample])
        oi, od, prk, _ = o.knn(qs, k, stats=True)
        gi = idx[:sample].cpu().numpy().view(np.uint32)
        gd = d2[:sample].cpu().numpy()
        bad = int(np.count_nonzero(np.any((gi != oi) | (gd.view(np.int64) != od.view(np.int64)), axis=1)))
        alg = 24.0 * float(prk.mean()) * nq
        r = dict(k=k, ms=round(best, 3), qps=round(nq / (best * 1e-3), 1), mismatching_rows=bad,
                 checked=sample, frac=round(alg / (best * 1e-3) / (peak * 1e9), 4),
                 alg_gb=round(alg / 1e9, 2), legacy=bool(os.environ.get("CMGPU_KNN_LEGACY")))
        print(json.dumps(r), flush=True)
        out.append(r)


if __name__ == "__main__":
    main()
