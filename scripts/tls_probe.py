"""TLS (config 2) digest probe: rate and tile statistics per radius."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import numpy as np
import torch
from paper_2502_11602_b200 import cheesemap as cm, synth, _native
cloud = synth.config_cloud(2)
q = synth.config_queries(2, cloud)
m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Mixed, cell=cm.CellSize.uniform(0.25)))
L = _native.lib()
qd = torch.from_numpy(np.ascontiguousarray(q)).cuda()
nq = qd.shape[0]
cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
dig = torch.empty(nq, dtype=torch.int64, device="cuda")
tested = torch.zeros(nq, dtype=torch.int64, device="cuda")
for r in (0.05, 0.1, 0.25):
    for rep in range(2):
        _native.query_stats(reset=True)
        torch.cuda.synchronize(); t = time.perf_counter()
        cm._check(L.cm_radius_digest(m.handle, ctypes.c_void_p(qd.data_ptr()), nq, 0, r,
                                     ctypes.c_void_p(cnt.data_ptr()), ctypes.c_void_p(dig.data_ptr()), None))
        torch.cuda.synchronize(); ms = (time.perf_counter() - t) * 1e3
    st = _native.query_stats()
    cm._check(L.cm_radius_count(m.handle, ctypes.c_void_p(qd.data_ptr()), nq, 0, r, None,
                                ctypes.c_void_p(tested.data_ptr()), None))
    tt = tested.cpu().numpy()
    c = cnt.cpu().numpy()
    print(f"r={r}: {ms:.1f} ms {nq/ms/1e3:.2f} M q/s  hits/q {c.mean():.0f} max {c.max()} tested/q {tt.mean():.0f} p99 {np.percentile(tt,99):.0f} max {tt.max()} stats {st}", flush=True)
