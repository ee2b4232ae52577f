"""e2e chunk-plan probe: cm_radius_search_to_host on config 1 (r = 1 m) for
several chunk weightings (CMGPU_CHUNK_W), best of 3 each."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_11602_b200 import _native, synth  # noqa: E402
from paper_2502_11602_b200 import cheesemap as cm  # noqa: E402

cloud = synth.config_cloud(1)
m = cm.Cheesemap.build(torch.from_numpy(cloud).cuda(), cm.BuildOptions(flavor=cm.Flavor.Mixed))
L = _native.lib()
qh = torch.from_numpy(cloud).pin_memory()
row = torch.empty(cloud.shape[0] + 1, dtype=torch.int64).pin_memory()
cols = torch.empty(900_000_000, dtype=torch.int32).pin_memory()
nnz = ctypes.c_uint64()
plans = sys.argv[1:] or ["", "1,2,2,2", "1,2,4,4,4", "1,3,4,4,4", "1,2,3,4,4,4", "1,1,2,4,4,4"]
for plan in plans:
    if plan:
        os.environ["CMGPU_CHUNK_W"] = plan
    else:
        os.environ.pop("CMGPU_CHUNK_W", None)
    best = 1e30
    for _ in range(4):
        torch.cuda.synchronize()
        t = time.perf_counter()
        rc = L.cm_radius_search_to_host(m.handle, ctypes.c_void_p(qh.data_ptr()), cloud.shape[0], 0,
                                        1.0, ctypes.c_void_p(row.data_ptr()),
                                        ctypes.c_void_p(cols.data_ptr()), cols.numel(),
                                        ctypes.byref(nnz), None)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
        assert rc == 0
    print(f"plan [{plan or 'default'}]: {best * 1e3:.1f} ms  nnz={nnz.value}", flush=True)
