"""Probe host<->device copy rates and the host-buffer search pipeline."""
import ctypes
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2502_11602_b200 import _native, synth
from paper_2502_11602_b200 import cheesemap as cm

cloud = synth.config_cloud(1)
m = cm.Cheesemap.build(torch.from_numpy(cloud).cuda(), cm.BuildOptions(flavor=cm.Flavor.Mixed))
L = _native.lib()
nbytes = 3_500_000_000
d = torch.empty(nbytes // 4, dtype=torch.int32, device="cuda")
h = torch.empty(nbytes // 4, dtype=torch.int32).pin_memory()
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    print(f"D2H {nbytes/1e9:.1f} GB: {(time.perf_counter()-t)*1e3:.1f} ms", flush=True)
    t = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    print(f"H2D {nbytes/1e9:.1f} GB: {(time.perf_counter()-t)*1e3:.1f} ms", flush=True)
del d, h
qh = torch.from_numpy(cloud).pin_memory()
row = torch.empty(cloud.shape[0] + 1, dtype=torch.int64).pin_memory()
cols = torch.empty(900_000_000, dtype=torch.int32).pin_memory()
nnz = ctypes.c_uint64()
for i in range(4):
    torch.cuda.synchronize(); t = time.perf_counter()
    rc = L.cm_radius_search_to_host(m.handle, ctypes.c_void_p(qh.data_ptr()), cloud.shape[0], 0, 1.0,
                                    ctypes.c_void_p(row.data_ptr()), ctypes.c_void_p(cols.data_ptr()),
                                    cols.numel(), ctypes.byref(nnz), None)
    torch.cuda.synchronize()
    print(f"to_host rc={rc} nnz={nnz.value} {(time.perf_counter()-t)*1e3:.1f} ms", flush=True)
qd = torch.from_numpy(cloud).cuda()
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    csr = ctypes.c_void_p()
    L.cm_radius_search(m.handle, ctypes.c_void_p(qd.data_ptr()), cloud.shape[0], 0, 1.0, None, ctypes.byref(csr))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    L.cm_csr_download(csr, ctypes.c_void_p(row.data_ptr()), ctypes.c_void_p(cols.data_ptr()), None)
    t2 = time.perf_counter()
    L.cm_csr_free(csr)
    print(f"device search {(t1-t)*1e3:.1f} ms, download {(t2-t1)*1e3:.1f} ms", flush=True)
print("pool (reserved, in use) bytes:", _native.pool_bytes(0), flush=True)
