"""Device-memory probe: repeated radius searches must not grow the library's
pool beyond what it caches (diagnostic for long sweeps)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_11602_b200 import cheesemap as cm, synth, _native
cloud = synth.config_cloud(1)
m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Mixed))
qd = torch.from_numpy(cloud).cuda()
import ctypes
L = _native.lib()
for r in (1.0, 2.5, 1.0, 2.5, 2.5):
    csr = ctypes.c_void_p()
    cm._check(L.cm_radius_search(m.handle, ctypes.c_void_p(qd.data_ptr()), qd.shape[0], 0, r, None, ctypes.byref(csr)))
    L.cm_csr_free(csr)
    torch.cuda.synchronize()
    fr, tot = torch.cuda.mem_get_info()
    res, used = _native.pool_bytes()
    print(f"r={r} free={fr/1e9:.1f} GB pool reserved={res/1e9:.1f} used={used/1e9:.2f} torch={torch.cuda.memory_reserved()/1e9:.1f}", flush=True)
res, used = _native.pool_bytes(trim=True)
fr, tot = torch.cuda.mem_get_info()
print(f"after trim: free={fr/1e9:.1f} pool reserved={res/1e9:.1f} used={used/1e9:.2f}")
