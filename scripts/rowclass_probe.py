"""Row-length classes of config 1 at large radii (the wide-FILL sort plan)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_11602_b200 import _native, synth  # noqa: E402
from paper_2502_11602_b200 import cheesemap as cm  # noqa: E402

L = _native.lib()
cloud = synth.config_cloud(1)
m = cm.Cheesemap.build(torch.from_numpy(cloud).cuda(), cm.BuildOptions(flavor=cm.Flavor.Mixed))
qd = torch.from_numpy(np.ascontiguousarray(cloud)).cuda()
for kern, r, frac in ((0, 2.5, 1), (1, 2.5, 1), (0, 5.0, 10), (1, 5.0, 10)):
    q = qd[: qd.shape[0] // frac]
    nq = q.shape[0]
    cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
    cm._check(L.cm_radius_count(m.handle, ctypes.c_void_p(q.data_ptr()), nq, kern, r,
                                ctypes.c_void_p(cnt.data_ptr()), None, None))
    c = cnt.to(torch.int64)
    cls = [int(((c > lo) & (c <= hi)).sum()) for lo, hi in ((0, 96), (96, 256), (256, 512), (512, 1024), (1024, 8192), (8192, 1 << 40))]
    sel = c[(c > 512) & (c <= 1024)]
    print(f"  (512,1024] mean {sel.float().mean().item():.0f}")
    print(f"kernel={kern} r={r} nq={nq} mean={c.float().mean().item():.0f} classes(<=96,..256,..512,..1024,..8192,>8192)={cls}", flush=True)
