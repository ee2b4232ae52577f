"""COUNT pass against the single-pass search on sparse centre sets (tile paths)."""
import sys, ctypes, numpy as np, torch
sys.path.insert(0,'.')
from paper_2502_11602_b200 import cheesemap as cm, synth, _native
for cfg, stride in ((0, 1), (1, 7), (1, 50)):
    cloud = synth.config_cloud(cfg)
    q = synth.config_queries(cfg, cloud) if cfg == 0 else np.ascontiguousarray(cloud[::stride])
    dc = torch.from_numpy(cloud).cuda(); qd = torch.from_numpy(q).cuda()
    m = cm.Cheesemap.build(dc, cm.BuildOptions(flavor=cm.Flavor.Mixed if cfg else cm.Flavor.Dense))
    cnt = torch.empty(q.shape[0], dtype=torch.int32, device="cuda")
    def t(f, n=5):
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n): f()
        e1.record(); e1.synchronize()
        return e0.elapsed_time(e1) / n
    tc = t(lambda: cm.radius_count(m, qd, 1.0, cm.SPHERE, counts=cnt))
    def search():
        r = cm.radius_search_batch(m, qd, 1.0, cm.SPHERE, device_out=True)
        return r
    try:
        ts = t(search)
    except TypeError:
        ts = float('nan')
    print(f"cfg{cfg} stride {stride}: nq={q.shape[0]} count {tc:.3f} ms  search {ts:.3f} ms  timing {_native.last_query_timing()}", flush=True)
