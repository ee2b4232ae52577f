"""kNN (config 3) probe: rate per k on the 20M cloud with 5M random centres,
optionally one k only (for ncu: KNN_K=64)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_11602_b200 import cheesemap as cm, synth  # noqa: E402

cloud = synth.config_cloud(3)
q = np.ascontiguousarray(synth.config_queries(3, cloud))
m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Mixed))
qd = torch.from_numpy(q).cuda()
ks = [int(os.environ["KNN_K"])] if "KNN_K" in os.environ else [8, 16, 32, 64]
reps = int(os.environ.get("KNN_REPS", "3"))
for k in ks:
    cm.knn_batch(m, qd, k, device_out=True)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t = time.perf_counter()
        cm.knn_batch(m, qd, k, device_out=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"k={k}: {best * 1e3:.1f} ms  {q.shape[0] / best / 1e6:.1f} M q/s", flush=True)
