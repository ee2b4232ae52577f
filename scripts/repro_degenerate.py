import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2502_11602_b200 import cheesemap as cm
rng = np.random.default_rng(1)
clouds = {
    "single": np.array([[1.0, 2.0, 3.0]]),
    "dup": np.repeat(np.array([[4.0, 4.0, 4.0]]), 300, axis=0),
    "flat": np.column_stack([rng.uniform(0, 50, 2000), rng.uniform(0, 50, 2000), np.zeros(2000)]),
    "line": np.column_stack([np.linspace(0, 100, 777), np.zeros(777), np.zeros(777)]),
}
for name, cloud in clouds.items():
    q = np.concatenate([cloud[::7], np.array([[-50.0, -50.0, -50.0], [1e6, 0, 0]])])
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Dense))
    for r in (0.0, 0.7, 3.0):
        print(name, r, flush=True)
        cm.radius_search_batch(m, q, r, 0)
print("ok")
