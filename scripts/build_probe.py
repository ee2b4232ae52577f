"""Build-phase probe: repeated builds of the config-1 cloud per flavour."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_11602_b200 import cheesemap as cm, synth  # noqa: E402

cloud = torch.from_numpy(synth.config_cloud(1)).cuda()
for fl in (cm.Flavor.Mixed, cm.Flavor.Dense, cm.Flavor.Sparse):
    for rep in range(4):
        m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=fl))
        t = m.build_timing()
        print(fl.name, {k: round(v, 3) if isinstance(v, float) else v for k, v in t.items()}, flush=True)
        del m
