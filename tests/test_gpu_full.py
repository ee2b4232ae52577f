"""Full-population parity at BASELINE size (driver-visible): the headline
workload — config 1, 20M points, mixed flavour, sphere r = 1 m, EVERY point a
query — checked query by query against the multithreaded CPU oracle, through
the digest pass, the self-query CSR (the bench path) and the general-centre
CSR. scripts/verify_full.py runs the same check over every config and radius
(profiles/r02/verify_full.json)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))


@pytest.mark.gpu
def test_config1_every_query_r1():
    import torch
    import verify_full as vf
    from paper_2502_11602_b200 import cheesemap as cm
    from paper_2502_11602_b200 import synth

    cloud = synth.config_cloud(1)
    nq = cloud.shape[0]
    oracle = vf.Oracle(cloud, 1.0, 0)
    oc, od, _ = oracle.radius(cloud, 0, 1.0)
    dc = torch.from_numpy(cloud).cuda()
    qd = dc.clone()
    m = cm.Cheesemap.build(dc, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    gc, gd, _ = vf.gpu_digest(m, qd, nq, 0, 1.0)
    assert vf.compare("digest", gc, gd, oc, od)["mismatches"] == 0
    for self_q in (True, False):
        cc, cd, uns, _, chunks = vf.gpu_csr(m, qd, nq, 0, 1.0, gc, 6_000_000_000, self_q)
        assert chunks == 1 and uns == 0
        assert vf.compare(f"csr self={self_q}", cc, cd, oc, od)["mismatches"] == 0
