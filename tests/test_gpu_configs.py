"""Parity on the BASELINE.json config shapes:

* config 1 at FULL size (20M points, every point a query, r = 1 m, mixed):
  size-independent properties over all 834M neighbours (rows sorted and
  duplicate-free, neighbour relation symmetric, sphere rows inside cube rows,
  counts equal the digest pass) plus exact rows for a query sample against the
  CPU oracle;
* config 2 (TLS, skewed density) and config 3 (kNN) on seeded samples of the
  full-size generators, against the CPU oracle.
"""
import numpy as np
import pytest
import torch

from oracle.oracle import CpuIndex
from paper_2502_11602_b200 import cheesemap as cm
from paper_2502_11602_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg1():
    cloud = synth.config_cloud(1)
    return cloud, torch.from_numpy(cloud).cuda()


def _rows_sorted_unique(row, cols):
    """Every row strictly ascending (device-side check)."""
    n = cols.numel()
    if n < 2:
        return True
    inc = cols[1:] > cols[:-1]
    starts = torch.zeros(n, dtype=torch.bool, device=cols.device)
    rs = row[1:-1]
    rs = rs[(rs > 0) & (rs < n)]
    starts[rs] = True
    return bool((inc | starts[1:]).all().item())


def test_cfg1_full_size_properties(cfg1):
    cloud, dc = cfg1
    m = cm.Cheesemap.build(dc, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    row, cols = cm.radius_search_batch(m, dc, 1.0, cm.SPHERE, device_out=True)
    n = cloud.shape[0]
    assert row.numel() == n + 1 and int(row[-1].item()) == cols.numel()
    assert _rows_sorted_unique(row, cols)
    # symmetry: p in N(q) <=> q in N(p) (fl(a-b) = -fl(b-a), so d^2 is symmetric)
    counts = (row[1:] - row[:-1])
    q_of = torch.repeat_interleave(torch.arange(n, device="cuda"), counts)
    fwd = q_of * n + cols.long()
    bwd = cols.long() * n + q_of
    assert torch.equal(torch.sort(fwd).values, torch.sort(bwd).values)
    del fwd, bwd, q_of
    # counts == digest pass counts; every point finds itself
    cnt, dig = cm.radius_digest_batch(m, dc, 1.0, cm.SPHERE)
    assert np.array_equal(cnt.astype(np.int64), counts.cpu().numpy())
    assert (cnt >= 1).all()
    # sphere rows are inside cube rows
    ccnt, _ = cm.radius_digest_batch(m, dc, 1.0, cm.CUBE)
    assert (ccnt >= cnt).all()
    # exact rows for a sample against the oracle
    rng = np.random.default_rng(7)
    samp = rng.choice(n, 3000, replace=False)
    o = CpuIndex(cloud, flavor=1)
    orow, ocols = o.radius_csr(cloud[samp], 0, 1.0)
    rh, ch = row.cpu().numpy(), cols.cpu().numpy()
    for i, q in enumerate(samp):
        assert np.array_equal(ch[rh[q]:rh[q + 1]].astype(np.uint32), ocols[orow[i]:orow[i + 1]])
    _, odig = o.radius(cloud[samp], 0, 1.0)
    assert np.array_equal(dig[samp], odig)


def test_cfg1_full_size_digests_all_radii(cfg1):
    cloud, dc = cfg1
    rng = np.random.default_rng(11)
    samp = np.ascontiguousarray(cloud[rng.choice(cloud.shape[0], 1500, replace=False)])
    o = CpuIndex(cloud, flavor=1)
    for flavor in (cm.Flavor.Sparse, cm.Flavor.Mixed):
        m = cm.Cheesemap.build(dc, cm.BuildOptions(flavor=flavor))
        for r in (0.5, 1.0, 2.5, 5.0):
            for kern in (cm.SPHERE, cm.CUBE):
                cnt, dig = cm.radius_digest_batch(m, samp, r, kern)
                ocnt, odig = o.radius(samp, kern, r)
                assert np.array_equal(cnt, ocnt) and np.array_equal(dig, odig), (flavor, r, kern)


def test_cfg2_tls_sample():
    """TLS-like cloud (1/16 of the rays: 5000 x 500 = 2.5M points, 0.25 m
    cells, mixed), query centres from CenterStream, r in {0.05, 0.1, 0.25}."""
    cloud = synth.tls(5000, 500, 50, seed=synth.SEED_BASE + 2)
    q = synth.config_queries(2, cloud, count=4000)
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Mixed,
                                                  cell=cm.CellSize.uniform(0.25)))
    o = CpuIndex(cloud, flavor=1, cell=(0.25, 0.25, 0.25))
    for r in (0.05, 0.1, 0.25):
        cnt, dig = cm.radius_digest_batch(m, q, r)
        ocnt, odig = o.radius(q, 0, r)
        assert np.array_equal(cnt, ocnt) and np.array_equal(dig, odig), r
    row, cols = cm.radius_search_batch(m, q[:500], 0.1)
    orow, ocols = o.radius_csr(q[:500], 0, 0.1)
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
    assert (np.diff(row.astype(np.int64)) > 1328).any()  # heavy rows near the scanner


def test_cfg3_knn_sample(cfg1):
    cloud, dc = cfg1
    q = synth.config_queries(3, cloud, count=20000)
    m = cm.Cheesemap.build(dc, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    o = CpuIndex(cloud, flavor=1)
    for k in (8, 16, 32, 64):
        idx, d2 = cm.knn_batch(m, q[:4000], k)
        oidx, od2 = o.knn(q[:4000], k)
        assert np.array_equal(idx, oidx) and np.array_equal(d2, od2), k
