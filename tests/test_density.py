"""the cylinder kernel (geometry.hpp:97-113) and the
dataset metrics that drive it (analysis.cpp:17-86), pinned like the
reference's test_analysis.cpp (:18-36 brute-force oracle, :96-103) and
acceptance criterion c9."""
import os

import numpy as np
import pytest

from oracle.oracle import CpuIndex, weighted_density
from paper_2502_11602_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAS_REF = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libcheesemap_ref.so"))


def brute_weighted_density(cloud):
    """O(N^2) restatement (test_analysis.cpp:18-36 style): per point, the
    points with dx^2 + dy^2 <= 1 (self included), count/pi floored, 256 bins."""
    xy = cloud[:, :2]
    bins = np.zeros(256, dtype=np.uint64)
    for p in xy:
        d = xy - p
        c = int(np.count_nonzero(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] <= 1.0))
        bins[min(255, int(c / np.pi))] += 1
    value = float((np.arange(256) * bins).sum()) / float(bins.sum())
    return value, bins


@pytest.mark.skipif(not HAS_REF, reason="oracle/_ref not built")
@pytest.mark.parametrize("sample", [0, 777])
def test_weighted_density_oracle_equals_reference(sample):
    cloud = synth.config_cloud(0, scale=0.02)
    a = weighted_density(cloud, sample, 5)
    b = weighted_density(cloud, sample, 5, which="reference")
    assert a[0] == b[0] and np.array_equal(a[1], b[1])


def test_weighted_density_oracle_equals_brute_force():
    rng = np.random.default_rng(3)
    cloud = np.column_stack([rng.uniform(0, 12, 1500), rng.uniform(0, 9, 1500),
                             rng.uniform(0, 3, 1500)])
    v, bins = weighted_density(cloud)
    bv, bb = brute_weighted_density(cloud)
    assert np.array_equal(bins, bb) and v == bv


@pytest.mark.skipif(not HAS_REF, reason="oracle/_ref not built")
def test_cylinder_kernel_oracle_equals_reference():
    cloud = synth.config_cloud(1, scale=0.005)
    q = cloud[::37]
    for mode in (0, 1):
        o = CpuIndex(cloud, flavor=2, mode=mode)
        r = CpuIndex(cloud, flavor=2, mode=mode, which="reference")
        for rad in (0.5, 1.0, 2.0):
            for x, y in zip(o.radius(q, 2, rad, stats=True), r.radius(q, 2, rad, stats=True)):
                assert np.array_equal(x, y)


@pytest.mark.gpu
def test_gpu_cylinder_rows_and_weighted_density():
    from paper_2502_11602_b200 import cheesemap as cm
    cloud = synth.config_cloud(0)  # 1M points
    q = cloud[::10]
    o = CpuIndex(cloud, flavor=1, mode=0)
    for mode in (cm.GridMode.TwoD, cm.GridMode.ThreeD):
        m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Sparse, mode=mode))
        row, cols = cm.radius_search_batch(m, q, 1.0, cm.CYLINDER)
        orow, ocols = o.radius_csr(q, 2, 1.0)
        assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
    for sample, seed in ((0, 0), (100_000, 9)):
        gv, gb = cm.weighted_density(cloud, sample, seed)
        ov, ob = weighted_density(cloud, sample, seed)
        assert gv == ov and np.array_equal(gb, ob)
    small = np.random.default_rng(4).uniform(0, 10, (800, 3))
    gv, gb = cm.weighted_density(small)
    bv, bb = brute_weighted_density(small)
    assert gv == bv and np.array_equal(gb, bb)
    gd = cm.global_density(cloud)
    ext = cloud.max(0) - cloud.min(0)
    assert gd == cloud.shape[0] / (ext[0] * ext[1])
    with pytest.raises(cm.InvalidArgumentError):
        cm.global_density(np.array([[1.0, 2.0, 3.0], [1.0, 5.0, 3.0]]))
