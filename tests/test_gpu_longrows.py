"""Rows longer than a warp buffer (> kSortCap handles), the TLS case of
config 2: merged from their per-voxel sorted runs (merge_big_rows_kernel) —
in shared memory, in global memory (rows > 27648), and through fixed
bitonic chunks when a row has more than 1024 runs — must equal the oracle's
sorted lists, through cm_radius_search and the host-buffer pipeline."""
import ctypes

import numpy as np
import pytest

from paper_2502_11602_b200 import cheesemap as cm
from paper_2502_11602_b200 import synth
from oracle.oracle import CpuIndex

pytestmark = pytest.mark.gpu


def check(cloud, q, r, flavor, cell):
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor, cell=cm.CellSize.uniform(cell)))
    o = CpuIndex(cloud, flavor=1, cell=(cell,) * 3)
    row, cols = cm.radius_search_batch(m, q, r)
    orow, ocols = o.radius_csr(q, 0, r)
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
    return np.diff(row.astype(np.int64))


@pytest.mark.parametrize("flavor", [cm.Flavor.Sparse, cm.Flavor.Mixed])
def test_long_rows_few_runs(flavor):
    # dense blobs: voxels of hundreds of points, rows of thousands to 60k
    rng = np.random.default_rng(11)
    blob = rng.normal(0.0, 0.35, size=(120_000, 3))
    cloud = np.ascontiguousarray(np.concatenate([blob, rng.uniform(-3, 3, size=(30_000, 3))]))
    q = np.ascontiguousarray(cloud[rng.choice(cloud.shape[0], 700, replace=False)])
    lens = check(cloud, q, 0.5, flavor, 0.25)
    assert lens.max() > 27648 and (lens > 1056).sum() > 100  # global-memory and smem merges


def test_long_rows_many_runs():
    # tiny cells: a row is thousands of runs of 1-3 handles (chunked path)
    rng = np.random.default_rng(12)
    cloud = np.ascontiguousarray(rng.uniform(0, 1, size=(60_000, 3)))
    q = np.ascontiguousarray(cloud[::600])
    lens = check(cloud, q, 0.3, cm.Flavor.Sparse, 0.03)
    assert (lens > 1056).all()


def test_long_rows_host_pipeline():
    rng = np.random.default_rng(13)
    cloud = np.ascontiguousarray(rng.normal(0.0, 0.4, size=(150_000, 3)))
    q = np.ascontiguousarray(cloud[::300])
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Mixed, cell=cm.CellSize.uniform(0.25)))
    o = CpuIndex(cloud, flavor=1, cell=(0.25,) * 3)
    orow, ocols = o.radius_csr(q, 0, 0.6)
    row = np.zeros(q.shape[0] + 1, dtype=np.uint64)
    cols = np.zeros(ocols.size, dtype=np.uint32)
    nnz = ctypes.c_uint64()
    L = cm._native.lib()
    cm._check(L.cm_radius_search_to_host(m.handle, q.ctypes.data_as(ctypes.c_void_p), q.shape[0], 0,
                                         0.6, row.ctypes.data_as(ctypes.c_void_p),
                                         cols.ctypes.data_as(ctypes.c_void_p), cols.size,
                                         ctypes.byref(nnz), None))
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)


def test_config2_scaled_csr():
    cloud = synth.config_cloud(2, scale=1 / 64)
    q = synth.config_queries(2, cloud, count=3000)
    check(cloud, np.ascontiguousarray(q), 0.1, cm.Flavor.Mixed, 0.25)
