"""Edge cases and error behaviour of the CUDA path through the C ABI, pinned
against the reference's conventions (errors.hpp, map.cpp:23-39,
grid.cpp:18-27, search.cpp:90-92) and the CPU oracle."""
import numpy as np
import pytest

from oracle.oracle import CpuIndex
from paper_2502_11602_b200 import cheesemap as cm

pytestmark = pytest.mark.gpu


def test_build_errors_in_reference_order():
    pts = np.array([[0.0, 0.0, 0.0], [10.0, 10.0, 10.0]])
    with pytest.raises(cm.EmptyCloudError):
        cm.Cheesemap.build(np.zeros((0, 3)))
    for tau in (0.0, -1.0, 1.01):
        with pytest.raises(cm.InvalidArgumentError):
            cm.Cheesemap.build(pts, cm.BuildOptions(densify_threshold=tau))
    with pytest.raises(cm.InvalidArgumentError):
        cm.Cheesemap.build(pts, cm.BuildOptions(cell=cm.CellSize(1.0, -1.0, 1.0)))
    with pytest.raises(cm.CapacityError):
        cm.Cheesemap.build(pts, cm.BuildOptions(dense_voxel_cap=100))
    cm.Cheesemap.build(pts, cm.BuildOptions(flavor=cm.Flavor.Sparse, dense_voxel_cap=100))
    # empty-cloud check precedes the tau check (map.cpp:23-28)
    with pytest.raises(cm.EmptyCloudError):
        cm.Cheesemap.build(np.zeros((0, 3)), cm.BuildOptions(densify_threshold=-1))


def test_grid_known_answer():
    m = cm.Cheesemap.build(np.array([[0.0, 0.0, 0.0], [500.0, 500.0, 168.4]]),
                           cm.BuildOptions(flavor=cm.Flavor.Sparse))
    g = m.grid()
    assert (g["nx"], g["ny"], g["nz"]) == (501, 501, 169)
    assert m.occupancy_stats()["total_voxels"] == 42_419_169


def test_query_errors():
    m = cm.Cheesemap.build(np.random.default_rng(0).uniform(0, 10, (500, 3)))
    with pytest.raises(cm.InvalidArgumentError):
        cm.knn_search(m, (1.0, 1.0, 1.0), 0)
    with pytest.raises(cm.InvalidArgumentError):
        cm.radius_digest_batch(m, np.zeros((3, 3)), 1.0, kernel=7)


@pytest.mark.parametrize("flavor", [cm.Flavor.Dense, cm.Flavor.Sparse, cm.Flavor.Mixed])
def test_degenerate_clouds(flavor):
    rng = np.random.default_rng(1)
    single = np.array([[1.0, 2.0, 3.0]])
    dup = np.repeat(np.array([[4.0, 4.0, 4.0]]), 300, axis=0)
    flat = np.column_stack([rng.uniform(0, 50, 2000), rng.uniform(0, 50, 2000), np.zeros(2000)])
    line = np.column_stack([np.linspace(0, 100, 777), np.zeros(777), np.zeros(777)])
    for cloud in (single, dup, flat, line):
        q = np.concatenate([cloud[::7], np.array([[-50.0, -50.0, -50.0], [1e6, 0, 0]])])
        m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
        o = CpuIndex(cloud, flavor=int(flavor))
        for kern in (cm.SPHERE, cm.CUBE):
            for r in (0.0, 0.7, 3.0):
                row, cols = cm.radius_search_batch(m, q, r, kern)
                orow, ocols = o.radius_csr(q, kern, r)
                assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
        for k in (1, 5, 400):
            idx, d2 = cm.knn_batch(m, q, k)
            oidx, od2 = o.knn(q, k)
            assert np.array_equal(idx, oidx) and np.array_equal(d2, od2), k


def test_two_d_mode_and_anisotropic_cells():
    rng = np.random.default_rng(2)
    cloud = rng.uniform(0, 30, size=(5000, 3)) * np.array([1.0, 0.5, 0.2])
    q = cloud[::9]
    for mode in (cm.GridMode.TwoD, cm.GridMode.ThreeD):
        for flavor in (cm.Flavor.Dense, cm.Flavor.Sparse, cm.Flavor.Mixed):
            opts = cm.BuildOptions(flavor=flavor, mode=mode, cell=cm.CellSize(1.5, 0.7, 0.4))
            m = cm.Cheesemap.build(cloud, opts)
            o = CpuIndex(cloud, flavor=int(flavor), mode=int(mode), cell=(1.5, 0.7, 0.4))
            row, cols = cm.radius_search_batch(m, q, 1.2, cm.SPHERE)
            orow, ocols = o.radius_csr(q, 0, 1.2)
            assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
            idx, d2 = cm.knn_batch(m, q, 9)
            oidx, od2 = o.knn(q, 9)
            assert np.array_equal(idx, oidx) and np.array_equal(d2, od2)


def test_device_and_host_buffers_agree():
    import torch
    rng = np.random.default_rng(3)
    cloud = rng.uniform(0, 20, size=(20000, 3))
    q = cloud[::5].copy()
    m_host = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    m_dev = cm.Cheesemap.build(torch.from_numpy(cloud).cuda(),
                               cm.BuildOptions(flavor=cm.Flavor.Mixed))
    a = cm.radius_search_batch(m_host, q, 1.0)
    b = cm.radius_search_batch(m_dev, torch.from_numpy(q).cuda(), 1.0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    row_d, cols_d = cm.radius_search_batch(m_dev, torch.from_numpy(q).cuda(), 1.0,
                                           device_out=True)
    assert np.array_equal(row_d.cpu().numpy().astype(np.uint64), a[0])
    assert np.array_equal(cols_d.cpu().numpy().astype(np.uint32), a[1])


@pytest.mark.gpu
def test_empty_query_batches():
    """Zero centres: every batched call returns empty outputs (no launch
    reads past an empty buffer), through host and device inputs."""
    import ctypes
    import torch
    from paper_2502_11602_b200 import _native
    cloud = np.random.default_rng(5).uniform(0, 10, (5000, 3))
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    for q in (np.zeros((0, 3)), torch.zeros((0, 3), dtype=torch.float64, device="cuda")):
        for kernel in (cm.SPHERE, cm.CUBE, cm.CYLINDER):
            for r in (1.0, 3.0):  # compact and wide paths
                row, cols = cm.radius_search_batch(m, q, r, kernel)
                assert row.tolist() == [0] and cols.size == 0
                c, d = cm.radius_digest_batch(m, q, r, kernel)
                assert c.size == 0 and d.size == 0
        idx, d2 = cm.knn_batch(m, q, 8)
        assert idx.shape == (0, 8) and d2.shape == (0, 8)
    row = np.zeros(1, dtype=np.uint64)
    nnz = ctypes.c_uint64(7)
    rc = _native.lib().cm_radius_search_to_host(m.handle, None, 0, 0, 1.0,
                                                row.ctypes.data_as(ctypes.c_void_p), None, 0,
                                                ctypes.byref(nnz), None)
    assert rc == 0 and nnz.value == 0 and row[0] == 0
