"""Explicit kernels through cm_kernel_search / cm_kernel_count (the reference's
Kernel concept, geometry.hpp:67-113): per-centre radii, general BoxKernel
Aabbs, bounded CylinderKernels, QueryStats (search.hpp:12-17), and
voxel_present / voxel_lookup (map.hpp:62-69) — against the oracle and the
reference's own definitions."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2502_11602_b200 import cheesemap as cm
from paper_2502_11602_b200 import synth
from oracle.oracle import CpuIndex

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FLAVORS = [cm.Flavor.Dense, cm.Flavor.Sparse, cm.Flavor.Mixed]


@pytest.fixture(scope="module")
def cloud():
    return synth.config_cloud(1, scale=0.003)  # 60k points with a building


def brute(cloud, inside):
    return np.nonzero(inside(cloud))[0].astype(np.uint32)


@pytest.mark.parametrize("flavor", FLAVORS)
def test_general_kernels_equal_linear_scan(cloud, flavor):
    rng = np.random.default_rng(5)
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
    ctr = cloud[rng.choice(cloud.shape[0], 60, replace=False)]
    rad = rng.uniform(0.2, 4.0, 60)
    x, y, z = cloud[:, 0], cloud[:, 1], cloud[:, 2]
    spheres = [cm.SphereKernel(tuple(c), float(r)) for c, r in zip(ctr, rad)]
    boxes = [cm.BoxKernel((c[0] - 2 * r, c[1] - 0.5 * r, c[2] - 0.25 * r),
                          (c[0] + r, c[1] + r, c[2] + 3 * r)) for c, r in zip(ctr, rad)]
    cyls = [cm.CylinderKernel(float(c[0]), float(c[1]), float(r), float(c[2] - 1.0),
                              float(c[2] + 0.5)) for c, r in zip(ctr, rad)]
    cyls_u = [cm.CylinderKernel(float(c[0]), float(c[1]), float(r)) for c, r in zip(ctr, rad)]
    for ks, inside in (
            (spheres, lambda k: ((x - k.center[0]) ** 2 + (y - k.center[1]) ** 2)
             + (z - k.center[2]) ** 2 <= k.radius * k.radius),
            (boxes, lambda k: (x >= k.min[0]) & (x <= k.max[0]) & (y >= k.min[1]) &
             (y <= k.max[1]) & (z >= k.min[2]) & (z <= k.max[2])),
            (cyls, lambda k: (z >= k.z_lo) & (z <= k.z_hi) &
             ((x - k.center_x) ** 2 + (y - k.center_y) ** 2 <= k.radius * k.radius)),
            (cyls_u, lambda k: (x - k.center_x) ** 2 + (y - k.center_y) ** 2
             <= k.radius * k.radius)):
        row, cols = cm.kernel_search_batch(m, ks)
        for q, k in enumerate(ks):
            want = brute(cloud, lambda _c, k=k: inside(k))
            assert np.array_equal(cols[row[q]:row[q + 1]], want), (type(k).__name__, q)


def test_sphere_batch_with_own_radii_equals_oracle(cloud):
    """A batch of spheres with per-centre radii = the uniform-radius batches."""
    o = CpuIndex(cloud, flavor=1)
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    q = np.ascontiguousarray(cloud[::50])
    rad = np.where(np.arange(q.shape[0]) % 2 == 0, 0.7, 2.2)
    row, cols = cm.kernel_search_batch(m, [cm.SphereKernel(tuple(c), float(r)) for c, r in zip(q, rad)])
    for r in (0.7, 2.2):
        sel = np.nonzero(rad == r)[0]
        orow, ocols = o.radius_csr(q[sel], 0, r)
        for t, qi in enumerate(sel):
            assert np.array_equal(cols[row[qi]:row[qi + 1]], ocols[orow[t]:orow[t + 1]])


@pytest.mark.parametrize("flavor", FLAVORS)
def test_query_stats(cloud, flavor):
    """voxels_visited = the voxels of the clamped range; points_tested = the
    points in them (search.hpp:116-119), as the oracle counts them."""
    o = CpuIndex(cloud, flavor=int(flavor))
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
    q = np.ascontiguousarray(cloud[::997])
    _, _, pt, vv = cm.kernel_search_batch(m, [cm.SphereKernel(tuple(c), 1.5) for c in q], stats=True)
    _, _, opt, ovv = o.radius(q, 0, 1.5, stats=True)
    assert np.array_equal(pt, opt) and np.array_equal(vv, ovv)
    st = cm.QueryStats()
    assert len(cm.kernel_search(m, cm.SphereKernel((1e6, 1e6, 1e6), 1.0), stats=st)) == 0
    assert st.voxels_visited == 0 and st.points_tested == 0
    g = m.grid()
    c = [(a + b) / 2 for a, b in zip(g["bounds_min"], g["bounds_max"])]
    allh = cm.kernel_search(m, cm.SphereKernel(tuple(c), 1e5), stats=st)
    assert len(allh) == cloud.shape[0] and st.points_tested == cloud.shape[0]
    assert st.voxels_visited == g["nx"] * g["ny"] * g["nz"]
    nn = cm.knn_search(m, tuple(q[0]), 10, cm.GrowthPolicy.Monotonic, stats=st)
    assert len(nn) == 10 and st.final_radius == nn[-1].distance and st.points_tested >= 10


def test_voxel_lookup(cloud):
    L = cm._native.lib()
    import ctypes
    for flavor in FLAVORS:
        m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
        keys, hs = m.export_voxels()
        g = m.grid()
        nyz = g["ny"] * g["nz"]
        for key in np.unique(keys)[::157]:
            i, j, k = int(key // nyz), int(key % nyz // g["nz"]), int(key % g["nz"])
            want = np.sort(hs[keys == key]).astype(np.uint32)
            out = np.zeros(want.size + 4, dtype=np.uint32)
            n, pres = ctypes.c_uint64(), ctypes.c_int()
            cm._check(L.cm_voxel_lookup(m.handle, i, j, k, ctypes.byref(pres),
                                        out.ctypes.data_as(ctypes.c_void_p), out.size,
                                        ctypes.byref(n)))
            assert pres.value == 1 and n.value == want.size
            assert np.array_equal(out[:want.size], want)
        # an empty voxel: present only for the dense flavour (map.hpp:62-63)
        occupied = set(int(v) for v in np.unique(keys))
        empty = next(v for v in range(g["nx"] * nyz) if v not in occupied)
        i, j, k = empty // nyz, empty % nyz // g["nz"], empty % g["nz"]
        n, pres = ctypes.c_uint64(), ctypes.c_int()
        cm._check(L.cm_voxel_lookup(m.handle, i, j, k, ctypes.byref(pres), None, 0, ctypes.byref(n)))
        assert n.value == 0
        if flavor == cm.Flavor.Dense:
            assert pres.value == 1
        elif flavor == cm.Flavor.Sparse:
            assert pres.value == 0
        assert L.cm_voxel_lookup(m.handle, g["nx"], 0, 0, ctypes.byref(pres), None, 0,
                                 ctypes.byref(n)) == 4  # CM_OUT_OF_DOMAIN


def test_knn_radius_brackets_parity():
    """The opt-in radius-bracket kNN (CMGPU_KNN_BRACKETS) stays exact."""
    code = ("import numpy as np, sys; sys.path.insert(0, %r)\n"
            "from paper_2502_11602_b200 import cheesemap as cm, synth\n"
            "from oracle.oracle import CpuIndex\n"
            "c = synth.config_cloud(1, scale=0.01); q = synth.config_queries(3, c, count=20000)\n"
            "m = cm.Cheesemap.build(c, cm.BuildOptions(flavor=cm.Flavor.Mixed)); o = CpuIndex(c, flavor=1)\n"
            "for k in (1, 8, 33, 64):\n"
            "    i, d = cm.knn_batch(m, q, k); oi, od = o.knn(q, k)\n"
            "    assert np.array_equal(i, oi) and np.array_equal(d, od), k\n"
            "print('brackets ok')\n") % ROOT
    env = dict(os.environ, CMGPU_KNN_BRACKETS="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "brackets ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("env", [
    {},                                                      # defaults: thread pass 1 + register-list pass 2; histogram selection for k > 32
    {"CMGPU_KNN_THREAD_KMAX": "16"},                         # histogram selection for 16 < k <= 64, register list for its leftovers
    {"CMGPU_KNN_THREAD_KMAX": "16", "CMGPU_KNN_HIST": "2"},
    {"CMGPU_KNN_THREAD_KMAX": "16", "CMGPU_KNN_HIST": "0"},  # register-list walk alone for k <= 32, shell walk above
    {"CMGPU_KNN_REDO": "thread"},                            # per-thread second pass
    {"CMGPU_KNN_REDO_L0": "1"},
    {"CMGPU_KNN_REDO_L0": "4"},
], ids=lambda e: ",".join(f"{k[10:]}={v}" for k, v in e.items()) or "default")
def test_knn_paths_parity(env):
    """Every kNN path (pruned per-thread block walk, register-list warp
    walk, histogram selection, shell walk) returns the oracle's rows: an ALS
    tile with sparse lifted points (several shells), all flavours, plus an
    integer lattice with duplicates (distance ties across bin edges, heavy
    bins) and a cloud smaller than k."""
    code = ("import numpy as np, sys; sys.path.insert(0, %r)\n"
            "from paper_2502_11602_b200 import cheesemap as cm, synth\n"
            "from oracle.oracle import CpuIndex\n"
            "c = synth.config_cloud(1, scale=0.01); q = synth.config_queries(3, c, count=12000)\n"
            "rng = np.random.default_rng(7)\n"
            "lat = rng.integers(0, 12, size=(6000, 3)).astype(np.float64) * 0.5\n"
            "few = rng.random((20, 3)) * 3.0\n"
            "far = np.array([[-50.0, 3.0, 1.0], [1e4, 1e4, 1e4], [3.0, 3.0, 500.0]])\n"
            "for fl in (cm.Flavor.Dense, cm.Flavor.Sparse, cm.Flavor.Mixed):\n"
            "    for cloud, qs, ks in ((c, q, (5, 8, 16, 17, 24, 32, 33, 48, 64)), (lat, np.vstack([lat[:1500], far]), (8, 16, 32, 64)), (few, np.vstack([few, far]), (8, 32, 64))):\n"
            "        m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=fl)); o = CpuIndex(cloud, flavor=int(fl))\n"
            "        for k in ks:\n"
            "            i, d = cm.knn_batch(m, qs, k); oi, od = o.knn(qs, k)\n"
            "            assert np.array_equal(i, oi) and np.array_equal(d, od), (int(fl), cloud.shape, k)\n"
            "    # 2D grid mode and anisotropic cells (the z bounds drop out of every prune / stop test)\n"
            "    for mode in (cm.GridMode.TwoD, cm.GridMode.ThreeD):\n"
            "        opts = cm.BuildOptions(flavor=fl, mode=mode, cell=cm.CellSize(1.5, 0.7, 0.4))\n"
            "        m = cm.Cheesemap.build(c, opts); o = CpuIndex(c, flavor=int(fl), mode=int(mode), cell=(1.5, 0.7, 0.4))\n"
            "        for k in (8, 24, 40, 64):\n"
            "            i, d = cm.knn_batch(m, q[:3000], k); oi, od = o.knn(q[:3000], k)\n"
            "            assert np.array_equal(i, oi) and np.array_equal(d, od), (int(fl), int(mode), k)\n"
            "print('paths ok')\n") % ROOT
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "paths ok" in r.stdout, (r.stdout[-500:], r.stderr[-2000:])


@pytest.mark.parametrize("stride", [3, 11, 50, 400])
def test_sparse_query_tiles_split(stride):
    """Sparse centre sets (a tile's hull exceeds 32 columns) go through the
    COLLECT kernel's part splitting (halves, quarters, ... of the tile, then
    one query per warp): the CSR must equal the oracle's for every density,
    flavour and kernel, and for centres off the cloud."""
    c = synth.config_cloud(1, scale=0.02)
    rng = np.random.default_rng(stride)
    q = np.ascontiguousarray(c[::stride][:20000])
    q = np.vstack([q, q[:200] + rng.normal(0, 3.0, size=(200, 3)), [[-1e3, 0, 0], [1e6, 1e6, 1e6]]])
    for fl in (cm.Flavor.Dense, cm.Flavor.Sparse, cm.Flavor.Mixed):
        m = cm.Cheesemap.build(c, cm.BuildOptions(flavor=fl))
        o = CpuIndex(c, flavor=int(fl))
        for kernel, r in ((cm.SPHERE, 1.0), (cm.CUBE, 1.0), (cm.SPHERE, 0.4), (cm.SPHERE, 1.45)):
            row, cols = cm.radius_search_batch(m, q, r, kernel)
            orow, ocols = o.radius_csr(q, int(kernel), r)
            assert np.array_equal(row, orow) and np.array_equal(cols, ocols), (int(fl), int(kernel), r)


def test_voxel_lookup_mirror(cloud):
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Sparse))
    keys, hs = m.export_voxels()
    g = m.grid()
    key = int(keys[len(keys) // 2])
    nyz = g["ny"] * g["nz"]
    v = (key // nyz, key % nyz // g["nz"], key % g["nz"])
    assert m.voxel_present(v)
    assert np.array_equal(m.voxel_lookup(v), np.sort(hs[keys == key]).astype(np.uint64))
