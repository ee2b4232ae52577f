"""x-slab layout on one GPU ("virtual slabs"): every slab indexed on the
global grid with cm_build_in_bounds, owned queries answered locally and
mapped back to global ids, must equal the global index's rows exactly."""
import numpy as np
import pytest
import torch

from paper_2502_11602_b200 import cheesemap as cm
from paper_2502_11602_b200 import cluster, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
def test_virtual_slabs_equal_global(world):
    cloud = synth.config_cloud(4, scale=0.002)  # 400k points, config-4 generator
    glob = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Sparse))
    for r in (1.0, 2.5):
        grow, gcols = cm.radius_search_batch(glob, cloud, r)
        seen = 0
        for s in range(world):
            part = cluster.VirtualSlab(cloud, s, world, halo=5.0)
            m = cluster.gpu_slab_index(part, cm.BuildOptions(flavor=cm.Flavor.Sparse))
            assert m.grid()["nx"] == glob.grid()["nx"]  # the global grid
            q = cloud[part.owned_ids.numpy()]
            row, cols = cm.radius_search_batch(m, q, r)
            cols_g = part.to_global(torch.from_numpy(cols.astype(np.int64))).numpy()
            for i, qg in enumerate(part.owned_ids.numpy()):
                assert np.array_equal(cols_g[row[i]:row[i + 1]], gcols[grow[qg]:grow[qg + 1]])
            seen += part.n_owned
        assert seen == cloud.shape[0]


def test_build_in_bounds_rejects_points_outside():
    import ctypes
    from paper_2502_11602_b200 import _native
    pts = np.random.default_rng(0).uniform(0, 10, (100, 3))
    lo = np.zeros(3)
    hi = np.full(3, 5.0)
    h = ctypes.c_void_p()
    c = cm.BuildOptions().to_c()
    rc = _native.lib().cm_build_in_bounds(pts.ctypes.data_as(ctypes.c_void_p), 100,
                                          ctypes.byref(c), lo.ctypes.data_as(ctypes.c_void_p),
                                          hi.ctypes.data_as(ctypes.c_void_p), 0, None,
                                          ctypes.byref(h))
    assert rc == 4  # CM_OUT_OF_DOMAIN
