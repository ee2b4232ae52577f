"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists and oracle/_ref/libcheesemap_ref.so
is built from the reference's own sources by `make -C oracle ref`):

    python tests/golden/make_golden.py

Every expected output is produced by the unmodified reference library
(Cheesemap::build / kernel_search / knn_search / occupancy_stats through
oracle/refshim.cpp). The fixtures are small .npz files; the tests replay the
same inputs through the CPU restatement (tests/test_oracle_golden.py) and the
CUDA path (tests/test_gpu_golden.py).
"""
import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import CpuIndex, lib  # noqa: E402
from paper_2502_11602_b200 import synth  # noqa: E402


def ref_uniform(seed, n, ex, ey, ez):
    L = lib("reference").lib
    fn = L.ref_generate_uniform
    fn.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                   ctypes.c_double, ctypes.c_void_p]
    fn.restype = ctypes.c_int
    out = np.zeros((n, 3))
    assert fn(seed, n, ex, ey, ez, out.ctypes.data_as(ctypes.c_void_p)) == 0
    return out


def case(name, cloud, queries, builds, radii, ks, **extra):
    """builds: list of (flavor, mode, cell, tau). One fixture per build."""
    out = {}
    for bi, (flavor, mode, cell, tau) in enumerate(builds):
        ref = CpuIndex(cloud, flavor=flavor, mode=mode, cell=cell, tau=tau, which="reference")
        g = ref.grid()
        keys, handles = ref.export()
        dense, ne = ref.slice_flags()
        p = f"b{bi}_"
        out[p + "build"] = np.array([flavor, mode, cell[0], cell[1], cell[2], tau])
        out[p + "origin"] = g["origin"]
        out[p + "dims"] = g["dims"]
        out[p + "bmin"], out[p + "bmax"] = g["bmin"], g["bmax"]
        out[p + "keys"], out[p + "handles"] = keys, handles
        out[p + "non_empty"] = np.array([ref.non_empty()], dtype=np.uint64)
        out[p + "slice_dense"], out[p + "slice_non_empty"] = dense, ne
        if bi == 0:
            for kern in (0, 1):
                for r in radii:
                    row, cols = ref.radius_csr(queries, kern, r)
                    _, _, tested, visited = ref.radius(queries, kern, r, stats=True)
                    tag = f"r{kern}_{r:g}_"
                    out[tag + "row"], out[tag + "cols"] = row, cols
                    out[tag + "tested"], out[tag + "visited"] = tested, visited
            for k in ks:
                idx, d2 = ref.knn(queries, k)
                out[f"k{k}_idx"], out[f"k{k}_d2"] = idx, d2
    out["cloud"] = cloud
    out["queries"] = queries
    out["radii"] = np.array(radii, dtype=np.float64)
    out["ks"] = np.array(ks, dtype=np.int64)
    out["nbuilds"] = np.array([len(builds)])
    for k, v in extra.items():
        out[k] = v
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **out)
    print(f"{path}: {os.path.getsize(path) / 1024:.0f} KiB")


def main():
    rng = np.random.default_rng(11602)
    # 1. the reference's own uniform generator (io.cpp:266-272), as in
    #    tests/test_util.hpp:13-23; centres from the cloud + outside the bbox
    cloud = ref_uniform(42, 4000, 30.0, 20.0, 10.0)
    assert np.array_equal(cloud, synth.uniform(4000, 30.0, 20.0, 10.0, 42)), \
        "synth.uniform must be bit-identical to the reference generator"
    q = np.concatenate([cloud[::20], rng.uniform([-5, -5, -5], [35, 25, 15], size=(60, 3))])
    builds = [(0, 1, (1.0, 1.0, 1.0), 0.8), (1, 1, (2.5, 2.5, 2.5), 0.8),
              (2, 1, (1.0, 1.0, 1.0), 0.8), (2, 1, (3.0, 2.0, 1.5), 0.5),
              (1, 0, (2.0, 2.0, 2.0), 0.8)]
    case("uniform4k", cloud, q, builds, [0.5, 1.7, 3.0], [1, 5, 20])

    # 2. config-0 generator (ALS terrain + vegetation) at 1/50 scale
    als = synth.config_cloud(0, scale=0.02)
    case("als20k", als, np.ascontiguousarray(als[::25]), [(0, 1, (1.0, 1.0, 1.0), 0.8),
                                                          (2, 1, (1.0, 1.0, 1.0), 0.8)],
         [1.0, 2.5], [8, 16])

    # 3. lattice with exact ties: integer coordinates, centres on lattice
    #    points (distance ties at every shell; sphere boundary points)
    g = np.stack(np.meshgrid(np.arange(8.0), np.arange(6.0), np.arange(4.0), indexing="ij"),
                 -1).reshape(-1, 3)
    g = np.concatenate([g, g[:40]])  # duplicates: equal points, distinct handles
    case("lattice", g, np.ascontiguousarray(g[::7]), [(0, 1, (1.0, 1.0, 1.0), 0.8),
                                                      (1, 1, (2.0, 2.0, 2.0), 0.8)],
         [1.0, 1.5, 2.0], [1, 7, 27])

    # 4. mixed densify boundary (test_map.cpp:152-187 idea): a 10x10
    #    footprint, slice 0 with 79 occupied cells, slice 1 with 80
    cells = [(i, j) for i in range(10) for j in range(10)]
    pts = []
    for (i, j) in cells[:78] + [(9, 9)]:
        pts.append([i + 0.5, j + 0.5, 0.25])
    for (i, j) in cells[:79] + [(9, 9)]:
        pts.append([i + 0.5, j + 0.5, 1.25])
    pts = np.array(pts)
    case("tau_boundary", pts, np.ascontiguousarray(pts[::9]),
         [(2, 1, (1.0, 1.0, 1.0), 0.8), (2, 1, (1.0, 1.0, 1.0), 0.5)], [1.0], [3])


if __name__ == "__main__":
    main()
