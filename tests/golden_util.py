"""Replay of the golden fixtures (tests/golden/*.npz, made by the reference
through tests/golden/make_golden.py) against any implementation."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fixtures():
    return sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))


def fixture_ids():
    return [os.path.basename(p)[:-4] for p in fixtures()]


def builds(d):
    for bi in range(int(d["nbuilds"][0])):
        b = d[f"b{bi}_build"]
        yield bi, int(b[0]), int(b[1]), (float(b[2]), float(b[3]), float(b[4])), float(b[5])


def check_build(d, bi, grid, keys, handles, non_empty, slice_dense, slice_ne):
    p = f"b{bi}_"
    assert np.array_equal(np.asarray(grid["dims"], dtype=np.uint64), d[p + "dims"])
    assert np.array_equal(np.asarray(grid["origin"]), d[p + "origin"])
    assert np.array_equal(np.asarray(grid["bmin"]), d[p + "bmin"])
    assert np.array_equal(np.asarray(grid["bmax"]), d[p + "bmax"])
    assert np.array_equal(np.asarray(keys, dtype=np.uint64), d[p + "keys"])
    assert np.array_equal(np.asarray(handles, dtype=np.uint64), d[p + "handles"])
    assert int(non_empty) == int(d[p + "non_empty"][0])
    if d[p + "slice_dense"].size:  # the reference reports slices for mixed maps only
        assert np.array_equal(np.asarray(slice_dense, dtype=bool), d[p + "slice_dense"])
        assert np.array_equal(np.asarray(slice_ne, dtype=np.uint64), d[p + "slice_non_empty"])


def radius_cases(d):
    for kern in (0, 1):
        for r in d["radii"]:
            tag = f"r{kern}_{float(r):g}_"
            yield kern, float(r), d[tag + "row"], d[tag + "cols"], d[tag + "tested"]


def knn_cases(d):
    for k in d["ks"]:
        yield int(k), d[f"k{int(k)}_idx"], d[f"k{int(k)}_d2"]
