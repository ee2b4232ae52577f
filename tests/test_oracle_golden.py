"""The CPU restatement (oracle/cheesemap_oracle.cpp) reproduces every golden
fixture the reference produced (tests/golden/make_golden.py)."""
import numpy as np
import pytest

from golden_util import builds, check_build, fixture_ids, fixtures, knn_cases, radius_cases
from oracle.oracle import CpuIndex


@pytest.mark.parametrize("path", fixtures(), ids=fixture_ids())
def test_oracle_matches_golden(path):
    d = np.load(path)
    cloud, q = d["cloud"], d["queries"]
    for bi, flavor, mode, cell, tau in builds(d):
        o = CpuIndex(cloud, flavor=flavor, mode=mode, cell=cell, tau=tau)
        g = o.grid()
        keys, handles = o.export()
        dense, ne = o.slice_flags()
        check_build(d, bi, g, keys, handles, o.non_empty(), dense, ne)
        if bi:
            continue
        for kern, r, row, cols, tested in radius_cases(d):
            orow, ocols = o.radius_csr(q, kern, r, threads=2)
            assert np.array_equal(orow, row) and np.array_equal(ocols, cols), (kern, r)
            _, _, otested, _ = o.radius(q, kern, r, threads=2, stats=True)
            assert np.array_equal(otested, tested)
        for k, idx, d2 in knn_cases(d):
            oidx, od2 = o.knn(q, k, threads=2)
            assert np.array_equal(oidx, idx) and np.array_equal(od2, d2), k


def test_golden_fixtures_present():
    assert len(fixtures()) >= 4
