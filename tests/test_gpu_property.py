"""Property-based parity (hypothesis): random clouds (uniform, clustered,
duplicated, flat), random anisotropic cells, both grid modes, every flavour
and kernel, radii from far below to far above the cell size (compact tiles,
wide tiles, one query per warp), kNN with k up to 300 — the CUDA path must
equal the CPU oracle exactly on every drawn case."""
import numpy as np
import pytest

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

from oracle.oracle import CpuIndex  # noqa: E402
from paper_2502_11602_b200 import cheesemap as cm  # noqa: E402

pytestmark = pytest.mark.gpu


def make_cloud(kind, n, seed, ext):
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.uniform(0, ext, (n, 3))
    if kind == "clusters":
        c = rng.uniform(0, ext, (5, 3))
        return c[rng.integers(0, 5, n)] + rng.normal(0, ext / 20, (n, 3))
    if kind == "duplicates":
        base = rng.uniform(0, ext, (max(1, n // 20), 3))
        return base[rng.integers(0, base.shape[0], n)]
    # flat: a plane with a few outliers (thin z extent)
    pts = np.column_stack([rng.uniform(0, ext, n), rng.uniform(0, ext, n), np.zeros(n)])
    pts[: max(1, n // 50), 2] = rng.uniform(0, ext / 10, max(1, n // 50))
    return pts


cases = st.fixed_dictionaries({
    "kind": st.sampled_from(["uniform", "clusters", "duplicates", "flat"]),
    "n": st.integers(200, 6000),
    "seed": st.integers(0, 2 ** 31),
    "ext": st.sampled_from([5.0, 30.0, 120.0]),
    "cell": st.tuples(st.sampled_from([0.3, 1.0, 2.5]), st.sampled_from([0.3, 1.0, 2.5]),
                      st.sampled_from([0.3, 1.0, 2.5])),
    "mode": st.sampled_from([0, 1]),
    "flavor": st.sampled_from([0, 1, 2]),
    "kernel": st.sampled_from([0, 1, 2]),
    "r": st.sampled_from([0.05, 0.5, 1.0, 3.0, 8.0]),
    "k": st.sampled_from([1, 7, 32, 300]),
})


@settings(max_examples=250, deadline=None, suppress_health_check=list(HealthCheck))
@given(case=cases)
def test_random_cases_equal_oracle(case):
    cloud = make_cloud(case["kind"], case["n"], case["seed"], case["ext"])
    rng = np.random.default_rng(case["seed"] + 1)
    q = np.vstack([cloud[rng.integers(0, cloud.shape[0], 150)],
                   rng.uniform(-0.2 * case["ext"], 1.2 * case["ext"], (50, 3))])
    q = np.ascontiguousarray(q)
    opts = cm.BuildOptions(flavor=cm.Flavor(case["flavor"]), mode=cm.GridMode(case["mode"]),
                           cell=cm.CellSize(*case["cell"]))
    try:
        m = cm.Cheesemap.build(cloud, opts)
    except cm.CapacityError:
        return  # dense grids over the cap are the reference's CapacityError too
    o = CpuIndex(cloud, flavor=case["flavor"], mode=case["mode"], cell=case["cell"])
    row, cols = cm.radius_search_batch(m, q, case["r"], case["kernel"])
    orow, ocols = o.radius_csr(q, case["kernel"], case["r"])
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
    c, d = cm.radius_digest_batch(m, q, case["r"], case["kernel"])
    oc, od = o.radius(q, case["kernel"], case["r"])
    assert np.array_equal(c, oc) and np.array_equal(d, od)
    idx, d2 = cm.knn_batch(m, q[:60], case["k"])
    oidx, od2 = o.knn(q[:60], case["k"])
    assert np.array_equal(idx, oidx) and np.array_equal(d2, od2)
