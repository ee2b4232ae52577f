"""GPU parity: the CUDA path through the C ABI against the CPU oracle on the
same seeded inputs (bit-exact for sets, indices and fp64 distances)."""
import numpy as np
import pytest

from paper_2502_11602_b200 import cheesemap as cm
from paper_2502_11602_b200 import synth
from oracle.oracle import CpuIndex

pytestmark = pytest.mark.gpu

FLAVORS = [cm.Flavor.Dense, cm.Flavor.Sparse, cm.Flavor.Mixed]


@pytest.fixture(scope="module")
def cfg0():
    cloud = synth.config_cloud(0)
    return cloud, synth.config_queries(0, cloud)


@pytest.fixture(scope="module")
def cfg0_oracle(cfg0):
    return CpuIndex(cfg0[0], flavor=0)


@pytest.mark.parametrize("flavor", FLAVORS)
def test_build_parity_cfg0(cfg0, flavor):
    cloud, _ = cfg0
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
    ref = CpuIndex(cloud, flavor=int(flavor))
    g, og = m.grid(), ref.grid()
    assert [g["nx"], g["ny"], g["nz"]] == og["dims"].tolist()
    assert np.array_equal(np.array(g["origin"]), og["origin"])
    keys, hs = m.export_voxels()
    okeys, ohs = ref.export()
    assert np.array_equal(keys, okeys)
    assert np.array_equal(hs.astype(np.uint64), ohs)
    occ = m.occupancy_stats()
    assert occ["non_empty"] == ref.non_empty()
    if flavor == cm.Flavor.Mixed:  # the reference reports slices for mixed maps
        dense, ne = ref.slice_flags()
        assert np.array_equal(occ["slice_dense"], dense)
        assert np.array_equal(occ["slice_non_empty"], ne)


@pytest.mark.parametrize("flavor", FLAVORS)
@pytest.mark.parametrize("kernel", [cm.SPHERE, cm.CUBE])
def test_radius_csr_cfg0(cfg0, cfg0_oracle, flavor, kernel):
    cloud, q = cfg0
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
    row, cols = cm.radius_search_batch(m, q, 1.0, kernel)
    orow, ocols = cfg0_oracle.radius_csr(q, kernel, 1.0)
    assert np.array_equal(row, orow)
    assert np.array_equal(cols, ocols)


@pytest.mark.parametrize("flavor", FLAVORS)
@pytest.mark.parametrize("r", [0.05, 0.5, 2.5, 5.0])
def test_radius_digest_cfg0(cfg0, cfg0_oracle, flavor, r):
    cloud, q = cfg0
    q = q[::4]
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
    for kernel in (cm.SPHERE, cm.CUBE):
        cnt, dig = cm.radius_digest_batch(m, q, r, kernel)
        ocnt, odig = cfg0_oracle.radius(q, kernel, r)
        assert np.array_equal(cnt, ocnt)
        assert np.array_equal(dig, odig)
        tested = np.zeros(q.shape[0], dtype=np.uint64)
        cm.radius_count(m, q, r, kernel, points_tested=tested)
        _, _, opt, _ = cfg0_oracle.radius(q, kernel, r, stats=True)
        assert np.array_equal(tested, opt)


@pytest.mark.parametrize("flavor", FLAVORS)
@pytest.mark.parametrize("k", [1, 8, 16, 64])
def test_knn_cfg0(cfg0, cfg0_oracle, flavor, k):
    cloud, q = cfg0
    q = q[:20000]
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
    idx, d2 = cm.knn_batch(m, q, k)
    oidx, od2 = cfg0_oracle.knn(q, k)
    assert np.array_equal(idx, oidx)
    assert np.array_equal(d2, od2)


def test_big_rows_sorted(cfg0, cfg0_oracle):
    """r = 8 m gives rows above the per-warp buffer (block-sort path)."""
    cloud, q = cfg0
    q = q[:3000]
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Sparse))
    row, cols = cm.radius_search_batch(m, q, 8.0, cm.SPHERE)
    orow, ocols = cfg0_oracle.radius_csr(q, 0, 8.0)
    assert (np.diff(row.astype(np.int64)) > 2048).any()
    assert np.array_equal(row, orow)
    assert np.array_equal(cols, ocols)


def test_corruption_detected(cfg0, cfg0_oracle):
    cloud, q = cfg0
    for flavor in FLAVORS:
        m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
        m.corrupt_for_testing()
        cnt, dig = cm.radius_digest_batch(m, cloud, 1.0)
        ocnt, odig = cfg0_oracle.radius(cloud, 0, 1.0)
        assert not (np.array_equal(cnt, ocnt) and np.array_equal(dig, odig))


@pytest.mark.parametrize("recollect", [True, False])
def test_arena_overflow_falls_back(cfg0, cfg0_oracle, monkeypatch, recollect):
    """A small-radius call shrinks the arena estimate; the next, larger query
    overflows it and must rerun the collect into an arena of the exact size
    (or, with CMGPU_NO_RECOLLECT, take count + fill) with identical results."""
    from paper_2502_11602_b200 import _native
    if not recollect:
        monkeypatch.setenv("CMGPU_NO_RECOLLECT", "1")
    cloud, q = cfg0
    q = q[:60000]
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    for _ in range(90):  # the estimate decays by 0.95 per call
        cm.radius_search_batch(m, q[:1000], 0.05, cm.SPHERE)
    row, cols = cm.radius_search_batch(m, q, 1.4, cm.SPHERE)
    assert _native.last_query_timing()["two_pass"] == (2 if recollect else 1)
    orow, ocols = cfg0_oracle.radius_csr(q, 0, 1.4)
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
    row, cols = cm.radius_search_batch(m, q, 1.4, cm.SPHERE)
    assert _native.last_query_timing()["two_pass"] == 0
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)


@pytest.mark.parametrize("flavor", FLAVORS)
@pytest.mark.parametrize("kernel", [cm.SPHERE, cm.CUBE, cm.CYLINDER])
@pytest.mark.parametrize("r", [2.5, 4.0])
def test_wide_radius_csr(cfg0, cfg0_oracle, flavor, kernel, r):
    """Large radii: wide tiles (hulls of > 32 columns in batches of 32), count
    + scan + unsorted fill + in-place row sort."""
    from paper_2502_11602_b200 import _native
    cloud, _ = cfg0
    # a spatially dense query set (every point of a corner), so tiles are compact
    q = cloud[(cloud[:, 0] < cloud[:, 0].min() + 40) & (cloud[:, 1] < cloud[:, 1].min() + 40)]
    q = np.ascontiguousarray(q[:8000])
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
    _native.query_stats(reset=True)
    row, cols = cm.radius_search_batch(m, q, r, kernel)
    assert _native.last_query_timing()["two_pass"] == 1
    st = _native.query_stats()
    # most fill tiles went wide, not one query per warp (the tile counters
    # are compiled into the checked library only: scripts/checked_probe.py
    # asserts the same there)
    if st["fill_tiles"]:
        assert st["fill_fallback_tiles"] < st["fill_tiles"] // 4
    orow, ocols = cfg0_oracle.radius_csr(q, int(kernel), r)
    assert np.array_equal(row, orow)
    assert np.array_equal(cols, ocols)


def test_wide_tall_columns():
    """A dense vertical column: spans past the 11-bit key range (key base
    moves up mid-column) and rows past the warp sort (block sort)."""
    rng = np.random.default_rng(17)
    tower = np.column_stack([rng.uniform(0, 1.5, 30000), rng.uniform(0, 1.5, 30000),
                             rng.uniform(0, 3, 30000)])
    bg = rng.uniform(0, 20, (20000, 3))
    cloud = np.ascontiguousarray(np.vstack([bg, tower]))
    q = np.ascontiguousarray(np.vstack([tower[::50], bg[::10]]))
    o = CpuIndex(cloud, flavor=1)
    for flavor in FLAVORS:
        m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
        for r in (2.5, 3.5):
            row, cols = cm.radius_search_batch(m, q, r, cm.SPHERE)
            orow, ocols = o.radius_csr(q, 0, r)
            assert (np.diff(orow.astype(np.int64)) > 4096).any()
            assert np.array_equal(row, orow) and np.array_equal(cols, ocols)


@pytest.mark.parametrize("flavor", FLAVORS)
@pytest.mark.parametrize("r", [1.5, 2.5])
def test_count_then_fill_api(cfg0, cfg0_oracle, flavor, r):
    """The two-call CSR API (cm_radius_count, caller scan, cm_radius_fill)."""
    import ctypes
    from paper_2502_11602_b200 import _native
    cloud, q = cfg0
    q = np.ascontiguousarray(q[:30000])
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
    L = _native.lib()
    counts = np.zeros(q.shape[0], dtype=np.uint32)
    qp = q.ctypes.data_as(ctypes.c_void_p)
    cm._check(L.cm_radius_count(m.handle, qp, q.shape[0], 1, r,
                                counts.ctypes.data_as(ctypes.c_void_p), None, None))
    row = np.zeros(q.shape[0] + 1, dtype=np.uint64)
    np.cumsum(counts, out=row[1:])
    cols = np.zeros(int(row[-1]), dtype=np.uint32)
    cm._check(L.cm_radius_fill(m.handle, qp, q.shape[0], 1, r,
                               row.ctypes.data_as(ctypes.c_void_p),
                               cols.ctypes.data_as(ctypes.c_void_p), None))
    orow, ocols = cfg0_oracle.radius_csr(q, 1, r)
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)


@pytest.mark.parametrize("chunks,r", [(None, 1.0), ("3", 1.0), ("8", 1.0), ("3", 2.5)])
def test_search_to_host_pipeline(cfg0, cfg0_oracle, monkeypatch, chunks, r):
    """cm_radius_search_to_host (chunked host<->device overlap, every chunk's
    CSR streamed during its gather) returns the same CSR; a too-small capacity
    (before or in the middle of the chunks) reports CM_CAPACITY and the size
    needed."""
    import ctypes
    import torch
    from paper_2502_11602_b200 import _native
    if chunks:
        monkeypatch.setenv("CMGPU_CHUNKS", chunks)
    cloud, _ = cfg0
    q = np.ascontiguousarray(cloud[:600_000 if r < 2 else 100_000])
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    orow, ocols = cfg0_oracle.radius_csr(q, 0, r)
    qh = torch.from_numpy(q).pin_memory()
    row = torch.zeros(q.shape[0] + 1, dtype=torch.int64).pin_memory()
    cols = torch.zeros(len(ocols), dtype=torch.int32).pin_memory()
    nnz = ctypes.c_uint64()
    L = _native.lib()
    rc = L.cm_radius_search_to_host(m.handle, ctypes.c_void_p(qh.data_ptr()), q.shape[0], 0, r,
                                    ctypes.c_void_p(row.data_ptr()),
                                    ctypes.c_void_p(cols.data_ptr()), cols.numel(),
                                    ctypes.byref(nnz), None)
    assert rc == 0 and nnz.value == len(ocols)
    assert np.array_equal(row.numpy().astype(np.uint64), orow)
    assert np.array_equal(cols.numpy().astype(np.uint32), ocols)
    small = np.zeros(10, dtype=np.uint32)
    rc = L.cm_radius_search_to_host(m.handle, q.ctypes.data_as(ctypes.c_void_p), q.shape[0], 0,
                                    r, ctypes.c_void_p(row.data_ptr()),
                                    small.ctypes.data_as(ctypes.c_void_p), 10, ctypes.byref(nnz),
                                    None)
    assert rc == 3 and nnz.value == len(ocols)
    half = torch.zeros(len(ocols) // 2, dtype=torch.int32).pin_memory()
    rc = L.cm_radius_search_to_host(m.handle, ctypes.c_void_p(qh.data_ptr()), q.shape[0], 0, r,
                                    ctypes.c_void_p(row.data_ptr()),
                                    ctypes.c_void_p(half.data_ptr()), half.numel(),
                                    ctypes.byref(nnz), None)
    assert rc == 3 and nnz.value == len(ocols)
    assert np.array_equal(row.numpy().astype(np.uint64), orow)  # row pointers still complete


@pytest.mark.parametrize("order", ["cells", "x"])
def test_wide_radius_clustered_handles(cfg0, cfg0_oracle, order):
    """Wide-fill rows whose handles are clustered (a cloud stored in cell or x
    order): the bucket-rank row sort sees skewed buckets (rank scans over many
    values, or the bitonic fallback) and must still equal the oracle."""
    cloud, _ = cfg0
    if order == "cells":
        key = np.floor(cloud[:, 0]) * 1e4 + np.floor(cloud[:, 1])
    else:
        key = cloud[:, 0]
    c2 = np.ascontiguousarray(cloud[np.argsort(key, kind="stable")][:300000])
    q = c2[(c2[:, 0] < c2[:, 0].min() + 30) & (c2[:, 1] < c2[:, 1].min() + 30)]
    q = np.ascontiguousarray(q[:6000])
    o = CpuIndex(c2, flavor=1)
    m = cm.Cheesemap.build(c2, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    for r in (2.5, 3.5):
        row, cols = cm.radius_search_batch(m, q, r, cm.SPHERE)
        orow, ocols = o.radius_csr(q, 0, r)
        assert np.array_equal(row, orow) and np.array_equal(cols, ocols)


def test_csr_digest_checker(cfg0, cfg0_oracle):
    """cm_csr_digest (the full-size verification of a device CSR) reproduces
    the digest pass and flags an unsorted row."""
    import ctypes

    import torch

    from paper_2502_11602_b200 import _native
    L = _native.lib()
    cloud, q = cfg0
    q = np.ascontiguousarray(q[:5000])
    m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    row, cols = cm.radius_search_batch(m, q, 2.5, cm.SPHERE, device_out=True)
    nq = q.shape[0]
    cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
    dig = torch.empty(nq, dtype=torch.int64, device="cuda")
    bad = ctypes.c_uint64()

    def check():
        cm._check(L.cm_csr_digest(ctypes.c_void_p(row.data_ptr()), ctypes.c_void_p(cols.data_ptr()),
                                  nq, ctypes.c_void_p(cnt.data_ptr()),
                                  ctypes.c_void_p(dig.data_ptr()), ctypes.byref(bad), None))

    check()
    c2, d2 = cm.radius_digest_batch(m, q, 2.5, cm.SPHERE)
    assert bad.value == 0
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint32), c2)
    assert np.array_equal(dig.cpu().numpy().view(np.uint64), d2)
    # swap two handles of a long row
    r0 = int(torch.argmax(row[1:] - row[:-1]).item())
    b = int(row[r0].item())
    cols[b], cols[b + 1] = cols[b + 1].clone(), cols[b].clone()
    check()
    assert bad.value == 1


def test_self_queries_explicit(cfg0, cfg0_oracle):
    """cm_radius_search_self: every indexed point a centre, row q = point q;
    centres come from the index's records (no key sort; range-corner radii
    materialise them). Results equal the oracle's with the cloud as centres.
    A batch that merely shares the build buffer's address takes the general
    path: rewriting that buffer changes the centres, not the index."""
    import torch

    cloud, _ = cfg0
    d = torch.from_numpy(np.ascontiguousarray(cloud)).cuda()
    for flavor in FLAVORS:
        m = cm.Cheesemap.build(d, cm.BuildOptions(flavor=flavor))
        for kernel, r in ((cm.SPHERE, 1.0), (cm.CUBE, 1.0), (cm.SPHERE, 2.5), (cm.SPHERE, 0.4)):
            row, cols = cm.radius_search_self(m, r, kernel)
            orow, ocols = cfg0_oracle.radius_csr(cloud, int(kernel), r)
            assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
        idx, d2 = cm.knn_batch(m, d[:4000], 8)
        oidx, od2 = cfg0_oracle.knn(cloud[:4000], 8)
        assert np.array_equal(idx, oidx) and np.array_equal(d2, od2)
    # rewrite the build buffer (reversed points): same address and size, other centres
    rev = np.ascontiguousarray(cloud[::-1])
    d.copy_(torch.from_numpy(rev))
    row, cols = cm.radius_search_batch(m, d, 1.0, cm.SPHERE)
    orow, ocols = cfg0_oracle.radius_csr(rev, 0, 1.0)
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
    # the index owns its points: self queries still answer the original cloud
    row, cols = cm.radius_search_self(m, 1.0)
    orow, ocols = cfg0_oracle.radius_csr(cloud, 0, 1.0)
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)


def test_torch_inputs_are_validated(cfg0):
    """Torch buffers are passed by address, so a wrong dtype or width must be
    refused before the native code reads it (float32 points, (n, 4) points,
    int16 counts, a tensor on another device)."""
    import torch

    cloud, _ = cfg0
    m = cm.Cheesemap.build(cloud[:5000], cm.BuildOptions(flavor=cm.Flavor.Sparse))
    good = torch.from_numpy(np.ascontiguousarray(cloud[:100])).cuda()
    with pytest.raises(cm.InvalidArgumentError):
        cm.radius_search_batch(m, good.float(), 1.0)
    with pytest.raises(cm.InvalidArgumentError):
        cm.radius_search_batch(m, torch.zeros((10, 4), dtype=torch.float64, device="cuda"), 1.0)
    with pytest.raises(cm.InvalidArgumentError):
        cm.radius_count(m, good, 1.0, counts=torch.zeros(100, dtype=torch.int16, device="cuda"))
    with pytest.raises(cm.InvalidArgumentError):
        cm.radius_count(m, good, 1.0, counts=torch.zeros(10, dtype=torch.int32, device="cuda"))
    c = torch.zeros(100, dtype=torch.int32, device="cuda")
    cm.radius_count(m, good, 1.0, counts=c)
    assert int(c.sum().item()) > 0
