"""Every device code path once, on small inputs, against the CPU oracle —
run with the checked library (device invariant checks compiled in):

    make -C paper_2502_11602_b200/csrc checked
    CMGPU_LIB=libcmgpu_checked.so python scripts/checked_probe.py

compute-sanitizer is closed on this pool's GPUs (profiles/r02/
sanitizer_unavailable.log), so out-of-bounds evidence is the CM_DCHECK
invariants (common.cuh: span bounds, arena / row / flush bounds, count-pass
vs fill-pass row lengths, gather row lengths, slab pack bounds, kNN list
bounds) — a failed check traps and the process exits non-zero — plus the
oracle comparisons below.

Builds (dense / sparse / mixed, 3D and 2D), radius count / fill / single-pass
collect + gather / digest / self queries / the large-radius count + fill +
row-sort path / the one-query-per-warp path (sparse random centres), kNN
(tile path k <= 8 and the shell walk), the brute-force baselines, the
density metrics, LAS decode, the host-buffer pipeline and a 2-rank x-slab
build (in-process transport).
"""
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import CpuIndex  # noqa: E402
from paper_2502_11602_b200 import _native  # noqa: E402
from paper_2502_11602_b200 import cheesemap as cm  # noqa: E402
from paper_2502_11602_b200 import synth  # noqa: E402


def main():
    import torch

    cloud = synth.config_cloud(1, scale=0.002)  # 40k points, ~1 building
    n = cloud.shape[0]
    rng = np.random.default_rng(3)
    q = np.ascontiguousarray(cloud[rng.choice(n, 3000, replace=False)])
    far = np.array([[1e6, 1e6, 1e6]])
    qs = np.ascontiguousarray(np.concatenate([q, far]))
    checks = 0
    for flavor in (cm.Flavor.Dense, cm.Flavor.Sparse, cm.Flavor.Mixed):
        m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
        o = CpuIndex(cloud, flavor=int(flavor))
        for kernel in (cm.SPHERE, cm.CUBE):
            for r in (0.3, 1.0, 3.0):
                row, cols = cm.radius_search_batch(m, qs, r, kernel)
                orow, ocols = o.radius_csr(qs, int(kernel), r)
                assert np.array_equal(row, orow) and np.array_equal(cols, ocols), (flavor, kernel, r)
                c, dg = cm.radius_digest_batch(m, qs, r, kernel)
                oc, od = o.radius(qs, int(kernel), r)
                assert np.array_equal(c, oc) and np.array_equal(dg, od)
                checks += 2
        _native.query_stats(reset=True)
        cnt = cm.radius_count(m, qs, 1.0)
        assert np.array_equal(cnt, o.radius(qs, 0, 1.0)[0])
        # the tile counters live in this (checked) library only
        st = _native.query_stats()
        assert st["count_tiles"] > 0 and st["in_range"] > 0, st
        row, cols = cm.radius_search_self(m, 1.0)
        orow, ocols = o.radius_csr(cloud, 0, 1.0)
        assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
        for k in (1, 8, 16, 32, 64, 70):
            idx, d2 = cm.knn_batch(m, qs[:600], k)
            oidx, od2 = o.knn(qs[:600], k)
            assert np.array_equal(idx, oidx) and np.array_equal(d2, od2), (flavor, k)
            checks += 1
        del m
    # 2D mode (cylinder kernel through the density metric)
    v, bins = cm.weighted_density(cloud, sample_size=2000, sample_seed=5)
    from oracle.oracle import weighted_density as owd
    ov, obins = owd(cloud, 2000, 5)
    assert v == ov and np.array_equal(bins, obins)
    cm.global_density(cloud)
    # brute-force baselines
    c, dg = cm.brute_radius(cloud, q[:200], 1.0)
    o = CpuIndex(cloud, flavor=1)
    oc, od = o.radius(q[:200], 0, 1.0)
    assert np.array_equal(c, oc) and np.array_equal(dg, od)
    idx, d2 = cm.brute_knn(cloud, q[:100], 16)
    oidx, od2 = o.knn(q[:100], 16)
    assert np.array_equal(idx, oidx) and np.array_equal(d2, od2)
    # host-buffer pipeline (chunked, streamed to host)
    os.environ["CMGPU_CHUNKS"] = "3"
    m = cm.Cheesemap.build(torch.from_numpy(cloud).cuda(), cm.BuildOptions(flavor=cm.Flavor.Mixed))
    L = cm._native.lib()
    import ctypes
    nq = q.shape[0]
    orow, ocols = o.radius_csr(q, 0, 1.0)
    row = np.zeros(nq + 1, dtype=np.uint64)
    cols = np.zeros(int(orow[-1]), dtype=np.uint32)
    nnz = ctypes.c_uint64()
    cm._check(L.cm_radius_search_to_host(m.handle, q.ctypes.data_as(ctypes.c_void_p), nq, 0, 1.0,
                                         row.ctypes.data_as(ctypes.c_void_p),
                                         cols.ctypes.data_as(ctypes.c_void_p), cols.size,
                                         ctypes.byref(nnz), None))
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
    # LAS decode
    raw = np.array([[12345, -200, 0], [0, 1, 2], [-7, 2 ** 31 - 1, -2 ** 31]], dtype=np.int32)
    hdr = bytearray(227)
    hdr[0:4], hdr[24], hdr[25] = b"LASF", 1, 2
    struct.pack_into("<HI", hdr, 94, 227, 227)
    struct.pack_into("<BHI", hdr, 104, 0, 20, raw.shape[0])
    struct.pack_into("<3d3d", hdr, 131, 0.01, 0.01, 0.01, 100.0, 100.0, 100.0)
    recs = np.zeros((raw.shape[0], 5), dtype=np.int32)
    recs[:, :3] = raw
    xyz, _ = cm.decode_las(bytes(hdr) + recs.tobytes())
    assert np.array_equal(xyz, raw.astype(np.float64) * 0.01 + 100.0)
    # x-slabs: 2 ranks as threads (in-process transport), rows in global ids
    import threading
    from paper_2502_11602_b200.cluster import Cluster, Slab
    uid = Cluster.unique_id("in-process")
    res, errs = {}, []

    def rank_main(rk):
        try:
            cl = Cluster(uid, 2, rk, 0, "in-process")
            lo, hi = n * rk // 2, n * (rk + 1) // 2
            sl = Slab(cl, cloud[lo:hi], gid_base=lo, halo=3.0,
                      opts=cm.BuildOptions(flavor=cm.Flavor.Sparse))
            res[rk] = (sl.owned_ids(), sl.radius_digest(2.0))
        except Exception as ex:  # noqa: BLE001
            errs.append(repr(ex))

    th = [threading.Thread(target=rank_main, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    oc, od = o.radius(cloud, 0, 2.0)
    for rk in range(2):
        ids, (c, dg) = res[rk]
        assert np.array_equal(c, oc[ids]) and np.array_equal(dg, od[ids])
    checks += 1
    print(f"checked probe ok ({checks} parity checks, library {cm._native.LIB_PATH})")


if __name__ == "__main__":
    main()
