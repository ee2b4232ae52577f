"""Multi-GPU x-slabs through the C ABI (cm_cluster_* / cm_build_slab /
cm_slab_radius_*). The box has one GPU, so the multi-rank
build runs with the in-process transport — 2, 3 and 4 ranks as host threads
on one device, the same bbox all-reduce, classify / pack kernels, size
all-to-all, bucket exchange, global-id sort and relabel as over NCCL, only
the byte movement differs — and NCCL runs with one rank. Every owned centre's
row (global ids) must equal the single global index's, i.e. the oracle's
(reference contracts: map.hpp:50-52 immutable map, grid.cpp:41-61 bbox
grid)."""
import threading

import numpy as np
import pytest

from paper_2502_11602_b200 import cheesemap as cm
from paper_2502_11602_b200 import synth
from paper_2502_11602_b200.cluster import Cluster, Slab
from oracle.oracle import CpuIndex

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cloud():
    return synth.config_cloud(4, scale=0.002)  # 400k points, 6400 x 6250 m^2 scaled


@pytest.fixture(scope="module")
def oracle(cloud):
    return CpuIndex(cloud, flavor=1)


def run_ranks(cloud, P, halo, flavor, split, r, kernel=cm.SPHERE):
    uid = Cluster.unique_id("in-process")
    n = cloud.shape[0]
    out = [None] * P
    errs = []

    def work(rank):
        try:
            cl = Cluster(uid, P, rank, 0, "in-process")
            if split == "contiguous":
                lo, hi = n * rank // P, n * (rank + 1) // P
                sl = Slab(cl, cloud[lo:hi], gid_base=lo, halo=halo,
                          opts=cm.BuildOptions(flavor=flavor))
            else:  # strided handles with explicit global ids
                ids = np.arange(rank, n, P, dtype=np.uint32)
                sl = Slab(cl, cloud[ids], gids=ids, halo=halo, opts=cm.BuildOptions(flavor=flavor))
            row, cols = sl.radius_search(r, kernel)
            cnt, dig = sl.radius_digest(r, kernel)
            out[rank] = dict(info=sl.info(), owned=sl.owned_ids(), row=row, cols=cols, cnt=cnt,
                             dig=dig)
            del sl, cl
        except Exception as ex:  # noqa: BLE001
            errs.append((rank, repr(ex)))

    th = [threading.Thread(target=work, args=(i,), daemon=True) for i in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a rank is stuck in a collective"
    assert not errs, errs
    return out


@pytest.mark.parametrize("P,split,flavor", [(2, "contiguous", cm.Flavor.Sparse),
                                            (3, "strided", cm.Flavor.Mixed),
                                            (4, "contiguous", cm.Flavor.Dense)])
def test_in_process_slabs_equal_global_index(cloud, oracle, P, split, flavor):
    r = 2.5
    res = run_ranks(cloud, P, 5.0, flavor, split, r)
    owned = np.concatenate([o["owned"] for o in res])
    assert np.array_equal(np.sort(owned), np.arange(cloud.shape[0], dtype=np.uint32))
    orow, ocols = oracle.radius_csr(cloud, 0, r)
    ocnt, odig = oracle.radius(cloud, 0, r)
    for o in res:
        ids = o["owned"].astype(np.int64)
        assert np.all(np.diff(ids) > 0)  # ascending global ids = row order
        inf = o["info"]
        assert inf["n_local"] == inf["n_owned"] + inf["n_halo"]
        e = inf["edges"]
        x = cloud[ids, 0]
        assert np.all(x >= e[inf["rank"]]) and (inf["rank"] == P - 1 or np.all(x < e[inf["rank"] + 1]))
        assert np.array_equal(o["cnt"], ocnt[ids]) and np.array_equal(o["dig"], odig[ids])
        lens = np.diff(o["row"].astype(np.int64))
        assert np.array_equal(lens, (orow[ids + 1] - orow[ids]).astype(np.int64))
        exp = np.concatenate([ocols[orow[i]:orow[i + 1]] for i in ids]) if ids.size else ocols[:0]
        assert np.array_equal(o["cols"], exp)


def test_slab_radius_beyond_halo_is_refused(cloud):
    uid = Cluster.unique_id("in-process")
    errs, seen = [], []

    def work(rank):
        try:
            cl = Cluster(uid, 2, rank, 0, "in-process")
            n = cloud.shape[0]
            sl = Slab(cl, cloud[rank * n // 2:(rank + 1) * n // 2], gid_base=rank * n // 2, halo=1.0)
            with pytest.raises(cm.InvalidArgumentError):
                sl.radius_search(2.5)
            seen.append(rank)
        except Exception as ex:  # noqa: BLE001
            errs.append(repr(ex))

    th = [threading.Thread(target=work, args=(i,), daemon=True) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs and sorted(seen) == [0, 1]


def test_nccl_single_rank(cloud, oracle):
    """NCCL transport, one rank: the communicator, the MIN all-reduce, the
    grouped self send/recv and the build all run through NCCL."""
    import torch

    uid = Cluster.unique_id("nccl")
    cl = Cluster(uid, 1, 0, 0, "nccl")
    d = torch.from_numpy(cloud).cuda()
    sl = Slab(cl, d, halo=5.0, opts=cm.BuildOptions(flavor=cm.Flavor.Mixed))
    inf = sl.info()
    assert inf["n_owned"] == cloud.shape[0] and inf["n_halo"] == 0
    row, cols = sl.radius_search(1.0)
    orow, ocols = oracle.radius_csr(cloud, 0, 1.0)
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
    # the slab index answers general centres in global ids too
    q = np.ascontiguousarray(cloud[::97])
    row, cols = sl.radius_search(1.0, cm.CUBE, centers=q)
    orow, ocols = oracle.radius_csr(q, 1, 1.0)
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
