"""The N > 1 host logic on CPU with gloo, world_size 2 and 3: global bbox
all-reduce, x-slab ownership, halo exchange, local indexing on the global
grid, and global-id assembly. Each rank indexes its slab with the CPU oracle
(on the GPU box the same SlabPartition feeds cluster.gpu_slab_index); the
union of the ranks' rows must equal the single global index's rows exactly.
Also checks the replicated layout's query sharding."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_11602_b200 import cluster, synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir, radii, halo):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import CpuIndex
        cloud = torch.from_numpy(synth.config_cloud(4, scale=0.0005))  # 100k pts, 1 building
        xyz, ids = cluster.SlabPartition.owned_from_global(cloud, rank, world)
        part = cluster.SlabPartition(xyz, ids, rank, world, halo)
        lo, hi = part.bounds()
        idx = CpuIndex(part.local_xyz.numpy(), flavor=1, bounds=np.concatenate([lo, hi]))
        q = xyz.numpy()
        res = {"qids": ids.numpy(), "n_halo": part.n_halo}
        for r in radii:
            for kern in (0, 1):
                row, cols = idx.radius_csr(q, kern, r, threads=1)
                grow, gcols = cluster.assemble_rows(row, cols, part)
                res[f"row_{kern}_{r}"] = grow
                res[f"cols_{kern}_{r}"] = gcols
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
        # replicated layout: contiguous query blocks cover the batch once
        lo_q, hi_q = cluster.query_shard(1003, rank, world)
        t = torch.tensor([hi_q - lo_q], dtype=torch.int64)
        dist.all_reduce(t)
        assert int(t.item()) == 1003
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_partition_matches_global_index(world):
    from oracle.oracle import CpuIndex
    radii = [1.0, 2.5]
    halo = 5.0
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, radii, halo), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    cloud = synth.config_cloud(4, scale=0.0005)
    qids = np.concatenate([p["qids"] for p in parts])
    assert np.array_equal(np.sort(qids), np.arange(cloud.shape[0]))  # every point owned once
    assert all(int(p["n_halo"]) > 0 for p in parts)
    glob = CpuIndex(cloud, flavor=1)
    for r in radii:
        for kern in (0, 1):
            grow, gcols = glob.radius_csr(cloud, kern, r, threads=4)
            for p in parts:
                row, cols = p[f"row_{kern}_{r}"], p[f"cols_{kern}_{r}"]
                for i, qg in enumerate(p["qids"][::97]):
                    i *= 97
                    mine = cols[row[i]:row[i + 1]]
                    want = gcols[grow[qg]:grow[qg + 1]]
                    assert np.array_equal(mine, want), (world, r, kern, qg)
                # totals per rank agree with the global rows of its queries
                assert int(row[-1]) == int(sum(grow[q + 1] - grow[q] for q in p["qids"]))
