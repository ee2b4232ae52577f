"""Multi-GPU layouts: one process per GPU.

The product path for x-slabs is the C ABI (include/cmgpu.h "Multi-GPU",
csrc/cluster.cu): `Cluster` + `Slab` below wrap cm_cluster_init /
cm_build_slab / cm_slab_radius_search — device bbox, NCCL MIN all-reduce,
device classify + pack, NCCL grouped send/recv, local index on the global
grid, results in global ids. The torch.distributed helpers further down
restate the same partition rule on the host (SlabPartition) for the gloo
multi-process tests and as the oracle-side reference of the partition.

Two layouts:

* Replicated index (configs 1-3): every rank holds the whole index and
  answers a contiguous block of the queries (`query_shard`). There is no
  data-path collective; totals are summed at the end.

* x-slabs with a halo (config 4): the cloud's global bounding box is
  all-reduced (MIN/MAX of 6 doubles), the x extent is cut into `world`
  equal slabs, rank s owns the points with x in its slab, and the points
  within `halo` metres of each slab face are exchanged with the neighbour
  slab (point-to-point send/recv, counts first). Each rank indexes owned +
  halo points ON THE GLOBAL GRID (cm_build_in_bounds), so every voxel key and
  clamped range is the one the single global index would use; a query owned
  by the rank then sees exactly the global candidate set inside
  [x - r, x + r] as long as r <= halo, and its neighbour set equals the
  global one. Local handles are assigned in ascending global-id order, so
  sorted local rows stay sorted after mapping back to global ids.
"""
import ctypes

import numpy as np
import torch
import torch.distributed as dist


class Cluster:
    """cm_cluster: this rank's membership of a group of `nranks` ranks.
    transport: "nccl" (one GPU per rank; `uid` from Cluster.unique_id on rank
    0, passed to every rank by the caller) or "in-process" (ranks are host
    threads of this process)."""

    TRANSPORTS = {"nccl": 0, "in-process": 1}

    def __init__(self, uid, nranks, rank, device=0, transport="nccl"):
        from . import _native
        from . import cheesemap as cm
        self._L = _native.lib()
        self.nranks, self.rank, self.device = nranks, rank, device
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(bytes(uid), _native.CLUSTER_ID_BYTES)
        cm._check(self._L.cm_cluster_init(self.TRANSPORTS[transport], buf, nranks, rank, device,
                                          ctypes.byref(h)))
        self._h = h

    @staticmethod
    def unique_id(transport="nccl"):
        from . import _native
        from . import cheesemap as cm
        buf = ctypes.create_string_buffer(_native.CLUSTER_ID_BYTES)
        cm._check(_native.lib().cm_cluster_unique_id(Cluster.TRANSPORTS[transport], buf))
        return buf.raw

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.cm_cluster_free(h)
            self._h = None


class Slab:
    """cm_slab: this rank's x-slab index (owned + halo points, global grid)."""

    def __init__(self, cluster, xyz, gids=None, gid_base=0, opts=None, halo=5.0, stream=None):
        from . import cheesemap as cm
        opts = opts or cm.BuildOptions()
        self.cluster = cluster
        L = cluster._L
        p, keep = cm._in_ptr(xyz, device=cluster.device)
        n = cm._nrows(keep) if keep is not None else 0
        gp, gkeep = cm._in_ptr(gids, np.uint32, device=cluster.device) if gids is not None \
            else (None, None)
        h = ctypes.c_void_p()
        c = opts.to_c()
        cm._check(L.cm_build_slab(cluster._h, p, gp, int(gid_base), n, ctypes.byref(c),
                                  float(halo), cm._stream_ptr(stream), ctypes.byref(h)))
        self._h = h
        self._L = L
        self.opts = opts

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.cm_slab_free(h)
            self._h = None

    def info(self):
        from . import _native
        from . import cheesemap as cm
        o = _native.SlabInfoC()
        e = np.zeros(self.cluster.nranks + 1)
        cm._check(self._L.cm_slab_info(self._h, ctypes.byref(o), e.ctypes.data_as(ctypes.c_void_p),
                                       e.size))
        t = o.timing
        return dict(nranks=o.nranks, rank=o.rank, n_local=o.n_local, n_owned=o.n_owned,
                    n_halo=o.n_halo, halo=o.halo, bounds=list(o.bounds), edges=e,
                    timing=dict(total_ms=t.total_ms, wall_ms=t.wall_ms, index_ms=t.index_ms,
                                sent_points=t.sent_points, received_points=t.received_points))

    def owned_ids(self):
        from . import cheesemap as cm
        n = int(self.info()["n_owned"])
        out = np.zeros(n, dtype=np.uint32)
        cm._check(self._L.cm_slab_ids(self._h, out.ctypes.data_as(ctypes.c_void_p), None, None))
        return out

    def radius_search(self, r, kernel=0, centers=None, stream=None, device_out=False):
        """Sorted CSR in global ids; centers=None: every owned point (row i =
        owned_ids()[i])."""
        from . import cheesemap as cm
        L = self._L
        if centers is None:
            qp, nq = None, int(self.info()["n_owned"])
        else:
            qp, qk = cm._in_ptr(centers, device=self.cluster.device)
            nq = cm._nrows(qk)
        csr = ctypes.c_void_p()
        cm._check(L.cm_slab_radius_search(self._h, qp, nq, int(kernel), float(r),
                                          cm._stream_ptr(stream), ctypes.byref(csr)))
        return cm._take_csr(L, csr, nq, self.cluster.device, stream, device_out)

    def radius_digest(self, r, kernel=0, centers=None, stream=None):
        from . import cheesemap as cm
        if centers is None:
            qp, nq = None, int(self.info()["n_owned"])
        else:
            qp, qk = cm._in_ptr(centers, device=self.cluster.device)
            nq = cm._nrows(qk)
        cnt = np.zeros(nq, dtype=np.uint32)
        dig = np.zeros(nq, dtype=np.uint64)
        cm._check(self._L.cm_slab_radius_digest(self._h, qp, nq, int(kernel), float(r),
                                                cnt.ctypes.data_as(ctypes.c_void_p),
                                                dig.ctypes.data_as(ctypes.c_void_p),
                                                cm._stream_ptr(stream)))
        return cnt, dig


def query_shard(n, rank, world):
    """[lo, hi) of the contiguous query block of `rank`."""
    return n * rank // world, n * (rank + 1) // world


def global_bbox(xyz, group=None):
    """(6,) float64 tensor: all-reduced per-axis min then max
    (aabb_of_points, geometry.cpp:7-21, over the union of the ranks)."""
    if xyz.shape[0]:
        lo = xyz.min(0).values
        hi = xyz.max(0).values
    else:
        lo = torch.full((3,), float("inf"), dtype=torch.float64, device=xyz.device)
        hi = torch.full((3,), float("-inf"), dtype=torch.float64, device=xyz.device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    return torch.cat([lo, hi])


def slab_edges(bbox, world):
    """world + 1 x coordinates; slab s is [e[s], e[s+1]) (the last one closed)."""
    lo, hi = float(bbox[0]), float(bbox[3])
    e = [lo + (hi - lo) * s / world for s in range(world)] + [hi]
    return torch.tensor(e, dtype=torch.float64)


def slab_owner(x, edges):
    """Owning slab of each x coordinate (tensor of int64)."""
    inner = edges[1:-1].to(x.device)
    return torch.searchsorted(inner, x.contiguous(), right=True)


def exchange_halo(xyz, ids, rank, world, edges, halo, group=None):
    """Send the owned points within `halo` of each slab face to that
    neighbour; receive theirs. Returns (halo_xyz, halo_ids)."""
    dev = xyz.device
    x = xyz[:, 0]
    lo_face, hi_face = float(edges[rank]), float(edges[rank + 1])
    send = {}
    if rank > 0:
        m = x < lo_face + halo
        send[rank - 1] = (xyz[m].contiguous(), ids[m].contiguous())
    if rank < world - 1:
        m = x >= hi_face - halo
        send[rank + 1] = (xyz[m].contiguous(), ids[m].contiguous())
    peers = sorted(send)
    # counts first
    cnt_out = {p: torch.tensor([send[p][1].numel()], dtype=torch.int64, device=dev) for p in peers}
    cnt_in = {p: torch.zeros(1, dtype=torch.int64, device=dev) for p in peers}
    ops = []
    for p in peers:
        ops.append(dist.P2POp(dist.isend, cnt_out[p], p, group))
        ops.append(dist.P2POp(dist.irecv, cnt_in[p], p, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    recv = {p: (torch.empty((int(cnt_in[p].item()), 3), dtype=torch.float64, device=dev),
                torch.empty(int(cnt_in[p].item()), dtype=torch.int64, device=dev)) for p in peers}
    ops = []
    for p in peers:
        if send[p][1].numel():
            ops.append(dist.P2POp(dist.isend, send[p][0], p, group))
            ops.append(dist.P2POp(dist.isend, send[p][1], p, group))
        if recv[p][1].numel():
            ops.append(dist.P2POp(dist.irecv, recv[p][0], p, group))
            ops.append(dist.P2POp(dist.irecv, recv[p][1], p, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    if not peers:
        return (torch.empty((0, 3), dtype=torch.float64, device=dev),
                torch.empty(0, dtype=torch.int64, device=dev))
    return (torch.cat([recv[p][0] for p in peers]), torch.cat([recv[p][1] for p in peers]))


class SlabPartition:
    """This rank's slab: owned points, halo points, and the local point set
    (owned + halo) in ascending global-id order, ready to index on the
    global grid."""

    def __init__(self, xyz_owned, ids_owned, rank, world, halo, group=None):
        self.rank, self.world, self.halo = rank, world, halo
        self.bbox = global_bbox(xyz_owned, group)
        self.edges = slab_edges(self.bbox.cpu(), world)
        hx, hid = exchange_halo(xyz_owned, ids_owned, rank, world, self.edges, halo, group)
        local_xyz = torch.cat([xyz_owned, hx])
        local_ids = torch.cat([ids_owned, hid])
        order = torch.argsort(local_ids)
        self.local_xyz = local_xyz[order].contiguous()
        self.local_ids = local_ids[order].contiguous()
        self.n_owned = int(ids_owned.numel())
        self.n_halo = int(hid.numel())

    @staticmethod
    def owned_from_global(cloud, rank, world, group=None):
        """The owned block of a cloud every rank can produce (deterministic
        generators): points whose x falls in this rank's slab."""
        bbox = global_bbox(cloud, group)
        edges = slab_edges(bbox.cpu(), world)
        own = slab_owner(cloud[:, 0], edges) == rank
        ids = torch.nonzero(own).flatten()
        return cloud[own].contiguous(), ids.to(torch.int64)

    def bounds(self):
        b = self.bbox.cpu().numpy()
        return b[:3].copy(), b[3:].copy()

    def to_global(self, cols_local):
        """Local handles -> global ids (order preserved: ascending)."""
        return self.local_ids[cols_local.long()]


def gpu_slab_index(part, opts=None, device=0, stream=None):
    """Index a SlabPartition on the GPU on the global grid."""
    import ctypes

    from . import _native
    from . import cheesemap as cm
    opts = opts or cm.BuildOptions()
    L = _native.lib()
    lo, hi = part.bounds()
    h = ctypes.c_void_p()
    xyz = part.local_xyz.contiguous()
    c = opts.to_c()
    cm._check(L.cm_build_in_bounds(ctypes.c_void_p(xyz.data_ptr()), xyz.shape[0], ctypes.byref(c),
                                   lo.ctypes.data_as(ctypes.c_void_p),
                                   hi.ctypes.data_as(ctypes.c_void_p), device,
                                   cm._stream_ptr(stream), ctypes.byref(h)))
    return cm.Cheesemap(h, opts, device, xyz.shape[0])


def assemble_rows(local_row_ptr, local_cols, part):
    """Per-query CSR with global ids from a slab index's local CSR."""
    cols = part.to_global(torch.as_tensor(np.asarray(local_cols, dtype=np.int64)))
    return np.asarray(local_row_ptr, dtype=np.uint64), cols.numpy().astype(np.uint32)


class VirtualSlab:
    """Slab `rank` of `world` computed from the whole cloud in one process
    (no collectives): the same owned/halo sets SlabPartition produces, for
    running several slabs on one device (SURVEY.md §4 "virtual slab" mode)."""

    def __init__(self, cloud, rank, world, halo):
        cloud = torch.as_tensor(cloud)
        self.bbox = torch.cat([cloud.min(0).values, cloud.max(0).values])
        self.edges = slab_edges(self.bbox, world)
        x = cloud[:, 0]
        own = slab_owner(x, self.edges) == rank
        lo_face, hi_face = float(self.edges[rank]), float(self.edges[rank + 1])
        left = (slab_owner(x, self.edges) == rank - 1) & (x >= lo_face - halo) if rank > 0 else \
            torch.zeros_like(own)
        right = (slab_owner(x, self.edges) == rank + 1) & (x < hi_face + halo) \
            if rank < world - 1 else torch.zeros_like(own)
        # a neighbour sends its points within `halo` of the shared face
        local = own | left | right
        self.owned_ids = torch.nonzero(own).flatten()
        self.local_ids = torch.nonzero(local).flatten()
        self.local_xyz = cloud[self.local_ids].contiguous()
        self.n_owned = int(self.owned_ids.numel())
        self.n_halo = int(self.local_ids.numel()) - self.n_owned

    def bounds(self):
        b = self.bbox.cpu().numpy()
        return b[:3].copy(), b[3:].copy()

    def to_global(self, cols_local):
        return self.local_ids[cols_local.long()]
