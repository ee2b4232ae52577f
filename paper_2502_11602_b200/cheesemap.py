"""Host-side mirror of the reference's C++ index API over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/core/include/cheesemap/{geometry,grid,map,search,errors}.hpp
so parity tests read like the reference's own tests:

  reference (C++)                               here
  Cheesemap::build(cloud, BuildOptions)          Cheesemap.build(cloud, BuildOptions())
  map.grid() / occupancy_stats()                 Cheesemap.grid() / .occupancy_stats()
  kernel_search(map, SphereKernel{c, r})         kernel_search(map, SphereKernel(c, r))
  kernel_search(map, BoxKernel{{lo},{hi}})       kernel_search(map, BoxKernel(lo, hi))
  knn_search(map, c, k)                          knn_search(map, c, k)
  cheesemap::EmptyCloudError, ...                EmptyCloudError, ...

plus the batched calls the reference lacks (radius_search_batch,
radius_digest_batch, knn_batch). Inputs may be numpy arrays (host) or CUDA
torch tensors (device); the C ABI stages host buffers itself.
"""
import ctypes
import os
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _native


# ---------------------------------------------------------------- errors --
class Error(RuntimeError):
    """cheesemap::Error (errors.hpp:8-11)."""


class EmptyCloudError(Error):
    pass


class InvalidArgumentError(Error):
    pass


class CapacityError(Error):
    pass


class OutOfDomainError(Error):
    pass


class CudaError(Error):
    pass


class NcclError(Error):
    pass


class ParseError(Error):  # errors.hpp:29-32
    pass


class IoError(Error):  # errors.hpp:39-42
    pass


_ERRORS = {1: EmptyCloudError, 2: InvalidArgumentError, 3: CapacityError, 4: OutOfDomainError,
           5: CudaError, 6: NcclError, 7: ParseError, 8: IoError}


def _check(status):
    if status != 0:
        raise _ERRORS.get(status, Error)(f"{_native.STATUS_NAMES.get(status, status)}: "
                                         f"{_native.last_error()}")


# ----------------------------------------------------------------- types --
class Flavor(IntEnum):  # map.hpp:15
    Dense = 0
    Sparse = 1
    Mixed = 2


class GridMode(IntEnum):  # grid.hpp:10
    TwoD = 0
    ThreeD = 1


@dataclass
class CellSize:  # grid.hpp:15-21
    x: float = 1.0
    y: float = 1.0
    z: float = 1.0

    @staticmethod
    def uniform(s):
        return CellSize(s, s, s)


@dataclass
class BuildOptions:  # map.hpp:17-26
    flavor: Flavor = Flavor.Dense
    mode: GridMode = GridMode.ThreeD
    cell: CellSize = field(default_factory=CellSize)
    reorder: bool = False
    densify_threshold: float = 0.80
    dense_voxel_cap: int = 1 << 32

    def to_c(self):
        c = _native.BuildOptionsC()
        c.flavor, c.mode = int(self.flavor), int(self.mode)
        c.cell_x, c.cell_y, c.cell_z = self.cell.x, self.cell.y, self.cell.z
        c.reorder = int(bool(self.reorder))
        c.densify_threshold = self.densify_threshold
        c.dense_voxel_cap = self.dense_voxel_cap
        return c


@dataclass
class SphereKernel:  # geometry.hpp:73-85
    center: tuple
    radius: float


@dataclass
class BoxKernel:  # geometry.hpp:87-92: any axis-aligned box, closed on all faces
    min: tuple
    max: tuple

    @staticmethod
    def cube(center, r):  # the cube the reference CLI builds (cmd_bench.cpp:107-111)
        c = [float(v) for v in center]
        return BoxKernel(tuple(v - r for v in c), tuple(v + r for v in c))


@dataclass
class CylinderKernel:  # geometry.hpp:97-113 (z range unbounded by default)
    center_x: float
    center_y: float
    radius: float
    z_lo: float = float("-inf")
    z_hi: float = float("inf")


@dataclass
class QueryStats:  # search.hpp:12-17
    voxels_visited: int = 0
    points_tested: int = 0
    growth_iterations: int = 0
    final_radius: float = 0.0


class GrowthPolicy(IntEnum):  # search.hpp:88 (the device kNN is exact for either)
    Density = 0
    Monotonic = 1


@dataclass
class Neighbor:  # search.hpp:19-24 (distance = sqrt of the fp64 d^2)
    handle: int
    distance: float


SPHERE, CUBE, CYLINDER = 0, 1, 2


# -------------------------------------------------------------- buffers --
def _is_torch(x):
    return type(x).__module__.startswith("torch")


# torch dtypes the native code may read as each element type (same width;
# torch has no unsigned 32/64-bit tensors in most builds, so the signed twins
# are accepted and reinterpreted)
_TORCH_DTYPES = {np.dtype(np.float64): ("float64",),
                 np.dtype(np.uint32): ("int32", "uint32"),
                 np.dtype(np.uint64): ("int64", "uint64")}


def _in_ptr(x, dtype=np.float64, device=None, output=False):
    """Pointer to a host (numpy) or device (torch) buffer, plus a keepalive.

    Torch tensors are passed by address, so they must already have the
    element type the C ABI reads (float64 points, u32 counts, u64 stats) and,
    for points, 3 values per row; a CUDA tensor must live on the index's
    device. Anything else raises InvalidArgumentError instead of letting the
    native code read n*24 bytes out of a smaller buffer. Outputs must be
    contiguous (a copy would not be written back)."""
    if x is None:
        return None, None
    dt = np.dtype(dtype)
    if _is_torch(x):
        tname = str(x.dtype).replace("torch.", "")
        if tname not in _TORCH_DTYPES[dt]:
            raise InvalidArgumentError(f"tensor dtype {x.dtype} where {dt.name} is expected")
        if dt == np.float64 and not (x.dim() == 2 and x.shape[1] == 3) and \
                not (x.dim() == 1 and x.shape[0] % 3 == 0):
            raise InvalidArgumentError(f"points must be (n, 3) float64, got {tuple(x.shape)}")
        if x.is_cuda and device is not None and x.device.index != device:
            raise InvalidArgumentError(f"tensor on {x.device}, index on cuda:{device}")
        if not x.is_contiguous():
            if output:
                raise InvalidArgumentError("output tensor must be contiguous")
            x = x.contiguous()
        return ctypes.c_void_p(x.data_ptr()), x
    if output:
        if not (isinstance(x, np.ndarray) and x.dtype == dt and x.flags.c_contiguous):
            raise InvalidArgumentError(f"output array must be contiguous {dt.name}")
        return x.ctypes.data_as(ctypes.c_void_p), x
    a = np.ascontiguousarray(x, dtype=dtype)
    if dt == np.float64 and not (a.ndim == 2 and a.shape[1] == 3) and \
            not (a.ndim == 1 and a.shape[0] % 3 == 0):
        raise InvalidArgumentError(f"points must be (n, 3) float64, got {a.shape}")
    return a.ctypes.data_as(ctypes.c_void_p), a


def _stream_ptr(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def _nrows(q):
    return int(q.shape[0]) if len(q.shape) == 2 else int(q.shape[0]) // 3


# ---------------------------------------------------------------- index --
class Cheesemap:
    """Device-resident cheesemap (map.hpp:53-151). Immutable once built;
    owns its device copies of the points."""

    def __init__(self, handle, opts, device, n):
        self._h = handle
        self._opts = opts
        self.device = device
        self._n = n

    @staticmethod
    def build(cloud, opts=None, device=0, stream=None):
        opts = opts or BuildOptions()
        L = _native.lib()
        p, keep = _in_ptr(cloud, device=device)
        n = _nrows(keep) if keep is not None else 0
        h = ctypes.c_void_p()
        c = opts.to_c()
        _check(L.cm_build(p, n, ctypes.byref(c), device, _stream_ptr(stream), ctypes.byref(h)))
        return Cheesemap(h, opts, device, n)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _native.lib().cm_free(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def flavor(self):
        return self._opts.flavor

    def mode(self):
        return self._opts.mode

    def size(self):
        return self._n

    def grid(self):
        g = _native.GridParamsC()
        _check(_native.lib().cm_get_grid(self._h, ctypes.byref(g)))
        return dict(origin=tuple(g.origin), cell=tuple(g.cell), nx=g.nx, ny=g.ny, nz=g.nz,
                    mode=GridMode(g.mode), bounds_min=tuple(g.bounds_min),
                    bounds_max=tuple(g.bounds_max))

    def occupancy_stats(self):
        """OccupancyStats (map.hpp:34-39) + per-slice mixed flags."""
        nz = self.grid()["nz"]
        dense = np.zeros(nz, dtype=np.uint8)
        ne = np.zeros(nz, dtype=np.uint64)
        o = _native.OccupancyC()
        _check(_native.lib().cm_get_occupancy(self._h, ctypes.byref(o),
                                              dense.ctypes.data_as(ctypes.c_void_p),
                                              ne.ctypes.data_as(ctypes.c_void_p), nz))
        return dict(total_voxels=o.total_voxels, non_empty=o.non_empty,
                    empty_fraction=o.empty_fraction, n_columns=o.n_columns,
                    slice_dense=dense.astype(bool), slice_non_empty=ne)

    def memory_report(self):
        """MemoryReport (map.hpp:41-48): the reference's analytic byte model,
        plus device_bytes (this index's actual HBM)."""
        r = _native.MemoryReportC()
        _check(_native.lib().cm_get_memory_report(self._h, ctypes.byref(r)))
        return {k: int(getattr(r, k)) for k, _ in r._fields_}

    def voxel_present(self, v):
        """Cheesemap::voxel_present (map.hpp:62-63) for v = (i, j, k)."""
        n, pres = ctypes.c_uint64(), ctypes.c_int()
        _check(_native.lib().cm_voxel_lookup(self._h, int(v[0]), int(v[1]), int(v[2]),
                                             ctypes.byref(pres), None, 0, ctypes.byref(n)))
        return bool(pres.value)

    def voxel_lookup(self, v):
        """Cheesemap::voxel_lookup (map.hpp:65-67): the voxel's handles
        (ascending), or None when the voxel is not materialized."""
        L = _native.lib()
        n, pres = ctypes.c_uint64(), ctypes.c_int()
        _check(L.cm_voxel_lookup(self._h, int(v[0]), int(v[1]), int(v[2]), ctypes.byref(pres),
                                 None, 0, ctypes.byref(n)))
        if not pres.value:
            return None
        out = np.zeros(n.value, dtype=np.uint32)
        if n.value:
            _check(L.cm_voxel_lookup(self._h, int(v[0]), int(v[1]), int(v[2]), ctypes.byref(pres),
                                     out.ctypes.data_as(ctypes.c_void_p), out.size,
                                     ctypes.byref(n)))
        return out.astype(np.uint64)

    def reordered(self):
        return bool(self._opts.reorder)

    def structure_name(self):
        return structure_name(self._opts.flavor, self._opts.mode, self._opts.reorder)

    def build_timing(self):
        t = _native.BuildTimingC()
        _check(_native.lib().cm_get_build_timing(self._h, ctypes.byref(t)))
        return {k: getattr(t, k) for k, _ in t._fields_}

    def export_voxels(self):
        """(keys u64, handles u32) in stored order (per-voxel handle sets)."""
        keys = np.zeros(self._n, dtype=np.uint64)
        hs = np.zeros(self._n, dtype=np.uint32)
        _check(_native.lib().cm_export_voxels(self._h, keys.ctypes.data_as(ctypes.c_void_p),
                                              hs.ctypes.data_as(ctypes.c_void_p)))
        return keys, hs

    def corrupt_for_testing(self):
        _check(_native.lib().cm_corrupt_for_testing(self._h))


def structure_name(flavor, mode, reordered=False):
    """structure_name (map.cpp:225-238): "dense3", "mixed2-reordered", ..."""
    name = ["dense", "sparse", "mixed"][int(flavor)] + ("3" if int(mode) == 1 else "2")
    return name + ("-reordered" if reordered else "")


# -------------------------------------------------------------- queries --
def _kernel_params(kernels):
    """Explicit kernels of one type -> (kind, params rows) for cm_kernel_search."""
    k0 = kernels[0]
    if isinstance(k0, SphereKernel):
        rows = [[*map(float, k.center), float(k.radius)] for k in kernels]
        return SPHERE, np.asarray(rows, dtype=np.float64).reshape(-1, 4)
    if isinstance(k0, BoxKernel):
        rows = [[*map(float, k.min), *map(float, k.max)] for k in kernels]
        return CUBE, np.asarray(rows, dtype=np.float64).reshape(-1, 6)
    if isinstance(k0, CylinderKernel):
        rows = [[k.center_x, k.center_y, k.radius, k.z_lo, k.z_hi] for k in kernels]
        return CYLINDER, np.asarray(rows, dtype=np.float64).reshape(-1, 5)
    raise InvalidArgumentError("kernel must be SphereKernel, BoxKernel or CylinderKernel")


def kernel_search_batch(m, kernels, stats=False, stream=None):
    """kernel_search over explicit kernels of one type (each with its own
    radius / box / z range): sorted CSR (row_ptr, cols), plus the per-kernel
    (points_tested, voxels_visited) when stats=True."""
    kind, prm = _kernel_params(list(kernels))
    L = _native.lib()
    nq = prm.shape[0]
    csr = ctypes.c_void_p()
    _check(L.cm_kernel_search(m.handle, kind, prm.ctypes.data_as(ctypes.c_void_p), nq,
                              _stream_ptr(stream), ctypes.byref(csr)))
    row, cols = _take_csr(L, csr, nq, m.device, stream, False)
    if not stats:
        return row, cols
    pt = np.zeros(nq, dtype=np.uint64)
    vv = np.zeros(nq, dtype=np.uint64)
    _check(L.cm_kernel_count(m.handle, kind, prm.ctypes.data_as(ctypes.c_void_p), nq, None,
                             pt.ctypes.data_as(ctypes.c_void_p), vv.ctypes.data_as(ctypes.c_void_p),
                             _stream_ptr(stream)))
    return row, cols, pt, vv


def radius_count(m, centers, r, kernel=SPHERE, counts=None, points_tested=None, stream=None):
    """Per-centre neighbour counts (and QueryStats::points_tested)."""
    qp, qk = _in_ptr(centers, device=m.device)
    nq = _nrows(qk)
    if counts is None:
        counts = np.zeros(nq, dtype=np.uint32)
    cp, ck = _in_ptr(counts, np.uint32, device=m.device, output=True)
    tp, tk = (_in_ptr(points_tested, np.uint64, device=m.device, output=True)
              if points_tested is not None else (None, None))
    for o in (ck, tk):
        if o is not None and (o.numel() if _is_torch(o) else o.size) < nq:
            raise InvalidArgumentError("output buffer holds fewer than one entry per centre")
    _check(_native.lib().cm_radius_count(m.handle, qp, nq, kernel, float(r), cp, tp,
                                         _stream_ptr(stream)))
    return counts if not isinstance(counts, np.ndarray) else ck


def radius_search_batch(m, centers, r, kernel=SPHERE, stream=None, device_out=False):
    """Sorted CSR of kernel_search over every centre: (row_ptr u64[nq+1],
    cols u32[nnz]) as numpy arrays, or as CUDA torch tensors when
    device_out=True. centers=None: every indexed point is a centre (row q =
    point q, cm_radius_search_self)."""
    L = _native.lib()
    csr = ctypes.c_void_p()
    if centers is None:
        nq = m.size()
        _check(L.cm_radius_search_self(m.handle, kernel, float(r), _stream_ptr(stream),
                                       ctypes.byref(csr)))
    else:
        qp, qk = _in_ptr(centers, device=m.device)
        nq = _nrows(qk)
        _check(L.cm_radius_search(m.handle, qp, nq, kernel, float(r), _stream_ptr(stream),
                                  ctypes.byref(csr)))
    return _take_csr(L, csr, nq, m.device, stream, device_out)


def radius_search_self(m, r, kernel=SPHERE, stream=None, device_out=False):
    """Every indexed point as a centre: radius_search_batch(m, None, ...)."""
    return radius_search_batch(m, None, r, kernel, stream, device_out)


def pool_configure(device=0, keep_bytes=0, reserve_bytes=0):
    """cm_pool_configure: how much device memory the library's private pool
    keeps cached across synchronisations, and an up-front reservation."""
    _check(_native.lib().cm_pool_configure(int(device), int(keep_bytes), int(reserve_bytes)))


def _take_csr(L, csr, nq, device, stream, device_out):
    try:
        nnz = ctypes.c_uint64()
        _check(L.cm_csr_info(csr, None, ctypes.byref(nnz), None, None))
        if device_out:
            import torch
            row = torch.empty(nq + 1, dtype=torch.int64, device=f"cuda:{device}")
            cols = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=f"cuda:{device}")
            _check(L.cm_csr_download(csr, ctypes.c_void_p(row.data_ptr()),
                                     ctypes.c_void_p(cols.data_ptr()), _stream_ptr(stream)))
            return row, cols[: nnz.value]
        row = np.zeros(nq + 1, dtype=np.uint64)
        cols = np.zeros(nnz.value, dtype=np.uint32)
        _check(L.cm_csr_download(csr, row.ctypes.data_as(ctypes.c_void_p),
                                 cols.ctypes.data_as(ctypes.c_void_p), _stream_ptr(stream)))
        return row, cols
    finally:
        L.cm_csr_free(csr)


def radius_digest_batch(m, centers, r, kernel=SPHERE, stream=None):
    """Per-centre (count u32, digest u64 = sum(mix64(handle)))."""
    qp, qk = _in_ptr(centers, device=m.device)
    nq = _nrows(qk)
    counts = np.zeros(nq, dtype=np.uint32)
    dig = np.zeros(nq, dtype=np.uint64)
    _check(_native.lib().cm_radius_digest(m.handle, qp, nq, kernel, float(r),
                                          counts.ctypes.data_as(ctypes.c_void_p),
                                          dig.ctypes.data_as(ctypes.c_void_p),
                                          _stream_ptr(stream)))
    return counts, dig


def knn_batch(m, centers, k, stream=None, device_out=False):
    """(idx u32[nq, k], d2 f64[nq, k]) ordered by (d^2, handle); with
    device_out=True, CUDA tensors (int32 / float64) that stay on the device."""
    qp, qk = _in_ptr(centers, device=m.device)
    nq = _nrows(qk)
    if device_out:
        import torch
        dev = f"cuda:{m.device}"
        idx = torch.empty((nq, k), dtype=torch.int32, device=dev)
        d2 = torch.empty((nq, k), dtype=torch.float64, device=dev)
        _check(_native.lib().cm_knn(m.handle, qp, nq, int(k), ctypes.c_void_p(idx.data_ptr()),
                                    ctypes.c_void_p(d2.data_ptr()), _stream_ptr(stream)))
        return idx, d2
    idx = np.zeros((nq, k), dtype=np.uint32)
    d2 = np.zeros((nq, k), dtype=np.float64)
    _check(_native.lib().cm_knn(m.handle, qp, nq, int(k), idx.ctypes.data_as(ctypes.c_void_p),
                                d2.ctypes.data_as(ctypes.c_void_p), _stream_ptr(stream)))
    return idx, d2


def kernel_search(m, kernel, stats=None):
    """kernel_search (search.hpp:102-127) for one kernel: the handles inside
    it, sorted ascending; a QueryStats passed as `stats` gets the reference's
    voxels_visited / points_tested."""
    if stats is None:
        _, cols = kernel_search_batch(m, [kernel])
    else:
        _, cols, pt, vv = kernel_search_batch(m, [kernel], stats=True)
        stats.points_tested, stats.voxels_visited = int(pt[0]), int(vv[0])
        stats.growth_iterations, stats.final_radius = 0, 0.0
    return cols.astype(np.uint64)


def knn_search(m, c, k, policy=GrowthPolicy.Density, stats=None):
    """knn_search (search.cpp:87-146): min(k, N) nearest, by (d^2, handle).
    Exact for either policy; `stats` gets the candidates of kernel_search at
    the exact k-th distance (points_tested, voxels_visited) and that distance
    as final_radius."""
    if k == 0:
        raise InvalidArgumentError("k must be at least 1")
    idx, d2 = knn_batch(m, np.asarray(c, dtype=np.float64).reshape(1, 3), k)
    out = [Neighbor(int(i), float(np.sqrt(d))) for i, d in zip(idx[0], d2[0])
           if i != 0xFFFFFFFF]
    if stats is not None:
        r = out[-1].distance if out else 0.0
        _, _, pt, vv = kernel_search_batch(m, [SphereKernel(tuple(map(float, c)), r)], stats=True)
        stats.points_tested, stats.voxels_visited = int(pt[0]), int(vv[0])
        stats.growth_iterations, stats.final_radius = 0, r
    return out


# -------------------------------------------------------------- analysis --
def global_density(cloud, device=0):
    """global_density (analysis.cpp:17-24): points per m^2 of the xy box."""
    p, keep = _in_ptr(cloud)
    v = ctypes.c_double()
    _check(_native.lib().cm_global_density(p, _nrows(keep), device, None, ctypes.byref(v)))
    return v.value


def weighted_density(cloud, sample_size=None, sample_seed=0, device=0):
    """weighted_density (analysis.cpp:26-86) -> (value, bins[256])."""
    p, keep = _in_ptr(cloud)
    v = ctypes.c_double()
    bins = np.zeros(256, dtype=np.uint64)
    _check(_native.lib().cm_weighted_density(p, _nrows(keep), int(sample_size or 0),
                                             int(sample_seed), device, None, ctypes.byref(v),
                                             bins.ctypes.data_as(ctypes.c_void_p)))
    return v.value, bins


# ------------------------------------------------------------- io.hpp ------
def las_header(image):
    """Header of an in-memory LAS image (bytes-like, host): read_las's header
    checks (io.cpp:38-89) without decoding -> dict (cm_las_header fields)."""
    buf = np.frombuffer(bytes(image) if not isinstance(image, np.ndarray) else image,
                        dtype=np.uint8)
    h = _native.LasHeaderC()
    _check(_native.lib().cm_las_parse_header(buf.ctypes.data_as(ctypes.c_void_p), buf.size,
                                             ctypes.byref(h)))
    return h.as_dict()


def decode_las(image, device_out=False, device=0, stream=None):
    """read_las on an in-memory LAS image (bytes-like host buffer, or a CUDA
    uint8 tensor): (cloud (n, 3) float64, header dict). The records are
    decoded on the device; device_out=True returns a CUDA tensor."""
    if _is_torch(image):
        ptr, nbytes, keep = ctypes.c_void_p(image.data_ptr()), image.numel(), image
    else:
        keep = np.frombuffer(bytes(image) if not isinstance(image, np.ndarray) else image,
                             dtype=np.uint8)
        ptr, nbytes = keep.ctypes.data_as(ctypes.c_void_p), keep.size
    h = _native.LasHeaderC()
    L = _native.lib()
    _check(L.cm_las_decode(ptr, nbytes, None, 0, ctypes.byref(h), device, None))
    n = int(h.point_count)
    out = _alloc_points(n, device_out, device)
    _check(L.cm_las_decode(ptr, nbytes, _out_ptr(out), n, ctypes.byref(h), device,
                           _stream_ptr(stream)))
    return out, h.as_dict()


def read_las(path, device_out=False, device=0, stream=None):
    """read_las(path) (io.hpp:39-42): IoError when the file cannot be opened,
    ParseError (the reference's messages) when it is malformed."""
    h = _native.LasHeaderC()
    L = _native.lib()
    bpath = os.fsencode(path)
    _check(L.cm_las_read(bpath, None, 0, ctypes.byref(h), device, None))
    n = int(h.point_count)
    out = _alloc_points(n, device_out, device)
    _check(L.cm_las_read(bpath, _out_ptr(out), n, ctypes.byref(h), device, _stream_ptr(stream)))
    return out, h.as_dict()


def _alloc_points(n, device_out, device):
    if device_out:
        import torch
        return torch.empty((n, 3), dtype=torch.float64, device=f"cuda:{device}")
    return np.empty((n, 3), dtype=np.float64)


def _out_ptr(a):
    if _is_torch(a):
        return ctypes.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ctypes.c_void_p)


# -------------------------------------------------------- baseline.hpp ------
def brute_radius(cloud, centers, r, kernel=SPHERE, device=0, stream=None):
    """brute_radius (baseline.hpp:11-21) on the device: every point tested
    against every centre -> (counts u32[nq], digests u64[nq])."""
    pp, pk = _in_ptr(cloud)
    qp, qk = _in_ptr(centers, device=device)
    nq = _nrows(qk)
    counts = np.zeros(nq, dtype=np.uint32)
    digests = np.zeros(nq, dtype=np.uint64)
    _check(_native.lib().cm_brute_radius(pp, _nrows(pk), qp, nq, int(kernel), float(r),
                                         counts.ctypes.data_as(ctypes.c_void_p),
                                         digests.ctypes.data_as(ctypes.c_void_p), device,
                                         _stream_ptr(stream)))
    return counts, digests


def brute_knn(cloud, centers, k, device=0, stream=None):
    """brute_knn (baseline.cpp:8-25) on the device, ordered by (d^2, handle):
    (idx u32[nq, k], d2 f64[nq, k]); k <= 64."""
    pp, pk = _in_ptr(cloud)
    qp, qk = _in_ptr(centers, device=device)
    nq = _nrows(qk)
    idx = np.zeros((nq, k), dtype=np.uint32)
    d2 = np.zeros((nq, k), dtype=np.float64)
    _check(_native.lib().cm_brute_knn(pp, _nrows(pk), qp, nq, int(k),
                                      idx.ctypes.data_as(ctypes.c_void_p),
                                      d2.ctypes.data_as(ctypes.c_void_p), device,
                                      _stream_ptr(stream)))
    return idx, d2
