"""ctypes binding of libcmgpu.so (include/cmgpu.h).

The product path: there is no CPU fallback. Loading fails loudly when the
library is missing; calls fail loudly when no CUDA device is present.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CMGPU_LIB=libcmgpu_checked.so selects the build with device invariant
# checks (make -C csrc checked); the default is the product library
LIB_PATH = os.path.join(_HERE, os.environ.get("CMGPU_LIB", "libcmgpu.so"))

STATUS_NAMES = {0: "CM_OK", 1: "CM_EMPTY_CLOUD", 2: "CM_INVALID_ARGUMENT", 3: "CM_CAPACITY",
                4: "CM_OUT_OF_DOMAIN", 5: "CM_CUDA", 6: "CM_NCCL", 7: "CM_PARSE", 8: "CM_IO"}

EXPORTS = [
    "cm_default_options", "cm_build", "cm_build_in_bounds", "cm_free", "cm_get_grid", "cm_get_occupancy",
    "cm_get_build_timing", "cm_export_voxels", "cm_size", "cm_radius_count", "cm_radius_fill",
    "cm_radius_search", "cm_radius_search_to_host", "cm_csr_info", "cm_csr_download", "cm_csr_free", "cm_csr_digest", "cm_radius_digest",
    "cm_knn", "cm_corrupt_for_testing", "cm_last_error", "cm_status_name",
    "cm_get_last_query_timing", "cm_launch_count", "cm_debug_query_stats", "cm_debug_pool_bytes",
    "cm_global_density", "cm_weighted_density", "cm_las_parse_header", "cm_las_decode",
    "cm_las_read", "cm_get_memory_report", "cm_brute_radius", "cm_brute_knn",
]


class LasHeaderC(ctypes.Structure):  # cm_las_header
    _fields_ = [("version_major", ctypes.c_uint8), ("version_minor", ctypes.c_uint8),
                ("point_format", ctypes.c_uint8), ("header_size", ctypes.c_uint16),
                ("record_length", ctypes.c_uint16), ("data_offset", ctypes.c_uint32),
                ("point_count", ctypes.c_uint64), ("scale", ctypes.c_double * 3),
                ("offset", ctypes.c_double * 3), ("bounds_min", ctypes.c_double * 3),
                ("bounds_max", ctypes.c_double * 3)]

    def as_dict(self):
        d = {}
        for k, _ in self._fields_:
            v = getattr(self, k)
            d[k] = list(v) if hasattr(v, "__len__") else int(v)
        return d


class MemoryReportC(ctypes.Structure):  # cm_memory_report
    _fields_ = [("handle_bytes", ctypes.c_uint64), ("structure_bytes", ctypes.c_uint64),
                ("total_bytes", ctypes.c_uint64), ("device_bytes", ctypes.c_uint64)]


class BuildOptionsC(ctypes.Structure):
    _fields_ = [("flavor", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("cell_x", ctypes.c_double), ("cell_y", ctypes.c_double),
                ("cell_z", ctypes.c_double), ("reorder", ctypes.c_int32),
                ("densify_threshold", ctypes.c_double), ("dense_voxel_cap", ctypes.c_uint64)]


class GridParamsC(ctypes.Structure):
    _fields_ = [("origin", ctypes.c_double * 3), ("cell", ctypes.c_double * 3),
                ("nx", ctypes.c_uint64), ("ny", ctypes.c_uint64), ("nz", ctypes.c_uint64),
                ("mode", ctypes.c_int32), ("bounds_min", ctypes.c_double * 3),
                ("bounds_max", ctypes.c_double * 3)]


class OccupancyC(ctypes.Structure):
    _fields_ = [("total_voxels", ctypes.c_uint64), ("non_empty", ctypes.c_uint64),
                ("empty_fraction", ctypes.c_double), ("n_slices", ctypes.c_uint64),
                ("n_columns", ctypes.c_uint64)]


class BuildTimingC(ctypes.Structure):
    _fields_ = [("total_ms", ctypes.c_double), ("h2d_ms", ctypes.c_double),
                ("bbox_ms", ctypes.c_double), ("keys_ms", ctypes.c_double),
                ("sort_ms", ctypes.c_double), ("gather_ms", ctypes.c_double),
                ("tables_ms", ctypes.c_double), ("sort_passes", ctypes.c_uint32)]


class QueryTimingC(ctypes.Structure):
    _fields_ = [("order_ms", ctypes.c_double), ("pass1_ms", ctypes.c_double),
                ("rowsort_ms", ctypes.c_double), ("scan_ms", ctypes.c_double),
                ("pass2_ms", ctypes.c_double), ("total_ms", ctypes.c_double),
                ("nq", ctypes.c_uint64), ("nnz", ctypes.c_uint64), ("two_pass", ctypes.c_int32)]


_LIB = None


class SlabTimingC(ctypes.Structure):  # cm_slab_timing
    _fields_ = [("total_ms", ctypes.c_double), ("wall_ms", ctypes.c_double),
                ("index_ms", ctypes.c_double), ("sent_points", ctypes.c_uint64),
                ("received_points", ctypes.c_uint64)]


class SlabInfoC(ctypes.Structure):  # cm_slab_info_t
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("n_local", ctypes.c_uint64), ("n_owned", ctypes.c_uint64),
                ("n_halo", ctypes.c_uint64), ("halo", ctypes.c_double),
                ("bounds", ctypes.c_double * 6), ("timing", SlabTimingC)]


CLUSTER_ID_BYTES = 128
TRANSPORT_NCCL, TRANSPORT_IN_PROCESS = 0, 1


def lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing; build it with __graft_entry__.build() "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    p, u64, u32, i32, dbl = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int,
                             ctypes.c_double)
    sig = {
        "cm_default_options": ([ctypes.POINTER(BuildOptionsC)], None),
        "cm_build": ([p, u64, ctypes.POINTER(BuildOptionsC), i32, p, ctypes.POINTER(p)], i32),
        "cm_build_in_bounds": ([p, u64, ctypes.POINTER(BuildOptionsC), p, p, i32, p,
                                ctypes.POINTER(p)], i32),
        "cm_free": ([p], i32),
        "cm_get_grid": ([p, ctypes.POINTER(GridParamsC)], i32),
        "cm_get_occupancy": ([p, ctypes.POINTER(OccupancyC), p, p, u64], i32),
        "cm_get_build_timing": ([p, ctypes.POINTER(BuildTimingC)], i32),
        "cm_export_voxels": ([p, p, p], i32),
        "cm_size": ([p], u64),
        "cm_radius_count": ([p, p, u64, i32, dbl, p, p, p], i32),
        "cm_radius_fill": ([p, p, u64, i32, dbl, p, p, p], i32),
        "cm_radius_search": ([p, p, u64, i32, dbl, p, ctypes.POINTER(p)], i32),
        "cm_radius_search_self": ([p, i32, dbl, p, ctypes.POINTER(p)], i32),
        "cm_kernel_search": ([p, i32, p, u64, p, ctypes.POINTER(p)], i32),
        "cm_kernel_count": ([p, i32, p, u64, p, p, p, p], i32),
        "cm_voxel_lookup": ([p, u64, u64, u64, ctypes.POINTER(ctypes.c_int), p, u64,
                             ctypes.POINTER(u64)], i32),
        "cm_pool_configure": ([i32, u64, u64], i32),
        "cm_csr_info": ([p, ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(p),
                         ctypes.POINTER(p)], i32),
        "cm_csr_download": ([p, p, p, p], i32),
        "cm_csr_free": ([p], i32),
        "cm_csr_digest": ([p, p, u64, p, p, ctypes.POINTER(u64), p], i32),
        "cm_radius_search_to_host": ([p, p, u64, i32, dbl, p, p, u64, ctypes.POINTER(u64), p], i32),
        "cm_radius_digest": ([p, p, u64, i32, dbl, p, p, p], i32),
        "cm_knn": ([p, p, u64, u32, p, p, p], i32),
        "cm_global_density": ([p, u64, i32, p, ctypes.POINTER(dbl)], i32),
        "cm_weighted_density": ([p, u64, u64, u64, i32, p, ctypes.POINTER(dbl), p], i32),
        "cm_corrupt_for_testing": ([p], i32),
        "cm_last_error": ([], ctypes.c_char_p),
        "cm_status_name": ([i32], ctypes.c_char_p),
        "cm_get_last_query_timing": ([ctypes.POINTER(QueryTimingC)], i32),
        "cm_launch_count": ([], u64),
        "cm_debug_query_stats": ([p, i32], i32),
        "cm_debug_pool_bytes": ([i32, i32, p, p], i32),
        "cm_las_parse_header": ([p, u64, ctypes.POINTER(LasHeaderC)], i32),
        "cm_get_memory_report": ([p, ctypes.POINTER(MemoryReportC)], i32),
        "cm_brute_radius": ([p, u64, p, u64, i32, dbl, p, p, i32, p], i32),
        "cm_brute_knn": ([p, u64, p, u64, u32, p, p, i32, p], i32),
        "cm_las_decode": ([p, u64, p, u64, ctypes.POINTER(LasHeaderC), i32, p], i32),
        "cm_las_read": ([ctypes.c_char_p, p, u64, ctypes.POINTER(LasHeaderC), i32, p], i32),
        "cm_cluster_unique_id": ([i32, p], i32),
        "cm_cluster_init": ([i32, p, i32, i32, i32, ctypes.POINTER(p)], i32),
        "cm_cluster_free": ([p], i32),
        "cm_build_slab": ([p, p, p, u64, u64, ctypes.POINTER(BuildOptionsC), dbl, p,
                           ctypes.POINTER(p)], i32),
        "cm_slab_free": ([p], i32),
        "cm_slab_info": ([p, ctypes.POINTER(SlabInfoC), p, u64], i32),
        "cm_slab_index": ([p], p),
        "cm_slab_ids": ([p, p, p, p], i32),
        "cm_slab_radius_search": ([p, p, u64, i32, dbl, p, ctypes.POINTER(p)], i32),
        "cm_slab_radius_digest": ([p, p, u64, i32, dbl, p, p, p], i32),
    }
    # CMGPU_ALLOW_MISSING=1: bind what an older library build exports (A/B
    # measurements against earlier versions); the product binds everything
    lenient = bool(os.environ.get("CMGPU_ALLOW_MISSING"))
    for name, (args, res) in sig.items():
        try:
            fn = getattr(L, name)
        except AttributeError:
            if lenient:
                continue
            raise
        fn.argtypes, fn.restype = args, res
    _LIB = L
    return L


def last_error():
    return lib().cm_last_error().decode(errors="replace")


def last_query_timing():
    t = QueryTimingC()
    rc = lib().cm_get_last_query_timing(ctypes.byref(t))
    if rc != 0:
        raise RuntimeError(last_error())
    return {k: getattr(t, k) for k, _ in t._fields_}


def launch_count():
    return int(lib().cm_launch_count())


def query_stats(reset=True):
    import numpy as np
    out = np.zeros(8, dtype=np.uint64)
    lib().cm_debug_query_stats(out.ctypes.data_as(ctypes.c_void_p), int(reset))
    return dict(count_tiles=int(out[0]), count_fallback_tiles=int(out[1]),
                count_hull_points=int(out[2]), in_range=int(out[3]), fill_tiles=int(out[4]),
                fill_fallback_tiles=int(out[5]), fill_hull_points=int(out[6]),
                fill_long_rows=int(out[7]))


def pool_bytes(device=0, trim=False):
    """(reserved, in use) bytes of the library's device memory pool."""
    r, u = ctypes.c_uint64(), ctypes.c_uint64()
    rc = lib().cm_debug_pool_bytes(device, int(trim), ctypes.byref(r), ctypes.byref(u))
    if rc != 0:
        raise RuntimeError(f"cm_debug_pool_bytes failed ({rc})")
    return r.value, u.value
