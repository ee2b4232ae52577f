"""TEST INFRASTRUCTURE — ctypes loader for the CPU oracle (liboracle.so,
the restatement) and the compiled reference (_ref/libcheesemap_ref.so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
Both libraries export the same ABI (prefix ``orc_`` / ``ref_``)."""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
STATUS = {0: "OK", 1: "EMPTY_CLOUD", 2: "INVALID_ARGUMENT", 3: "CAPACITY", 4: "OUT_OF_DOMAIN"}


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class CpuIndexLib:
    def __init__(self, which="oracle"):
        if which == "oracle":
            path, pre = os.path.join(_HERE, "liboracle.so"), "orc_"
        elif which == "reference":
            path, pre = os.path.join(_HERE, "_ref", "libcheesemap_ref.so"), "ref_"
        else:
            raise ValueError(which)
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.which, self.path = which, path
        lib = ctypes.CDLL(path)
        u64, u32, dbl, p, i = (ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double,
                               ctypes.c_void_p, ctypes.c_int)
        def f(name, args, res):
            fn = getattr(lib, pre + name)
            fn.argtypes, fn.restype = args, res
            return fn
        self.build_ = f("build", [p, u64, i, i, dbl, dbl, dbl, dbl, u64, ctypes.POINTER(p)], i)
        self.free_ = f("free", [p], None)
        self.grid_ = f("grid", [p, p, p, p, p, p], None)
        self.non_empty_ = f("non_empty", [p], u64)
        self.slice_flags_ = f("slice_flags", [p, p, p], u64)
        self.memory_report_ = f("memory_report", [p, p], None)
        self.export_ = f("export", [p, p, p], None)
        self.radius_ = f("radius", [p, p, u64, i, dbl, ctypes.c_uint, p, p, p, p], i)
        self.radius_fill_ = f("radius_fill", [p, p, u64, i, dbl, ctypes.c_uint, p, p], i)
        self.knn_ = f("knn", [p, p, u64, u32, ctypes.c_uint, p, p, p, p], i)
        self.weighted_density_ = f("weighted_density",
                                   [p, u64, u64, u64, ctypes.c_uint, ctypes.POINTER(dbl), p], i)
        self.lib = lib


_LIBS = {}


def lib(which="oracle"):
    if which not in _LIBS:
        _LIBS[which] = CpuIndexLib(which)
    return _LIBS[which]


class CpuIndex:
    """A built CPU index (restatement or reference)."""

    def __init__(self, xyz, flavor=0, mode=1, cell=(1.0, 1.0, 1.0), tau=0.8,
                 dense_cap=1 << 32, which="oracle", bounds=None):
        self.L = lib(which)
        self.xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        h = ctypes.c_void_p()
        if bounds is not None:  # explicit grid box (restatement only)
            b6 = np.ascontiguousarray(np.asarray(bounds, dtype=np.float64).reshape(6))
            fn = self.L.lib.orc_build_in_bounds
            fn.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                           ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                           ctypes.c_uint64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
            fn.restype = ctypes.c_int
            rc = fn(_p(self.xyz), self.xyz.shape[0], flavor, mode, cell[0], cell[1], cell[2], tau,
                    dense_cap, _p(b6), ctypes.byref(h))
        else:
            rc = self.L.build_(_p(self.xyz), self.xyz.shape[0], flavor, mode, cell[0], cell[1],
                               cell[2], tau, dense_cap, ctypes.byref(h))
        if rc != 0:
            raise RuntimeError(f"{which} build failed: {STATUS.get(rc, rc)}", rc)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.free_(self.h)
            self.h = None

    def grid(self):
        o, c, b0, b1 = (np.zeros(3) for _ in range(4))
        d = np.zeros(3, dtype=np.uint64)
        self.L.grid_(self.h, _p(o), _p(c), _p(d), _p(b0), _p(b1))
        return dict(origin=o, cell=c, dims=d, bmin=b0, bmax=b1)

    def non_empty(self):
        return int(self.L.non_empty_(self.h))

    def slice_flags(self):
        nz = int(self.grid()["dims"][2])
        dense = np.zeros(nz, dtype=np.uint8)
        ne = np.zeros(nz, dtype=np.uint64)
        got = self.L.slice_flags_(self.h, _p(dense), _p(ne))
        return dense[:got].astype(bool), ne[:got]

    def export(self):
        n = self.xyz.shape[0]
        k = np.zeros(n, dtype=np.uint64)
        h = np.zeros(n, dtype=np.uint64)
        self.L.export_(self.h, _p(k), _p(h))
        return k, h

    def radius(self, q, kernel=0, r=1.0, threads=0, stats=False):
        q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 3)
        nq = q.shape[0]
        cnt = np.zeros(nq, dtype=np.uint32)
        dig = np.zeros(nq, dtype=np.uint64)
        pt = np.zeros(nq, dtype=np.uint64) if stats else None
        vv = np.zeros(nq, dtype=np.uint64) if stats else None
        rc = self.L.radius_(self.h, _p(q), nq, kernel, r, threads, _p(cnt), _p(dig), _p(pt), _p(vv))
        if rc:
            raise RuntimeError(STATUS.get(rc, rc))
        return (cnt, dig, pt, vv) if stats else (cnt, dig)

    def memory_report(self):
        out = np.zeros(3, dtype=np.uint64)
        self.L.memory_report_(self.h, _p(out))
        return dict(handle_bytes=int(out[0]), structure_bytes=int(out[1]),
                    total_bytes=int(out[2]))

    def radius_csr(self, q, kernel=0, r=1.0, threads=0):
        q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 3)
        cnt, _ = self.radius(q, kernel, r, threads)
        row = np.zeros(q.shape[0] + 1, dtype=np.uint64)
        np.cumsum(cnt, out=row[1:])
        cols = np.zeros(int(row[-1]), dtype=np.uint32)
        rc = self.L.radius_fill_(self.h, _p(q), q.shape[0], kernel, r, threads, _p(row), _p(cols))
        if rc:
            raise RuntimeError(STATUS.get(rc, rc))
        return row, cols

    def knn(self, q, k, threads=0, stats=False):
        q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 3)
        nq = q.shape[0]
        idx = np.zeros((nq, k), dtype=np.uint32)
        d2 = np.zeros((nq, k), dtype=np.float64)
        prk = np.zeros(nq, dtype=np.uint64) if stats else None
        pa2 = np.zeros(nq, dtype=np.uint64) if stats else None
        rc = self.L.knn_(self.h, _p(q), nq, k, threads, _p(idx), _p(d2), _p(prk), _p(pa2))
        if rc:
            raise RuntimeError(STATUS.get(rc, rc))
        return (idx, d2, prk, pa2) if stats else (idx, d2)


def weighted_density(xyz, sample_size=0, seed=0, which="oracle", threads=0):
    """(value, bins[256]) from the restatement or the reference."""
    L = lib(which)
    xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
    v = ctypes.c_double()
    bins = np.zeros(256, dtype=np.uint64)
    rc = L.weighted_density_(_p(xyz), xyz.shape[0], sample_size, seed, threads, ctypes.byref(v),
                             _p(bins))
    if rc:
        raise RuntimeError(STATUS.get(rc, rc), rc)
    return v.value, bins


# ---- read_las / write_las (io.cpp:33-166) -----------------------------------
class LasHeader(ctypes.Structure):  # orc_las_header / ref_las_header
    _fields_ = [("version_major", ctypes.c_uint8), ("version_minor", ctypes.c_uint8),
                ("point_format", ctypes.c_uint8), ("header_size", ctypes.c_uint16),
                ("record_length", ctypes.c_uint16), ("data_offset", ctypes.c_uint32),
                ("point_count", ctypes.c_uint64), ("scale", ctypes.c_double * 3),
                ("offset", ctypes.c_double * 3), ("bounds_min", ctypes.c_double * 3),
                ("bounds_max", ctypes.c_double * 3)]


def las_read(image=None, path=None, which="oracle", name=None):
    """-> (status, message, header LasHeader, xyz or None). The restatement
    reads an in-memory image (`image`, or the file at `path`); the reference
    reads `path` through its own read_las."""
    L = lib(which).lib
    h = LasHeader()
    msg = ctypes.create_string_buffer(512)
    if which == "oracle":
        if image is None:
            with open(path, "rb") as f:
                image = f.read()
        buf = np.frombuffer(bytes(image), dtype=np.uint8)
        fn = L.orc_las_read
        fn.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.POINTER(LasHeader),
                       ctypes.c_void_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int]
        fn.restype = ctypes.c_int
        nm = os.fsencode(name if name is not None else (path or "<memory>"))
        rc = fn(buf.ctypes.data_as(ctypes.c_void_p), buf.size, nm, ctypes.byref(h), None, 0, msg,
                512)
        if rc != 0:
            return rc, msg.value.decode(), h, None
        xyz = np.empty((h.point_count, 3), dtype=np.float64)
        rc = fn(buf.ctypes.data_as(ctypes.c_void_p), buf.size, nm, ctypes.byref(h), _p(xyz),
                xyz.shape[0], msg, 512)
        return rc, msg.value.decode(), h, (xyz if rc == 0 else None)
    fn = L.ref_las_read
    fn.argtypes = [ctypes.c_char_p, ctypes.POINTER(LasHeader), ctypes.c_void_p, ctypes.c_uint64,
                   ctypes.c_char_p, ctypes.c_int]
    fn.restype = ctypes.c_int
    rc = fn(os.fsencode(path), ctypes.byref(h), None, 0, msg, 512)
    if rc != 0:
        return rc, msg.value.decode(), h, None
    xyz = np.empty((h.point_count, 3), dtype=np.float64)
    rc = fn(os.fsencode(path), ctypes.byref(h), _p(xyz), xyz.shape[0], msg, 512)
    return rc, msg.value.decode(), h, (xyz if rc == 0 else None)


def las_write_reference(xyz, path, scale=0.001):
    """The reference's write_las (io.cpp:108-166)."""
    L = lib("reference").lib
    fn = L.ref_las_write
    fn.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_double,
                   ctypes.c_char_p, ctypes.c_int]
    fn.restype = ctypes.c_int
    a = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
    msg = ctypes.create_string_buffer(512)
    rc = fn(_p(a), a.shape[0], os.fsencode(path), scale, msg, 512)
    if rc != 0:
        raise RuntimeError(f"ref write_las failed ({rc}): {msg.value.decode()}")


def generate_reference(text):
    """The reference's parse_synthetic_spec + generate -> (status, msg, xyz),
    run in a child process (oracle/ref_spec.py explains why)."""
    import subprocess
    import sys
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "spec.bin")
        subprocess.run([sys.executable, os.path.join(_HERE, "ref_spec.py"), text, out],
                       check=True)
        raw = open(out, "rb").read()
    l1 = raw.index(b"\n")
    l2 = raw.index(b"\n", l1 + 1)
    rc, n = (int(v) for v in raw[:l1].split())
    msg = raw[l1 + 1:l2].decode()
    if rc != 0:
        return rc, msg, None
    return rc, msg, np.frombuffer(raw[l2 + 1:], dtype=np.float64).reshape(n, 3).copy()
