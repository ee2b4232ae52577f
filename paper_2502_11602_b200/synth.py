"""Seeded synthetic inputs for the BASELINE.json configs (ctypes over the
host C++ generators in csrc/synth.cpp).

Config table (BASELINE.json ``configs``):
  0: ALS 1M pts over 250x250 m, dense, cell 1 m, queries = every 10th point
  1: ALS 20M pts over 1000x1000 m + 200 buildings, sparse/mixed, cell 1 m
  2: TLS 20000 az x 2000 el rays (40M pts), mixed, cell 0.25 m, 2M queries
  3: config-1 cloud, mixed, 5M kNN queries
  4: ALS 200M pts over 3200x3125 m + 2000 buildings, x-slabs
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

SEED_BASE = 11602


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libcmsynth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        u64, u32, dbl, p = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double, ctypes.c_void_p
        lib.cms_generate_als.argtypes = [u64, u64, dbl, dbl, u32, u32, p]
        lib.cms_generate_als.restype = ctypes.c_int
        lib.cms_als_building_points.argtypes = [u64, u64, dbl, dbl, u32]
        lib.cms_als_building_points.restype = u64
        lib.cms_generate_uniform.argtypes = [u64, u64, dbl, dbl, dbl, p]
        lib.cms_generate_uniform.restype = ctypes.c_int
        lib.cms_generate_tls.argtypes = [u64, u32, u32, u32, dbl, dbl, dbl, u32, p]
        lib.cms_generate_tls.restype = ctypes.c_int
        lib.cms_center_stream.argtypes = [u64, u64, u64, u64, p]
        lib.cms_center_stream.restype = None
        lib.cms_generate_spec.argtypes = [ctypes.c_int, u64, u64, dbl, dbl, dbl, dbl, dbl, dbl,
                                          dbl, u64, dbl, p, ctypes.c_char_p, ctypes.c_int]
        lib.cms_generate_spec.restype = ctypes.c_int
        lib.cms_center_stream_init.argtypes = [u64, u64]
        lib.cms_center_stream_init.restype = u64
        lib.cms_center_stream_next.argtypes = [ctypes.POINTER(u64), u64, u64, p]
        lib.cms_center_stream_next.restype = None
        lib.cms_mix64.argtypes = [u64]
        lib.cms_mix64.restype = u64
        _LIB = lib
    return _LIB


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def als(n, ex, ey, n_buildings=0, seed=SEED_BASE, threads=0):
    """(n, 3) float64 ALS-like cloud (terrain + 30% vegetation + buildings)."""
    out = np.empty((n, 3), dtype=np.float64)
    rc = _lib().cms_generate_als(seed, n, ex, ey, n_buildings, threads, _ptr(out))
    if rc != 0:
        raise ValueError(f"cms_generate_als failed ({rc})")
    return out


def uniform(n, ex, ey, ez, seed):
    """Bit-identical to the reference's UniformBox generator (io.cpp:266-272)."""
    out = np.empty((n, 3), dtype=np.float64)
    if _lib().cms_generate_uniform(seed, n, ex, ey, ez, _ptr(out)) != 0:
        raise ValueError("cms_generate_uniform failed")
    return out


def tls(n_az=20000, n_el=2000, n_boxes=50, seed=SEED_BASE + 2, max_range=200.0,
        scanner_z=1.5, sigma=0.002, threads=0):
    out = np.empty((n_az * n_el, 3), dtype=np.float64)
    rc = _lib().cms_generate_tls(seed, n_az, n_el, n_boxes, scanner_z, max_range, sigma,
                                 threads, _ptr(out))
    if rc != 0:
        raise ValueError(f"cms_generate_tls failed ({rc})")
    return out


def center_stream(seed, tag, cloud_size, count):
    """Query-centre indices with replacement (tools/common.cpp:109-125)."""
    out = np.empty(count, dtype=np.uint64)
    _lib().cms_center_stream(seed, tag, cloud_size, count, _ptr(out))
    return out


class CenterStream:
    """The reference's query-centre stream as an object (common.cpp:109-125):
    next(count) returns the next `count` indices."""

    def __init__(self, seed, tag, cloud_size):
        self._state = ctypes.c_uint64(_lib().cms_center_stream_init(seed, tag))
        self._n = cloud_size

    def next(self, count):
        out = np.empty(count, dtype=np.uint64)
        _lib().cms_center_stream_next(ctypes.byref(self._state), self._n, count, _ptr(out))
        return out


def mix64(x):
    return int(_lib().cms_mix64(x))


def config_cloud(cfg, scale=1.0, threads=0):
    """The cloud of BASELINE config ``cfg``; ``scale`` < 1 shrinks the point
    count and area together (same density) for quick tests."""
    if cfg == 0:
        n = int(1_000_000 * scale)
        side = 250.0 * scale ** 0.5
        return als(n, side, side, 0, SEED_BASE + 0, threads)
    if cfg in (1, 3):
        n = int(20_000_000 * scale)
        side = 1000.0 * scale ** 0.5
        nb = max(0, int(round(200 * scale)))
        return als(n, side, side, nb, SEED_BASE + 1, threads)
    if cfg == 2:
        f = scale ** 0.5
        return tls(max(1, int(20000 * f)), max(1, int(2000 * f)), 50, SEED_BASE + 2,
                   threads=threads)
    if cfg == 4:
        n = int(200_000_000 * scale)
        f = scale ** 0.5
        return als(n, 3200.0 * f, 3125.0 * f, max(0, int(round(2000 * scale))),
                   SEED_BASE + 4, threads)
    raise ValueError(cfg)


def config_queries(cfg, cloud, count=None):
    """Query centres (n, 3) for config ``cfg`` drawn from ``cloud``."""
    n = cloud.shape[0]
    if cfg == 0:
        return np.ascontiguousarray(cloud[::10])
    if cfg in (1, 4):
        return cloud
    default = {2: 2_000_000, 3: 5_000_000}[cfg]
    idx = center_stream(SEED_BASE + 100 + cfg, 0, n, count or default)
    return np.ascontiguousarray(cloud[idx.astype(np.int64)])


# ---- the reference's synthetic specs (io.hpp:44-70, io.cpp:252-399) --------
SPEC_KINDS = {"uniform": 0, "void-ellipse": 1, "clusters": 2}


def parse_synthetic_spec(text):
    """parse_synthetic_spec (io.cpp:337-399): "kind:key=value,..." -> dict.
    Raises cheesemap.ParseError with the reference's messages."""
    from .cheesemap import ParseError
    colon = text.find(":")
    if colon < 0:
        raise ParseError("synthetic spec needs the form kind:key=value,...")
    kind = text[:colon]
    if kind not in SPEC_KINDS:
        raise ParseError(f"unknown synthetic kind '{kind}'")
    spec = dict(kind=kind, n=0, seed=0, extent=(100.0, 100.0, 50.0), cx=0.0, cy=0.0, ax=0.0,
                ay=0.0, clusters=8, sigma=1.0)
    rest = text[colon + 1:]
    for item in (rest.split(",") if rest else []):
        if "=" not in item:
            raise ParseError(f"bad synthetic spec item '{item}'")
        key, value = item.split("=", 1)
        try:
            if key in ("n", "seed", "clusters"):
                v = int(value, 10) if value.strip().lstrip("+").isdigit() else None
                if v is None:
                    raise ValueError
                if v >= 1 << 64:
                    raise OverflowError
                spec[key] = v
            elif key == "extent":
                parts = value.split("x")
                if len(parts) != 3:
                    raise ParseError("extent must look like 100x100x50")
                try:
                    spec["extent"] = tuple(float(x) for x in parts)
                except ValueError:
                    raise ParseError("extent must look like 100x100x50")
            elif key in ("cx", "cy", "ax", "ay", "sigma"):
                spec[key] = float(value)
            else:
                raise ParseError(f"unknown synthetic spec key '{key}'")
        except OverflowError:
            raise ParseError(f"value out of range for synthetic spec key '{key}'")
        except ValueError:
            raise ParseError(f"bad value for synthetic spec key '{key}'")
    return spec


def generate(spec):
    """generate (io.cpp:252-335) for a parsed spec (dict or spec string):
    bit-identical to the reference for all three kinds. Raises
    cheesemap.InvalidArgumentError with the reference's messages."""
    from .cheesemap import InvalidArgumentError
    if isinstance(spec, str):
        spec = parse_synthetic_spec(spec)
    n = int(spec["n"])
    ex, ey, ez = spec["extent"]
    out = np.empty((max(n, 1), 3), dtype=np.float64)
    msg = ctypes.create_string_buffer(256)
    rc = _lib().cms_generate_spec(SPEC_KINDS[spec["kind"]], int(spec["seed"]), n, ex, ey, ez,
                                  spec["cx"], spec["cy"], spec["ax"], spec["ay"],
                                  int(spec["clusters"]), spec["sigma"], _ptr(out), msg, 256)
    if rc != 0:
        raise InvalidArgumentError(msg.value.decode())
    return out[:n]
