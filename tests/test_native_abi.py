"""The C-ABI library: loads, exports every entry point include/cmgpu.h
declares, and fails loudly (no CPU fallback) when no GPU is present."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cmgpu.h")
LIB = os.path.join(ROOT, "paper_2502_11602_b200", "libcmgpu.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cm_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for want in ("cm_build", "cm_free", "cm_radius_count", "cm_radius_fill", "cm_radius_search",
                 "cm_radius_digest", "cm_knn", "cm_get_grid", "cm_get_occupancy",
                 "cm_export_voxels", "cm_corrupt_for_testing", "cm_last_error"):
        assert want in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build with __graft_entry__.build()"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\sT\s(cm_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(LIB)
    for f in declared_functions():
        assert getattr(lib, f) is not None


def test_library_targets_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_no_fma_in_predicate_kernels():
    """-fmad=false: the sphere predicate ((dx*dx + dy*dy) + dz*dz <= r*r,
    geometry.hpp:26-31) must not be contracted into DFMA. The only DFMAs in
    the query kernels are inside IEEE division (axis_index, grid.cpp:31),
    which is correctly rounded by construction; so each sphere kernel has
    exactly as many DFMAs as its cube twin (whose predicate has no multiply)."""
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    counts = {}
    for b in sass.split("Function : ")[1:]:
        name = b.split("\n", 1)[0]
        m = re.search(r"radius_tile_kernelILi(\d)ELi(\d)ELi(\d)ELb(\d)E", name)
        if m:
            counts[m.groups()] = b.count("DFMA")
    assert len(counts) >= 24  # with and without per-centre radii / boxes
    for (flavor, mode, cube, xq), n in counts.items():
        if cube == "0":
            assert n == counts[(flavor, mode, "1", xq)], (flavor, mode, xq)


def test_status_names_and_default_options():
    from paper_2502_11602_b200 import _native
    L = _native.lib()
    assert L.cm_status_name(0) == b"CM_OK"
    assert L.cm_status_name(3) == b"CM_CAPACITY"
    o = _native.BuildOptionsC()
    L.cm_default_options(ctypes.byref(o))
    assert (o.flavor, o.mode, o.cell_x, o.densify_threshold, o.dense_voxel_cap) == \
        (0, 1, 1.0, 0.8, 1 << 32)


def test_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2502_11602_b200 import cheesemap as cm
    with pytest.raises(cm.CudaError):
        cm.Cheesemap.build(np.zeros((10, 3)))
