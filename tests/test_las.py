"""LAS ingestion (read_las, io.cpp:33-106).

Pinned like the reference's test_io.cpp: a hand-assembled LAS 1.2 file with
known coordinates (:58-72), malformed files rejected with ParseError (:74-99),
the write_las/read_las round trip (:101-118) — plus every point format's
record length, LAS 1.4 64-bit counts, extreme raw values and unaligned
images. The restatement (oracle/) is checked against the reference's own
read_las (oracle/_ref); the device decoder against both, bit for bit."""
import os
import struct

import numpy as np
import pytest

from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAS_REF = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libcheesemap_ref.so"))
needs_ref = pytest.mark.skipif(not HAS_REF, reason="oracle/_ref not built")

# point record length of formats 0-8 (LAS 1.4 R15, table 7-15)
FORMAT_LEN = {0: 20, 1: 28, 2: 26, 3: 34, 4: 57, 5: 63, 6: 30, 7: 36, 8: 38}


def make_las(raw, scale=0.001, offset=0.0, version=(1, 2), fmt=0, rl=None, header_size=227,
             data_offset=None, count=None, count64=None, extra=0, seed=0):
    """LAS image bytes, assembled field by field (independent of write_las).
    `raw` is (n, 3) int32; other record bytes are random filler."""
    raw = np.asarray(raw, dtype=np.int32).reshape(-1, 3)
    rl = rl if rl is not None else FORMAT_LEN[fmt] + extra
    data_offset = header_size if data_offset is None else data_offset
    hdr = bytearray(max(header_size, 227))
    hdr[0:4] = b"LASF"
    hdr[24], hdr[25] = version
    struct.pack_into("<H", hdr, 94, header_size)
    struct.pack_into("<I", hdr, 96, data_offset)
    hdr[104] = fmt
    struct.pack_into("<H", hdr, 105, rl)
    struct.pack_into("<I", hdr, 107, raw.shape[0] if count is None else count)
    sc = scale if isinstance(scale, (tuple, list)) else (scale,) * 3
    of = offset if isinstance(offset, (tuple, list)) else (offset,) * 3
    struct.pack_into("<3d", hdr, 131, *sc)
    struct.pack_into("<3d", hdr, 155, *of)
    struct.pack_into("<6d", hdr, 179, 1.0, -1.0, 2.0, -2.0, 3.0, -3.0)
    if count64 is not None:
        struct.pack_into("<Q", hdr, 247, count64)
    gap = bytes(max(0, data_offset - len(hdr)))
    rng = np.random.default_rng(seed)
    recs = rng.integers(0, 256, size=(raw.shape[0], rl), dtype=np.uint8)
    recs[:, 0:12] = raw.view(np.uint8).reshape(-1, 12)
    return bytes(hdr[:max(header_size, 227)]) + gap + recs.tobytes()


def write(tmp_path, name, image):
    p = tmp_path / name
    p.write_bytes(image)
    return str(p)


def rand_raw(n, seed, lo=-(2 ** 31), hi=2 ** 31 - 1):
    rng = np.random.default_rng(seed)
    raw = rng.integers(lo, hi, size=(n, 3), dtype=np.int64, endpoint=True).astype(np.int32)
    if n >= 4:
        raw[0] = [-(2 ** 31), 2 ** 31 - 1, 0]
        raw[1] = [2 ** 31 - 1, -(2 ** 31), -1]
    return raw


def bad_images():
    """(label, image) pairs the reference rejects (test_io.cpp:74-99 and the
    checks of io.cpp:44-96, one each)."""
    good = make_las([[0, 0, 0], [1, 1, 1]], 0.001, 0.0)
    cases = [("magic", b"X" + good[1:]), ("short", good[:200]), ("version9", None),
             ("version11", None), ("format9", None), ("reclen11", None), ("zero_scale", None),
             ("neg_scale_z", None), ("nan_scale", None), ("offset_below_header", None),
             ("offset_past_end", None), ("truncated", good[:-5]),
             ("truncated_first", make_las([[0, 0, 0]], 0.001, 0.0)[:230]),
             ("count_past_data", make_las([[0, 0, 0]], count=3))]
    out = []
    for label, img in cases:
        if img is None:
            b = bytearray(good)
            if label == "version9":
                b[24] = 9
            elif label == "version11":
                b[25] = 1
            elif label == "format9":
                b[104] = 9
            elif label == "reclen11":
                struct.pack_into("<H", b, 105, 11)
            elif label == "zero_scale":
                struct.pack_into("<d", b, 131, 0.0)
            elif label == "neg_scale_z":
                struct.pack_into("<d", b, 147, -0.5)
            elif label == "nan_scale":
                struct.pack_into("<d", b, 139, float("nan"))
            elif label == "offset_below_header":
                struct.pack_into("<I", b, 96, 100)
            elif label == "offset_past_end":
                struct.pack_into("<I", b, 96, len(b) + 1)
            img = bytes(b)
        out.append((label, img))
    return out


def good_images():
    out = [("known", make_las([[12345, -200, 0], [0, 1, 2]], 0.01, 100.0)),
           ("empty", make_las(np.zeros((0, 3)), 0.001, 5.0)),
           ("v13_fmt3", make_las(rand_raw(1000, 3), (0.01, 0.02, 0.001), (1e5, -3e6, 12.5),
                                 version=(1, 3), fmt=3)),
           ("v14_count64", make_las(rand_raw(777, 4), 1e-7, 0.25, version=(1, 4), fmt=6,
                                    header_size=375, count=0, count64=777)),
           ("gap_after_header", make_las(rand_raw(300, 5), 0.001, -7.0, data_offset=400))]
    for fmt in range(9):
        out.append((f"fmt{fmt}", make_las(rand_raw(513, 10 + fmt), 0.001 * (fmt + 1),
                                           1000.0 * fmt - 3.5, fmt=fmt, extra=fmt % 3)))
    return out


# ------------------------------------------------------------ CPU: pinning --
def test_known_answer_oracle():
    """test_io.cpp:58-72: raw * scale + offset."""
    img = make_las([[12345, -200, 0], [0, 1, 2]], 0.01, 100.0)
    rc, msg, h, xyz = orc.las_read(img)
    assert rc == 0
    assert xyz.shape == (2, 3)
    assert abs(xyz[0, 0] - 223.45) <= 1e-12 * 223.45 and xyz[0, 1] == 98.0 and xyz[0, 2] == 100.0
    assert abs(xyz[1, 1] - 100.01) <= 1e-12 * 100.01
    assert (h.version_minor, h.point_format, h.point_count, h.scale[0]) == (2, 0, 2, 0.01)


@needs_ref
@pytest.mark.parametrize("label,img", good_images())
def test_oracle_equals_reference_decode(tmp_path, label, img):
    path = write(tmp_path, label + ".las", img)
    a = orc.las_read(path=path)
    b = orc.las_read(path=path, which="reference")
    assert a[0] == b[0] == 0
    assert np.array_equal(a[3].view(np.uint64), b[3].view(np.uint64))  # bit for bit
    for f in ("version_major", "version_minor", "point_format", "point_count"):
        assert getattr(a[2], f) == getattr(b[2], f)
    for f in ("scale", "offset", "bounds_min", "bounds_max"):
        assert list(getattr(a[2], f)) == list(getattr(b[2], f))


@needs_ref
@pytest.mark.parametrize("label,img", bad_images())
def test_oracle_equals_reference_errors(tmp_path, label, img):
    path = write(tmp_path, label + ".las", img)
    a = orc.las_read(path=path)
    b = orc.las_read(path=path, which="reference")
    assert a[0] == b[0] == 7, (label, a[:2], b[:2])  # ParseError
    assert a[1] == b[1]


@needs_ref
def test_missing_file_is_io_error(tmp_path):
    rc, msg, _, _ = orc.las_read(path=str(tmp_path / "does_not_exist.las"), which="reference")
    assert rc == 8 and msg == "cannot open " + str(tmp_path / "does_not_exist.las")


@needs_ref
def test_write_read_round_trip(tmp_path):
    """test_io.cpp:101-118 through the reference writer; the restatement
    reads the reference's file bit for bit like the reference."""
    rng = np.random.default_rng(17)
    cloud = np.column_stack([rng.uniform(0, 100, 2000), rng.uniform(0, 100, 2000),
                             rng.uniform(0, 50, 2000)])
    path = str(tmp_path / "rt.las")
    orc.las_write_reference(cloud, path, 0.001)
    a = orc.las_read(path=path)
    b = orc.las_read(path=path, which="reference")
    assert a[0] == b[0] == 0
    assert np.array_equal(a[3], b[3])
    assert np.abs(a[3] - cloud).max() <= 0.001 / 2 + 1e-12


def test_header_parse_on_host_matches_oracle():
    """cm_las_parse_header is host code (no device): same header, same
    ParseError messages as the restatement."""
    from paper_2502_11602_b200 import cheesemap as cm
    for label, img in good_images():
        h = cm.las_header(img)
        rc, _, oh, _ = orc.las_read(img)
        assert rc == 0
        assert h["point_count"] == oh.point_count and h["record_length"] == oh.record_length
        assert h["scale"] == list(oh.scale) and h["bounds_min"] == list(oh.bounds_min)
    for label, img in bad_images():
        rc, omsg, _, _ = orc.las_read(img, name="<memory>")
        if label.startswith("truncated") or label == "count_past_data":
            continue  # record truncation is the decoder's check (io.cpp:92-96)
        with pytest.raises(cm.ParseError) as e:
            cm.las_header(img)
        assert str(e.value).endswith(omsg), (label, str(e.value), omsg)


# ------------------------------------------------------------ GPU: decode --
@pytest.mark.gpu
@pytest.mark.parametrize("label,img", good_images())
def test_gpu_decode_bit_exact(label, img):
    import torch
    from paper_2502_11602_b200 import cheesemap as cm
    rc, _, oh, oxyz = orc.las_read(img)
    assert rc == 0
    xyz, h = cm.decode_las(img)
    assert np.array_equal(xyz.view(np.uint64), oxyz.view(np.uint64))
    assert h["point_count"] == oh.point_count
    # device image at an odd address, device output
    dev = torch.zeros(len(img) + 3, dtype=torch.uint8, device="cuda")
    dev[3:] = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
    xyz2, _ = cm.decode_las(dev[3:], device_out=True)
    assert np.array_equal(xyz2.cpu().numpy().view(np.uint64), oxyz.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 31, 255, 256, 257, 100_003])
@pytest.mark.parametrize("rl", [12, 20, 34, 57, 1000, 2000])
def test_gpu_decode_tiles_and_record_lengths(n, rl):
    """Tile edges (T records per tile), record lengths that stage in shared
    memory and the direct path (> 1536 bytes)."""
    from paper_2502_11602_b200 import cheesemap as cm
    if rl * n > 60_000_000:
        n = 60_000_000 // rl
    img = make_las(rand_raw(n, n + rl), (0.001, 0.0025, 1e-4), (5e5, -2e5, 3.0), rl=rl,
                   seed=rl)
    rc, _, _, oxyz = orc.las_read(img)
    assert rc == 0
    xyz, _ = cm.decode_las(img)
    assert np.array_equal(xyz.view(np.uint64), oxyz.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("label,img", bad_images())
def test_gpu_errors_match_reference(tmp_path, label, img):
    from paper_2502_11602_b200 import cheesemap as cm
    path = write(tmp_path, label + ".las", img)
    rc, omsg, _, _ = orc.las_read(path=path)
    assert rc == 7
    with pytest.raises(cm.ParseError) as e:
        cm.read_las(path)
    assert str(e.value).endswith(omsg), (label, str(e.value), omsg)
    with pytest.raises(cm.IoError):
        cm.read_las(str(tmp_path / "missing.las"))


@pytest.mark.gpu
@needs_ref
def test_gpu_read_las_then_build_and_query(tmp_path):
    """End to end: the reference writes a LAS file, the device reads it
    (bit-exact with the reference's read_las), builds and answers queries
    identically to the oracle built from the reference-decoded cloud."""
    import torch
    from paper_2502_11602_b200 import cheesemap as cm, synth
    cloud = synth.config_cloud(0, scale=0.2)
    path = str(tmp_path / "cfg0.las")
    orc.las_write_reference(cloud, path, 0.001)
    rc, _, rh, rxyz = orc.las_read(path=path, which="reference")
    assert rc == 0
    dxyz, h = cm.read_las(path, device_out=True)
    assert isinstance(dxyz, torch.Tensor) and dxyz.is_cuda
    assert np.array_equal(dxyz.cpu().numpy().view(np.uint64), rxyz.view(np.uint64))
    assert h["point_count"] == rh.point_count and h["bounds_max"] == list(rh.bounds_max)
    m = cm.Cheesemap.build(dxyz, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    q = rxyz[::7]
    row, cols = cm.radius_search_batch(m, q, 1.0)
    orow, ocols = orc.CpuIndex(rxyz, flavor=1).radius_csr(q, 0, 1.0)
    assert np.array_equal(row, orow) and np.array_equal(cols, ocols)
