"""Command line for the device engine, mirroring the reference CLI
(proj/tools/main.cpp:9-107) for the paths it serves:

  bench     timed query sweeps -> the reference's 15-column CSV / JSON
            (cmd_bench.cpp:19-36, :88-164, :296-371), structures gpu-dense2 ..
            gpu-mixed3 [-reordered]; --geomean post-processes any CSV of that
            format, so the reference's own rows and these GPU rows can be
            summarised together (cmd_bench.cpp:231-292)
  report    dataset metrics + per-structure occupancy and memory accounting
            (cmd_report.cpp:11-78)
  verify    every flavour / mode / kernel against the device brute force
            (cmd_verify.cpp:31-114; exit 1 on a mismatch)
  generate  write a synthetic cloud (.las / .xyz) (cmd_report.cpp:80-100)

    python -m paper_2502_11602_b200.cli bench --synthetic uniform:n=1000000,extent=100x100x50,seed=1 \\
        --structures gpu-mixed3,gpu-dense3 --cell-sizes 1 --query sphere --radii 0.5,1

Timing differs from the reference by design: the device answers BATCHES of
centres (the reference times one call per centre). A bench row's queries
are --batch centres per call drawn from the reference's CenterStream
(common.cpp:109-125); mean_ns is total device time / queries, median_ns and
p95_ns are over the per-batch amortised times. Exit codes follow
common.hpp:16-20 (0 ok, 1 mismatch, 2 usage, 3 io/parse, 4 capacity).
"""
import argparse
import json
import math
import os
import sys

import numpy as np

from . import cheesemap as cm
from . import synth

EXIT_OK, EXIT_MISMATCH, EXIT_USAGE, EXIT_IO, EXIT_CAPACITY = 0, 1, 2, 3, 4

CSV_HEADER = ("dataset,structure,flavor,dims,cell_size,reordered,query_type,parameter,"
              "queries,mean_ns,median_ns,p95_ns,mean_voxels_visited,mean_result_size,status")
QUERY_TYPES = ("sphere", "cube", "cylinder", "knn")
KERNEL_OF = {"sphere": cm.SPHERE, "cube": cm.CUBE, "cylinder": cm.CYLINDER}


# ------------------------------------------------------------ structures --
class Structure:
    """A device map variant: gpu-{dense,sparse,mixed}{2,3}[-reordered]
    (the reference's map ids, common.cpp:16-44, prefixed gpu-)."""

    def __init__(self, text, force_reorder=False):
        base = text
        self.reordered = False
        if base.endswith("-reordered") and len(base) > len("-reordered"):
            self.reordered = True
            base = base[: -len("-reordered")]
        if base.startswith("gpu-"):
            base = base[4:]
        names = {"dense": cm.Flavor.Dense, "sparse": cm.Flavor.Sparse, "mixed": cm.Flavor.Mixed}
        if len(base) < 2 or base[:-1] not in names or base[-1] not in "23":
            raise cm.InvalidArgumentError(f"unknown structure '{text}'")
        self.flavor = names[base[:-1]]
        self.mode = cm.GridMode.TwoD if base[-1] == "2" else cm.GridMode.ThreeD
        self.reordered = self.reordered or force_reorder

    def name(self):
        return "gpu-" + cm.structure_name(self.flavor, self.mode, self.reordered)

    def flavor_label(self):
        return ["dense", "sparse", "mixed"][int(self.flavor)]

    def dims(self):
        return 2 if self.mode == cm.GridMode.TwoD else 3


# ----------------------------------------------------------------- input --
def read_xyz(path):
    """read_xyz (io.cpp:168-195): "x y z" lines, blank / '#' lines skipped."""
    try:
        f = open(path, "r")
    except OSError:
        raise cm.IoError(f"cannot open {path}")
    pts = []
    with f:
        for line_no, line in enumerate(f, 1):
            s = line.strip(" \t\r\n")
            if not s or s.startswith("#"):
                continue
            parts = s.split()
            try:
                x, y, z = (float(v) for v in parts[:3])
                if len(parts) < 3:
                    raise ValueError
            except ValueError:
                raise cm.ParseError(f"malformed point at line {line_no} of {path}")
            if not all(math.isfinite(v) for v in (x, y, z)):
                raise cm.ParseError(f"non-finite coordinate at line {line_no} of {path}")
            pts.append((x, y, z))
    return np.asarray(pts, dtype=np.float64).reshape(-1, 3)


def write_xyz(cloud, path):
    """write_xyz (io.cpp:197-212): %.17g, bit-exact round trip."""
    try:
        with open(path, "w") as f:
            for x, y, z in cloud:
                f.write("%.17g %.17g %.17g\n" % (x, y, z))
    except OSError:
        raise cm.IoError(f"cannot write {path}")


def _round_half_away(v):
    t = np.trunc(v)
    return t + np.where(np.abs(v - t) >= 0.5, np.sign(v), 0.0)


def write_las(cloud, path, scale=0.001):
    """write_las (io.cpp:108-166): LAS 1.2, format 0, offset = bbox min,
    coordinates quantised with round-half-away (std::round)."""
    if not scale > 0.0:
        raise cm.InvalidArgumentError("LAS scale must be positive")
    cloud = np.asarray(cloud, dtype=np.float64).reshape(-1, 3)
    lo = cloud.min(axis=0) if cloud.shape[0] else np.zeros(3)
    hi = cloud.max(axis=0) if cloud.shape[0] else np.zeros(3)
    q = _round_half_away((cloud - lo) / scale)
    if np.abs(q).max(initial=0.0) > 2147483647.0:
        raise cm.InvalidArgumentError("coordinate does not fit a 32-bit LAS record at this scale")
    import struct
    hdr = bytearray(b"LASF" + bytes(20) + bytes([1, 2]) + bytes(68))
    hdr += struct.pack("<HIIBHI", 227, 227, 0, 0, 20, cloud.shape[0]) + bytes(20)
    hdr += struct.pack("<3d3d", scale, scale, scale, *lo)
    hdr += struct.pack("<6d", hi[0], lo[0], hi[1], lo[1], hi[2], lo[2])
    assert len(hdr) == 227
    recs = np.zeros((cloud.shape[0], 5), dtype=np.int32)
    recs[:, :3] = q.astype(np.int32)
    try:
        with open(path, "wb") as f:
            f.write(bytes(hdr))
            f.write(recs.tobytes())
    except OSError:
        raise cm.IoError(f"cannot write {path}")


def load_cloud(input_path, synthetic):
    """load_cloud (common.cpp:56-86) -> (cloud, dataset name)."""
    if input_path and synthetic:
        raise cm.InvalidArgumentError("--input and --synthetic are exclusive")
    if input_path:
        stem, ext = os.path.splitext(os.path.basename(input_path))
        if ext == ".las":
            return cm.read_las(input_path)[0], stem
        if ext in (".xyz", ".txt"):
            return read_xyz(input_path), stem
        raise cm.InvalidArgumentError(f"unsupported input extension '{ext}' (expected .las or .xyz)")
    if not synthetic:
        raise cm.InvalidArgumentError("one of --input or --synthetic is required")
    return synth.generate(synth.parse_synthetic_spec(synthetic)), "synthetic"


# ------------------------------------------------------------ counters --
def voxels_visited(grid, centers, r, query):
    """QueryStats::voxels_visited (search.hpp:110-117): the clamped range's
    voxel count (grid.cpp:90-114), in the reference's fp64 arithmetic."""
    o = np.asarray(grid["origin"])
    s = np.asarray(grid["cell"])
    dims = np.array([grid["nx"], grid["ny"], grid["nz"]], dtype=np.int64)
    bmin, bmax = np.asarray(grid["bounds_min"]), np.asarray(grid["bounds_max"])
    lo, hi = centers - r, centers + r
    if query == "cylinder":  # unbounded z (geometry.hpp:97-113)
        lo[:, 2], hi[:, 2] = -np.inf, np.inf
    disjoint = np.any((lo > bmax) | (hi < bmin), axis=1)
    lo = np.where(lo < bmin, bmin, lo)
    hi = np.where(bmax < hi, bmax, hi)

    def axis_index(p):
        idx = np.floor((p - o) / s)
        idx = np.where(idx < 0, 0, idx)
        return np.minimum(idx.astype(np.int64), dims - 1)
    a, b = axis_index(lo), axis_index(hi)
    if grid["mode"] == cm.GridMode.TwoD:
        a[:, 2], b[:, 2] = 0, 0
    cnt = np.prod(b - a + 1, axis=1).astype(np.float64)
    return np.where(disjoint, 0.0, cnt)


# ----------------------------------------------------------------- bench --
def _g(v):
    """std::ostream's default formatting of a double (%g, 6 digits)."""
    return "%g" % v


def _row_csv(r):
    return ",".join([r["dataset"], r["structure"], r["flavor"], str(r["dims"]),
                     _g(r["cell_size"]), "1" if r["reordered"] else "0", r["query_type"],
                     _g(r["parameter"]), str(r["queries"]), _g(r["mean_ns"]), _g(r["median_ns"]),
                     _g(r["p95_ns"]), _g(r["mean_voxels_visited"]), _g(r["mean_result_size"]),
                     r["status"]])


def run_combination(args, cloud_dev, cloud, dataset, st, cell, qtype, param, tag, m):
    import torch
    n = cloud.shape[0]
    rec = dict(dataset=dataset, structure=st.name(), flavor=st.flavor_label(), dims=st.dims(),
               cell_size=cell, reordered=st.reordered, query_type=qtype, parameter=param,
               queries=0, mean_ns=0.0, median_ns=0.0, p95_ns=0.0, mean_voxels_visited=0.0,
               mean_result_size=0.0, status="ok")
    # deterministic counters on a fixed centre sample (cmd_bench.cpp:184-196)
    sample = max(1, args.counter_sample)
    idx = synth.center_stream(args.seed, tag, n, sample).astype(np.int64)
    cs = np.ascontiguousarray(cloud[idx])
    if qtype == "knn":
        rec["mean_result_size"] = float(min(int(param), n))
    else:
        cnt = np.zeros(sample, dtype=np.uint32)
        cm.radius_count(m, cs, param, KERNEL_OF[qtype], counts=cnt)
        rec["mean_result_size"] = float(cnt.astype(np.float64).mean())
        rec["mean_voxels_visited"] = float(voxels_visited(m.grid(), cs, param, qtype).mean())

    batch = max(1, args.batch)

    def run(centers_dev):
        if qtype == "knn":
            cm.knn_batch(m, centers_dev, int(param), device_out=True)
        else:
            cm.radius_search_batch(m, centers_dev, param, KERNEL_OF[qtype], device_out=True)

    # warm-up, then batches until the time budget is spent (cmd_bench.cpp:198-213)
    centers = synth.CenterStream(args.seed, tag, n)

    def next_batch():
        ids = centers.next(batch).astype(np.int64)
        return cloud_dev[torch.from_numpy(ids).to(cloud_dev.device)].contiguous()
    if args.warmup > 0:
        run(cloud_dev[torch.from_numpy(centers.next(args.warmup).astype(np.int64))
                      .to(cloud_dev.device)].contiguous())
    per = []
    total_ms = 0.0
    import time
    deadline = time.perf_counter() + max(args.seconds, 1e-3)
    while True:
        c = next_batch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(c)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        total_ms += ms
        per.append(ms * 1e6 / batch)
        if time.perf_counter() >= deadline:
            break
    per.sort()
    rec["queries"] = batch * len(per)
    rec["mean_ns"] = total_ms * 1e6 / rec["queries"]
    rec["median_ns"] = per[len(per) // 2]
    rec["p95_ns"] = per[min(len(per) - 1, len(per) * 95 // 100)]
    return rec


def geomean_summary(path, baseline, out):
    """geomean_summary (cmd_bench.cpp:231-292)."""
    try:
        f = open(path)
    except OSError:
        raise cm.IoError(f"cannot open {path}")
    with f:
        lines = f.read().splitlines()
    if not lines or lines[0] != CSV_HEADER:
        raise cm.ParseError(f"unexpected CSV header in {path}")
    rows = []
    for line in lines[1:]:
        fld = line.split(",")
        if len(fld) != 15:
            raise cm.ParseError(f"malformed CSV row: {line}")
        if fld[14] != "ok":
            continue
        rows.append(dict(structure=fld[1], query_type=fld[6], dataset=fld[0],
                         parameter=float(fld[7]), mean_ns=float(fld[9])))

    def key_of(r):
        return f"{r['dataset']}|{r['query_type']}|{r['parameter']:f}"
    base = {key_of(r): r["mean_ns"] for r in rows if r["structure"] == baseline}
    if not base:
        raise cm.InvalidArgumentError(f"baseline structure '{baseline}' not present in the CSV")
    acc = {}
    for r in rows:
        k = key_of(r)
        if k not in base or r["structure"] == baseline:
            continue
        a = acc.setdefault(f"{r['structure']},{r['query_type']},{r['parameter']:f}", [0.0, 0])
        a[0] += math.log(r["mean_ns"] / base[k])
        a[1] += 1
    out.write("structure,query_type,parameter,geomean_normalized_time\n")
    for k in sorted(acc):
        out.write(f"{k},{_g(math.exp(acc[k][0] / acc[k][1]))}\n")
    return EXIT_OK


def cmd_bench(args):
    if args.geomean:
        return geomean_summary(args.geomean, args.geomean_baseline, sys.stdout)
    import torch
    cloud, dataset = load_cloud(args.input, args.synthetic)
    if cloud.shape[0] == 0:
        raise cm.EmptyCloudError("point cloud is empty")
    if args.query not in QUERY_TYPES:
        raise cm.InvalidArgumentError(f"unknown query type '{args.query}'")
    params = [float(k) for k in args.k] if args.query == "knn" else args.radii
    if not params:
        raise cm.InvalidArgumentError("no query parameters given")
    structures = [Structure(s, args.reorder) for s in args.structures]
    if not structures:
        raise cm.InvalidArgumentError("no structures given")
    cloud_dev = torch.from_numpy(cloud).cuda(args.device)
    records = []
    tag = 0
    for st in structures:
        for cell in args.cell_sizes:
            m, err = None, None
            try:
                m = cm.Cheesemap.build(cloud_dev, cm.BuildOptions(
                    flavor=st.flavor, mode=st.mode, cell=cm.CellSize.uniform(cell),
                    reorder=st.reordered, densify_threshold=args.tau), device=args.device)
            except cm.CapacityError as e:
                err = str(e)
            for p in params:
                tag += 1
                if err is not None:
                    sys.stderr.write(f"skipping {st.name()} s={_g(cell)}: {err}\n")
                    records.append(dict(dataset=dataset, structure=st.name(),
                                        flavor=st.flavor_label(), dims=st.dims(), cell_size=cell,
                                        reordered=st.reordered, query_type=args.query,
                                        parameter=p, queries=0, mean_ns=0.0, median_ns=0.0,
                                        p95_ns=0.0, mean_voxels_visited=0.0,
                                        mean_result_size=0.0, status="skipped"))
                    continue
                records.append(run_combination(args, cloud_dev, cloud, dataset, st, cell,
                                               args.query, p, tag, m))
            del m
    if args.format == "json":
        text = json.dumps(records, indent=2) + "\n"
    elif args.format == "csv":
        text = CSV_HEADER + "\n" + "".join(_row_csv(r) + "\n" for r in records)
    else:
        raise cm.InvalidArgumentError(f"unknown format '{args.format}'")
    _emit(text, args.output)
    return EXIT_OK


def _emit(text, output):
    if not output:
        sys.stdout.write(text)
        return
    try:
        with open(output, "w") as f:
            f.write(text)
    except OSError:
        raise cm.IoError(f"cannot write {output}")


# ---------------------------------------------------------------- report --
def cmd_report(args):
    cloud, dataset = load_cloud(args.input, args.synthetic)
    if cloud.shape[0] == 0:
        raise cm.EmptyCloudError("point cloud is empty")
    doc = {"dataset": dataset, "points": int(cloud.shape[0]),
           "density": cm.global_density(cloud, device=args.device)}
    wd, hist = cm.weighted_density(cloud, args.density_sample or 0, args.seed, device=args.device)
    doc["weighted_density"] = wd
    doc["histogram"] = [int(v) for v in hist]
    doc["structures"] = []
    for text in args.structures:
        st = Structure(text, args.reorder)
        for cell in args.cell_sizes:
            e = {"structure": st.name(), "cell_size": cell}
            try:
                m = cm.Cheesemap.build(cloud, cm.BuildOptions(
                    flavor=st.flavor, mode=st.mode, cell=cm.CellSize.uniform(cell),
                    reorder=st.reordered, densify_threshold=args.tau), device=args.device)
                occ = m.occupancy_stats()
                e["total_voxels"] = int(occ["total_voxels"])
                e["non_empty"] = int(occ["non_empty"])
                e["empty_fraction"] = occ["empty_fraction"]
                if st.flavor == cm.Flavor.Mixed:  # slices reported for mixed (map.cpp:160-165)
                    g = m.grid()
                    e["slices"] = [{"dense": bool(d), "cells": int(g["nx"] * g["ny"]),
                                    "non_empty": int(ne)}
                                   for d, ne in zip(occ["slice_dense"], occ["slice_non_empty"])]
                mem = m.memory_report()
                e.update(handle_bytes=mem["handle_bytes"], structure_bytes=mem["structure_bytes"],
                         total_bytes=mem["total_bytes"], device_bytes=mem["device_bytes"])
            except cm.CapacityError as ex:
                e["skipped"] = str(ex)
            doc["structures"].append(e)
    _emit(json.dumps(doc, indent=2) + "\n", args.output)
    return EXIT_OK


def cmd_verify(args):
    """cmd_verify (cmd_verify.cpp:31-114): every flavour x mode x cell size,
    sphere / cube / cylinder at r in {0.5, 1, 2.5, 5} and kNN at k in
    {1, 5, 10, 20}, for --queries centres, against the device brute force.
    Sets are compared as (count, splitmix64 digest); kNN by (handle, d^2)."""
    cloud, dataset = load_cloud(args.input, args.synthetic)
    if cloud.shape[0] == 0:
        raise cm.EmptyCloudError("point cloud is empty")
    if cloud.shape[0] > args.cap:
        raise cm.CapacityError(f"cloud has {cloud.shape[0]} points, above the verification cap "
                               f"of {args.cap}; subsample the input first")
    radii = (0.5, 1.0, 2.5, 5.0)
    ks = (1, 5, 10, 20)
    kinds = (("sphere", cm.SPHERE), ("cube", cm.CUBE), ("cylinder", cm.CYLINDER))
    centers = np.ascontiguousarray(cloud[synth.center_stream(args.seed, 0, cloud.shape[0],
                                                             args.queries).astype(np.int64)])
    nq = centers.shape[0]
    brute = {}
    for r in radii:
        for kname, kind in kinds:
            brute[(kname, r)] = cm.brute_radius(cloud, centers, r, kind, device=args.device)
    for k in ks:
        brute[("knn", k)] = cm.brute_knn(cloud, centers, k, device=args.device)
    cases = failures = 0
    for flavor in (cm.Flavor.Dense, cm.Flavor.Sparse, cm.Flavor.Mixed):
        for mode in (cm.GridMode.TwoD, cm.GridMode.ThreeD):
            for cell in args.cell_sizes:
                m = cm.Cheesemap.build(cloud, cm.BuildOptions(
                    flavor=flavor, mode=mode, cell=cm.CellSize.uniform(cell),
                    densify_threshold=args.tau), device=args.device)
                if args.inject_fault:
                    m.corrupt_for_testing()
                name = cm.structure_name(flavor, mode, False)
                ok = {}
                for r in radii:
                    for kname, kind in kinds:
                        c, d = cm.radius_digest_batch(m, centers, r, kind)
                        bc, bd = brute[(kname, r)]
                        ok[(kname, r)] = (c == bc) & (d == bd)
                for k in ks:
                    idx, d2 = cm.knn_batch(m, centers, k)
                    bi, bd = brute[("knn", k)]
                    ok[("knn", k)] = np.all(idx == bi, axis=1) & np.all(d2 == bd, axis=1)
                for q in range(nq):  # the reference's case order (cmd_verify.cpp:69-106)
                    for r in radii:
                        for kname, _ in kinds:
                            cases += 1
                            if not ok[(kname, r)][q]:
                                failures += 1
                                sys.stderr.write(f"MISMATCH: {name} s={cell:f} {kname} r={r:f}\n")
                    for k in ks:
                        cases += 1
                        if not ok[("knn", k)][q]:
                            failures += 1
                            sys.stderr.write(f"MISMATCH: {name} s={cell:f} knn k={k}\n")
                del m
    print(f"verify: {dataset}: {cases - failures}/{cases} cases matched the oracle")
    return EXIT_OK if failures == 0 else EXIT_MISMATCH


def cmd_generate(args):
    if not args.output:
        raise cm.InvalidArgumentError("--output is required")
    cloud = synth.generate(synth.parse_synthetic_spec(args.synthetic))
    fmt = args.format or ("las" if os.path.splitext(args.output)[1] == ".las" else "xyz")
    if fmt == "las":
        write_las(cloud, args.output)
    elif fmt == "xyz":
        write_xyz(cloud, args.output)
    else:
        raise cm.InvalidArgumentError(f"unknown output format '{fmt}'")
    print(f"wrote {cloud.shape[0]} points to {args.output}")
    return EXIT_OK


# ------------------------------------------------------------------ main --
def _floats(s):
    return [float(v) for v in s.split(",") if v]


def _ints(s):
    return [int(v) for v in s.split(",") if v]


def _strs(s):
    return [v for v in s.split(",") if v]


def parser():
    ap = argparse.ArgumentParser(prog="paper_2502_11602_b200.cli",
                                 description="B200 cheesemap: device index + neighbour queries")
    sub = ap.add_subparsers(dest="cmd", required=True)
    maps = "gpu-dense2,gpu-dense3,gpu-sparse2,gpu-sparse3,gpu-mixed2,gpu-mixed3"
    b = sub.add_parser("bench", help="timed query sweeps -> CSV/JSON")
    b.add_argument("--input", default="")
    b.add_argument("--synthetic", default="")
    b.add_argument("--structures", type=_strs, default=_strs(maps))
    b.add_argument("--cell-sizes", type=_floats, default=[1.0, 2.5, 5.0, 7.5, 10.0])
    b.add_argument("--query", default="sphere")
    b.add_argument("--radii", type=_floats, default=[0.5, 1.0, 2.0, 3.0, 5.0, 7.5, 10.0])
    b.add_argument("--k", type=_ints, default=[5, 10, 20, 30, 40, 50])
    b.add_argument("--seconds", type=float, default=1.0)
    b.add_argument("--warmup", type=int, default=10)
    b.add_argument("--counter-sample", type=int, default=100)
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--reorder", action="store_true")
    b.add_argument("--tau", type=float, default=0.80)
    b.add_argument("--output", default="")
    b.add_argument("--format", default="csv")
    b.add_argument("--geomean", default="")
    b.add_argument("--geomean-baseline", default="kdtree")
    b.add_argument("--batch", type=int, default=1 << 20, help="centres per device call")
    b.add_argument("--device", type=int, default=0)
    r = sub.add_parser("report", help="dataset metrics + occupancy and memory per structure")
    r.add_argument("--input", default="")
    r.add_argument("--synthetic", default="")
    r.add_argument("--structures", type=_strs, default=_strs(maps))
    r.add_argument("--cell-sizes", type=_floats, default=[1.0])
    r.add_argument("--tau", type=float, default=0.80)
    r.add_argument("--reorder", action="store_true")
    r.add_argument("--density-sample", type=int, default=0)
    r.add_argument("--seed", type=int, default=1)
    r.add_argument("--output", default="")
    r.add_argument("--device", type=int, default=0)
    v = sub.add_parser("verify", help="check every flavour/mode/kernel against the brute force")
    v.add_argument("--input", default="")
    v.add_argument("--synthetic", default="")
    v.add_argument("--cell-sizes", type=_floats, default=[1.0, 2.5])
    v.add_argument("--seed", type=int, default=1)
    v.add_argument("--queries", type=int, default=25)
    v.add_argument("--cap", type=int, default=200000)
    v.add_argument("--tau", type=float, default=0.80)
    v.add_argument("--inject-fault", action="store_true", help=argparse.SUPPRESS)
    v.add_argument("--device", type=int, default=0)
    g = sub.add_parser("generate", help="write a synthetic cloud to a file")
    g.add_argument("--synthetic", required=True)
    g.add_argument("--output", required=True)
    g.add_argument("--format", default="")
    return ap


def main(argv=None):
    try:
        args = parser().parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    try:
        return {"bench": cmd_bench, "report": cmd_report, "verify": cmd_verify,
                "generate": cmd_generate}[args.cmd](args)
    except cm.CapacityError as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_CAPACITY
    except (cm.ParseError, cm.IoError) as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_IO
    except cm.Error as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
