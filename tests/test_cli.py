"""the reference CLI's bench / report / generate
over the device structures (tools/cmd_bench.cpp, cmd_report.cpp,
common.cpp), the synthetic specs (io.cpp:252-399) and memory accounting
(map.cpp:173-192), pinned against the reference where it can run here."""
import csv
import io
import os

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2502_11602_b200 import cheesemap as cm
from paper_2502_11602_b200 import cli, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAS_REF = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libcheesemap_ref.so"))
needs_ref = pytest.mark.skipif(not HAS_REF, reason="oracle/_ref not built")

SPECS = ["uniform:n=5000,extent=100x100x50,seed=42",
         "void-ellipse:n=20000,extent=100x100x50,seed=1,cx=50,cy=50,ax=20,ay=15",
         "clusters:n=50000,extent=100x100x50,seed=7,clusters=8,sigma=2.5",
         "clusters:n=999,extent=10x10x10,seed=3,clusters=1,sigma=0.5"]
BAD_SPECS = ["uniform", "bogus:n=1", "uniform:n", "uniform:n=abc", "uniform:extent=1x2",
             "uniform:extent=1y2y3", "uniform:foo=1", "uniform:n=0,extent=1x1x1",
             "uniform:n=10,extent=0x1x1", "void-ellipse:n=10,extent=100x100x50,ax=0,ay=1",
             "void-ellipse:n=10,extent=100x100x50,cx=5,cy=50,ax=20,ay=15",
             "clusters:n=10,extent=10x10x10,clusters=0", "clusters:n=10,extent=10x10x10,sigma=0"]


# ------------------------------------------------------------------ CPU --
@needs_ref
@pytest.mark.parametrize("spec", SPECS)
def test_generate_equals_reference(spec):
    rc, _, ref = orc.generate_reference(spec)
    assert rc == 0
    ours = synth.generate(spec)
    assert np.array_equal(ours.view(np.uint64), ref.view(np.uint64))


@needs_ref
@pytest.mark.parametrize("spec", BAD_SPECS)
def test_spec_errors_equal_reference(spec):
    rc, msg, _ = orc.generate_reference(spec)
    assert rc in (2, 7)
    err = cm.ParseError if rc == 7 else cm.InvalidArgumentError
    with pytest.raises(err) as e:
        synth.generate(spec)
    assert str(e.value) == msg


def test_structure_ids():
    assert cli.Structure("gpu-mixed3").name() == "gpu-mixed3"
    assert cli.Structure("dense2").name() == "gpu-dense2"
    assert cli.Structure("sparse3-reordered").name() == "gpu-sparse3-reordered"
    assert cli.Structure("mixed2", force_reorder=True).name() == "gpu-mixed2-reordered"
    for bad in ("kdtree", "gpu-mixed4", "mixed", "-reordered", "gpu-"):
        with pytest.raises(cm.InvalidArgumentError):
            cli.Structure(bad)
    assert cm.structure_name(cm.Flavor.Sparse, cm.GridMode.TwoD, True) == "sparse2-reordered"


def test_geomean_summary(tmp_path):
    rows = [cli.CSV_HEADER,
            "ds,kdtree,kdtree,3,0,0,sphere,1,100,1000,900,1500,0,10,ok",
            "ds,gpu-mixed3,mixed,3,1,0,sphere,1,100,10,9,15,27,10,ok",
            "ds,mixed3,mixed,3,1,0,sphere,1,100,500,450,700,27,10,ok",
            "ds,kdtree,kdtree,3,0,0,sphere,2,100,4000,3900,4500,0,80,ok",
            "ds,gpu-mixed3,mixed,3,1,0,sphere,2,100,40,39,45,64,80,ok",
            "ds,gpu-mixed3,mixed,3,2.5,0,sphere,2,100,10,9,15,8,80,ok",
            "ds,gpu-dense3,dense,3,1,0,sphere,2,0,0,0,0,0,0,skipped"]
    p = tmp_path / "b.csv"
    p.write_text("\n".join(rows) + "\n")
    out = io.StringIO()
    assert cli.geomean_summary(str(p), "kdtree", out) == 0
    lines = out.getvalue().splitlines()
    assert lines[0] == "structure,query_type,parameter,geomean_normalized_time"
    got = {tuple(l.split(",")[:3]): float(l.split(",")[3]) for l in lines[1:]}
    assert got[("gpu-mixed3", "sphere", "1.000000")] == pytest.approx(0.01)
    assert got[("gpu-mixed3", "sphere", "2.000000")] == pytest.approx(np.sqrt(0.01 * 0.0025))
    assert got[("mixed3", "sphere", "1.000000")] == pytest.approx(0.5)
    p.write_text("bad,header\n")
    with pytest.raises(cm.ParseError):
        cli.geomean_summary(str(p), "kdtree", io.StringIO())
    assert cli.main(["bench", "--geomean", str(tmp_path / "nope.csv")]) == cli.EXIT_IO


@needs_ref
def test_generate_command_writes_the_reference_files(tmp_path):
    """cmd_generate (cmd_report.cpp:80-100): our .las is byte-identical to
    the reference's write_las of the same cloud; .xyz round-trips."""
    spec = SPECS[1]
    las = str(tmp_path / "g.las")
    assert cli.main(["generate", "--synthetic", spec, "--output", las]) == 0
    ref = str(tmp_path / "ref.las")
    orc.las_write_reference(synth.generate(spec), ref, 0.001)
    assert open(las, "rb").read() == open(ref, "rb").read()
    xyz = str(tmp_path / "g.xyz")
    assert cli.main(["generate", "--synthetic", spec, "--output", xyz]) == 0
    back = cli.read_xyz(xyz)
    assert np.array_equal(back, synth.generate(spec))
    assert cli.main(["generate", "--synthetic", "uniform:n=0", "--output", xyz]) == cli.EXIT_USAGE
    assert cli.main(["generate", "--synthetic", "bogus", "--output", xyz]) == cli.EXIT_IO


def test_read_xyz_errors(tmp_path):
    p = tmp_path / "a.xyz"
    p.write_text("# comment\n\n1 2 3\n4 5\n")
    with pytest.raises(cm.ParseError, match="malformed point at line 4"):
        cli.read_xyz(str(p))
    p.write_text("1 2 nan\n")
    with pytest.raises(cm.ParseError, match="non-finite coordinate at line 1"):
        cli.read_xyz(str(p))
    with pytest.raises(cm.IoError):
        cli.read_xyz(str(tmp_path / "missing.xyz"))


@needs_ref
def test_memory_model_restatement_equals_reference():
    cloud = synth.generate(SPECS[1])
    for flavor in (0, 1, 2):
        for mode in (0, 1):
            a = orc.CpuIndex(cloud, flavor=flavor, mode=mode).memory_report()
            b = orc.CpuIndex(cloud, flavor=flavor, mode=mode, which="reference").memory_report()
            assert a == b


# ------------------------------------------------------------------ GPU --
@pytest.mark.gpu
def test_memory_report_matches_oracle_and_acceptance_c6():
    """acceptance.cpp:270-304 (criterion 6) on the device structures."""
    cloud = synth.generate(SPECS[1])
    reps = {}
    for flavor in (cm.Flavor.Dense, cm.Flavor.Sparse, cm.Flavor.Mixed):
        m = cm.Cheesemap.build(cloud, cm.BuildOptions(flavor=flavor))
        r = m.memory_report()
        o = orc.CpuIndex(cloud, flavor=int(flavor)).memory_report()
        assert {k: r[k] for k in o} == o
        assert r["device_bytes"] >= 32 * cloud.shape[0]
        reps[flavor] = r
    d, s, x = reps[cm.Flavor.Dense], reps[cm.Flavor.Sparse], reps[cm.Flavor.Mixed]
    assert s["structure_bytes"] < d["structure_bytes"]
    assert x["structure_bytes"] <= max(d["structure_bytes"], s["structure_bytes"])
    for r in reps.values():
        assert r["handle_bytes"] == 8 * cloud.shape[0]
        assert r["total_bytes"] == r["handle_bytes"] + r["structure_bytes"]


@pytest.mark.gpu
def test_bench_csv_rows(tmp_path):
    spec = "uniform:n=200000,extent=100x100x50,seed=1"
    out = str(tmp_path / "b.csv")
    rc = cli.main(["bench", "--synthetic", spec, "--structures", "gpu-mixed3,sparse2",
                   "--cell-sizes", "1,2.5", "--query", "sphere", "--radii", "1,2.5",
                   "--seconds", "0.05", "--counter-sample", "200", "--batch", "20000",
                   "--output", out])
    assert rc == 0
    lines = open(out).read().splitlines()
    assert lines[0] == cli.CSV_HEADER
    rows = list(csv.reader(lines[1:]))
    assert len(rows) == 2 * 2 * 2 and all(len(r) == 15 and r[14] == "ok" for r in rows)
    # counters: the reference's definitions on the same CenterStream sample
    cloud = synth.generate(spec)
    tag = 0
    for st in ("gpu-mixed3", "gpu-sparse2"):
        mode = 1 if st.endswith("3") else 0
        for cell in (1.0, 2.5):
            o = orc.CpuIndex(cloud, flavor=1, mode=mode, cell=(cell,) * 3)
            for r in (1.0, 2.5):
                tag += 1
                row = rows[tag - 1]
                assert row[1] == st and float(row[4]) == cell and float(row[7]) == r
                idx = synth.center_stream(1, tag, cloud.shape[0], 200).astype(np.int64)
                cnt, _, _, vv = o.radius(cloud[idx], 0, r, stats=True)
                assert float(row[13]) == pytest.approx(cnt.astype(np.float64).mean(), rel=1e-5)
                assert float(row[12]) == pytest.approx(vv.astype(np.float64).mean(), rel=1e-5)
                assert int(row[8]) >= 20000 and float(row[9]) > 0


@pytest.mark.gpu
def test_bench_knn_json_and_capacity(tmp_path):
    import json
    out = str(tmp_path / "k.json")
    rc = cli.main(["bench", "--synthetic", "uniform:n=100000,extent=100x100x50,seed=2",
                   "--structures", "gpu-mixed3", "--cell-sizes", "1", "--query", "knn",
                   "--k", "5,20", "--seconds", "0.05", "--batch", "10000", "--format", "json",
                   "--output", out])
    assert rc == 0
    doc = json.load(open(out))
    assert [d["parameter"] for d in doc] == [5.0, 20.0]
    assert [d["mean_result_size"] for d in doc] == [5.0, 20.0]
    # a dense build over the cap is a skipped row, not a failure (cmd_bench.cpp:338-352)
    out = str(tmp_path / "s.csv")
    rc = cli.main(["bench", "--synthetic", "uniform:n=1000,extent=100000x100000x100,seed=2",
                   "--structures", "gpu-dense3", "--cell-sizes", "0.01", "--radii", "1",
                   "--seconds", "0.01", "--output", out])
    assert rc == 0
    assert open(out).read().splitlines()[1].endswith(",skipped")


@pytest.mark.gpu
def test_report_json(tmp_path):
    import json
    out = str(tmp_path / "r.json")
    spec = SPECS[2]
    rc = cli.main(["report", "--synthetic", spec, "--structures", "gpu-dense3,gpu-mixed3",
                   "--cell-sizes", "1,2.5", "--output", out])
    assert rc == 0
    doc = json.load(open(out))
    cloud = synth.generate(spec)
    wd, bins = orc.weighted_density(cloud)
    assert doc["points"] == cloud.shape[0] and doc["weighted_density"] == wd
    assert doc["histogram"] == [int(b) for b in bins]
    assert [(e["structure"], e["cell_size"]) for e in doc["structures"]] == [
        ("gpu-dense3", 1.0), ("gpu-dense3", 2.5), ("gpu-mixed3", 1.0), ("gpu-mixed3", 2.5)]
    for e in doc["structures"]:
        o = orc.CpuIndex(cloud, flavor=0 if "dense" in e["structure"] else 2,
                         cell=(e["cell_size"],) * 3)
        assert e["non_empty"] == o.non_empty()
        mem = o.memory_report()
        assert (e["handle_bytes"], e["structure_bytes"], e["total_bytes"]) == (
            mem["handle_bytes"], mem["structure_bytes"], mem["total_bytes"])
        assert ("slices" in e) == ("mixed" in e["structure"])


@pytest.mark.gpu
def test_brute_force_baselines_match_oracle():
    """brute_radius / brute_knn on the device against the restatement's
    kernel_search / kNN (which the reference pins)."""
    rng = np.random.default_rng(11)
    cloud = rng.uniform(0, 20, (30000, 3))
    q = np.ascontiguousarray(cloud[::97])
    o = orc.CpuIndex(cloud, flavor=1)
    for kind in (cm.SPHERE, cm.CUBE, cm.CYLINDER):
        for r in (0.5, 2.0):
            c, d = cm.brute_radius(cloud, q, r, kind)
            oc, od = o.radius(q, int(kind), r)
            assert np.array_equal(c, oc) and np.array_equal(d, od)
    for k in (1, 7, 64):
        idx, d2 = cm.brute_knn(cloud, q, k)
        oi, od2 = o.knn(q, k)
        assert np.array_equal(idx, oi) and np.array_equal(d2, od2)
    with pytest.raises(cm.InvalidArgumentError):
        cm.brute_knn(cloud, q, 65)


@pytest.mark.gpu
def test_verify_command(capsys):
    """cmd_verify: all cases match; the fault hook must be detected."""
    spec = "uniform:n=20000,extent=50x50x25,seed=10"
    assert cli.main(["verify", "--synthetic", spec, "--queries", "10"]) == 0
    out = capsys.readouterr().out
    assert "verify: synthetic: 1920/1920 cases matched the oracle" in out
    # test_cli.cpp:152-154: a small cloud, so the corrupted voxel is in reach
    assert cli.main(["verify", "--synthetic", "uniform:n=2000,extent=20x20x10,seed=3",
                     "--cell-sizes", "1", "--queries", "10", "--inject-fault"]) == cli.EXIT_MISMATCH
    assert cli.main(["verify", "--synthetic", spec, "--cap", "100"]) == cli.EXIT_CAPACITY
