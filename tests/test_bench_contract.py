"""bench.py's JSON line keeps the driver contract: the reference arm on CPU
(the reference library compiled from its sources), our arm on the GPU, both
on a shrunken config-1 cloud."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def run_bench(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libcheesemap_ref.so")):
        pytest.skip("reference not compiled here (oracle/_ref)")
    d = run_bench("--impl", "reference", "--scale", "0.005", "--steps", "1", "--warmup", "1",
                  "--cpu-sample", "500")
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "queries/s"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_gpu_arm_line():
    d = run_bench("--scale", "0.01", "--steps", "3", "--warmup", "3", "--cpu-sample", "500")
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["dtype"] == "f64" and "workload" in d["config"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("reference", "port")
    assert d["gpu_launches"] > 0
    g = d["general_centres"]
    assert g["value"] > 0 and g["unit"] == "queries/s"
    assert "cm_radius_search_self" in d["config"]["call"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert set(d["build_ms"]) == {"dense", "sparse", "mixed"}
    assert all(v["frac"] > 0 for v in d["build_roofline"].values())


@pytest.mark.gpu
def test_gpu_slab_layout_line():
    """bench.py --layout slabs (config 4's x-slab layout through cm_build_slab)."""
    d = run_bench("--config", "4", "--layout", "slabs", "--flavor", "sparse", "--scale", "0.005",
                  "--steps", "2", "--warmup", "1")
    assert BASE_KEYS <= d.keys()
    assert d["value"] > 0 and d["build_ms"] > 0 and d["config"]["layout"] == "slabs"
    assert d["config"]["neighbours"] > 0 and d["gpu_launches"] > 0
