"""Every device path under the CHECKED library (libcmgpu_checked.so: device
invariant checks — span, arena, row, flush and pack bounds, count-vs-fill row
lengths — compiled in; a failed check traps). This stands in for
compute-sanitizer, which is closed on this pool's GPUs."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_checked_library_probe():
    lib = os.path.join(ROOT, "paper_2502_11602_b200", "libcmgpu_checked.so")
    assert os.path.exists(lib), "build it: make -C paper_2502_11602_b200/csrc checked"
    env = dict(os.environ, CMGPU_LIB="libcmgpu_checked.so")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "checked_probe.py")],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert "checked probe ok" in out.stdout and "libcmgpu_checked.so" in out.stdout
