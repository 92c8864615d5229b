"""The C ABI used from plain C (examples/c_api_demo.c): no Python or PyTorch between the
caller and libturbons.so.  CPU: the example compiles and links against the header and the
library; GPU: it runs and its orthogonality check passes."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2512_04632_b200")


def _build(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not found")
    if not os.path.exists(os.path.join(LIBDIR, "libturbons.so")):
        pytest.skip("libturbons.so not built")
    exe = str(tmp_path / "c_api_demo")
    cmd = [nvcc, "-O2", "-Wno-deprecated-gpu-targets", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "c_api_demo.c"), "-L", LIBDIR, "-lturbons",
           f"-Xlinker=-rpath={LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_compiles(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "flags 0" in r.stdout and "launches" in r.stdout
