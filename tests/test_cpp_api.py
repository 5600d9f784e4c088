"""Builds tests/cpp/test_actmap_api.cpp against include/ and the in-tree
libactmap_b200.so, then runs it (GPU).  The compile step alone runs on CPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2004_00540_b200")


def build(tmp_path):
    exe = os.path.join(str(tmp_path), "test_actmap_api")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_actmap_api.cpp"), "-L", LIBDIR, "-lactmap_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_api_compiles_against_headers(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libactmap_b200.so")):
        pytest.skip("library not built")
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_on_device(tmp_path):
    exe = build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout[-4000:])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
