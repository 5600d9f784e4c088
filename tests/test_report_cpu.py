"""RunReport JSON (report.hpp) on CPU: builds tests/cpp/test_report.cpp against include/ and the in-tree
library and runs it (serialisation is host code: no device needed)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2004_00540_b200")


def test_run_report_round_trip(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libactmap_b200.so")):
        pytest.skip("library not built")
    exe = os.path.join(str(tmp_path), "test_report")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_report.cpp"), "-L", LIBDIR, "-lactmap_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
