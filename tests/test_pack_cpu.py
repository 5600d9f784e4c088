"""Host occupancy packing (csrc/pack.cpp) on CPU: builds tests/cpp/test_pack.cpp against the
in-tree libactmap_b200.so and runs it once per vector ISA the host supports (AM_PACK_ISA)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2004_00540_b200")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    if not os.path.exists(os.path.join(LIBDIR, "libactmap_b200.so")):
        pytest.skip("library not built")
    path = os.path.join(str(tmp_path_factory.mktemp("pack")), "test_pack")
    subprocess.run(["g++", "-std=c++17", "-O1", os.path.join(ROOT, "tests", "cpp", "test_pack.cpp"), "-L", LIBDIR,
                    "-lactmap_b200", f"-Wl,-rpath,{LIBDIR}", "-o", path], check=True)
    return path


@pytest.mark.parametrize("isa", ["sse2", "avx2", "avx512", "auto"])
def test_pack_rows_matches_scalar(exe, isa):
    env = dict(os.environ)
    env.pop("AM_PACK_ISA", None)
    if isa != "auto":
        env["AM_PACK_ISA"] = isa  # an ISA the host lacks falls back to the best one it has
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches 0" in out.stdout
