"""The shipped C++ example runs on the device: examples/bfs_listing2.cpp (Listing 2 through the
C++ operator API of include/irgl/irgl.hpp over the C-ABI) checks the SPEC.md:438 path answer
itself and exits non-zero on a mismatch."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bfs_listing2_example_runs(irgl, tmp_path):
    src = os.path.join(ROOT, "examples", "bfs_listing2.cpp")
    exe = tmp_path / "bfs_listing2"
    libdir = os.path.dirname(irgl.LIB_PATH)
    subprocess.check_call(["/usr/bin/g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                           src, "-o", str(exe), "-L", libdir, "-lirgl_rt", f"-Wl,-rpath,{libdir}"])
    r = subprocess.run([str(exe), "14"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "level = [0, 1, 2, 3, 4]  invocations = 5" in r.stdout
    assert "RMAT-14 BFS: rounds=" in r.stdout
