"""GPU: the reference-shaped C++ API (include/p2s_b200.hpp) end to end."""
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def test_cxx_wrapper_known_answers():
    libdir = os.path.join(ROOT, "paper_1703_09619_b200")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "t")
        cuda_inc = "/usr/local/cuda/include"
        r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I", cuda_inc,
                            os.path.join(ROOT, "tests", "cpp", "test_wrapper.cpp"), "-o", exe,
                            os.path.join(libdir, "libp2s_b200.so"), f"-Wl,-rpath,{libdir}", "-lpthread",
                            "-L/usr/local/cuda/lib64", "-lcudart"],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "cxx wrapper ok" in r.stdout
