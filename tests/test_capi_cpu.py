"""CPU: the drop-in boundary.  libp2s_b200.so loads without a GPU, exports
every symbol include/p2s_b200.h declares, and refuses to run without a B200
(no CPU fallback).  No compute calls are made here."""
import ctypes as C
import os
import re

import pytest

from paper_1703_09619_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    h = open(os.path.join(ROOT, "include", "p2s_b200.h")).read()
    h = re.sub(r"/\*.*?\*/", "", h, flags=re.S)
    return sorted(set(re.findall(r"\b(p2s_[a-z_0-9]+)\s*\(", h)))


def test_library_exports_every_declared_symbol():
    names = _declared()
    assert len(names) >= 14
    lib = C.CDLL(capi.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(capi.EXPORTS)


def test_library_is_sm100a():
    # the cubin inside the .so targets sm_100a only
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_version_and_shape_registry():
    assert b"sm_100a" in capi.lib().p2s_version()
    assert capi.shape_supported(3, (6, 6, 6), [capi.PP, capi.DD], (14, 14, 14))
    assert capi.shape_supported(1, (8, 8, 8), [capi.PP, capi.DD], (20, 20, 20))
    assert not capi.shape_supported(1, (7, 3, 3), [capi.DP], (5, 5, 5))
    assert not capi.shape_supported(4, (3, 3, 3), [capi.PP], (5, 5, 5))   # n_comp > 3


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    with pytest.raises(capi.P2SError) as ei:
        capi.Context(1, (4, 4, 4), [capi.PP], (8, 8, 8))
    assert ei.value.status == capi.CUDA_ERROR
    assert "no CPU fallback" in str(ei.value)


def test_invalid_problem_rejected_before_device():
    with pytest.raises(capi.InvalidArgument):
        capi.Context(1, (0, 4, 4), [capi.PP], (8, 8, 8))
    with pytest.raises(capi.InvalidArgument):
        capi.Context(1, (4, 4, 4), [], (8, 8, 8))


def test_cxx_wrapper_header_compiles():
    import shutil
    import subprocess
    import tempfile
    if not shutil.which("g++"):
        pytest.skip("no g++")
    src = os.path.join(ROOT, "tests", "cpp", "test_wrapper.cpp")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "t")
        r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), src,
                            "-o", exe, os.path.join(ROOT, "paper_1703_09619_b200", "libp2s_b200.so"),
                            f"-Wl,-rpath,{os.path.join(ROOT, 'paper_1703_09619_b200')}"],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
