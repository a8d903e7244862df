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
    assert capi.shape_supported(1, (7, 3, 3), [capi.DP], (5, 5, 5))        # generated module
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
                            f"-Wl,-rpath,{os.path.join(ROOT, 'paper_1703_09619_b200')}",
                            "-I/usr/local/cuda/include", "-L/usr/local/cuda/lib64", "-lcudart"],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_every_grid_shape_is_supported():
    """p2s_shape_supported over the drop-in grid: isotropic N = 1..18 with every
    single kind and both bases, every two-kind mix at three orders, and the
    seeded coverage grid (no device needed: plans only, compiler present)."""
    from paper_1703_09619_b200 import shape_grid
    PP, DD, DP, PD = capi.PP, capi.DD, capi.DP, capi.PD
    cases = []
    for n in range(1, 19):
        for k in (PP, DD, DP, PD):
            for basis in (0, 1) if n >= 2 else (0,):
                cases.append((1, (n, n, n), [k], (n + 7,) * 3, basis))
    for n in (3, 11, 18):
        for k1 in (PP, DD, DP, PD):
            for k2 in (PP, DD, DP, PD):
                cases.append((3, (n, max(1, n - 2), 2), [(k1, k2, k1), (k2, k1, PP)], (n + 3, n, 4), 0))
    cases += [(1, (18, 18, 18), [PP, DD, DP, PD], (64, 64, 64), 1), (1, (1, 1, 1), [DD], (1, 1, 1), 0)]
    cases += shape_grid.ALL
    missing = [c for c in cases if not capi.shape_supported_basis(*c)]
    assert not missing, missing[:5]


def test_planner_rules_of_the_generated_families():
    """The planner's choices for grid shapes whose measured behaviour set the rules
    (profiles/r2z_sweep_fused.jsonl): small units run as many
    small CTAs per SM, a two-CTA tile must not starve stage C, the large family's
    moment kernel takes every k1 of a small rule in one chunk."""
    from paper_1703_09619_b200 import shape_grid
    by_id = {shape_grid.shape_id(c): c for c in shape_grid.ALL}  # (modules cached by build())
    small = capi.shape_prepare(*by_id["1c-1x1x12-DPDRLRDPRLDL-q3x6x16"])
    assert "fused fill" in small and "64 threads, 8 CTA/SM" in small, small
    mid = capi.shape_prepare(*by_id["1c-5x5x5-PD-q12x12x12"])
    assert "192 threads, 3 CTA/SM" in mid, mid
    wide = capi.shape_prepare(*by_id["1c-12x9x3-RLP-q15x10x4"])
    assert "n1 tile 9" in wide and "1 CTA/SM" in wide, wide
    c12 = capi.shape_prepare(*by_id["1c-12x12x12-PD-q18x18x18"])
    assert c12.startswith("large-order") and "k1 chunks of 12" in c12, c12
    n18 = capi.shape_prepare(*by_id["1c-18x18x18-PD-q25x25x25"])
    assert "staged in shared memory" in n18, n18


def test_cxx_host_logic_without_gpu():
    """Partition, first-exception rethrow, sizes and nq default of the C++ API
    (tests/cpp/test_wrapper_cpu.cpp), run here without a GPU."""
    import shutil
    import subprocess
    import tempfile
    if not shutil.which("g++"):
        pytest.skip("no g++")
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present: the rethrow check expects no device")
    except Exception:
        pass
    libdir = os.path.join(ROOT, "paper_1703_09619_b200")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "t")
        r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                            os.path.join(ROOT, "tests", "cpp", "test_wrapper_cpu.cpp"), "-o", exe,
                            os.path.join(libdir, "libp2s_b200.so"), f"-Wl,-rpath,{libdir}", "-lpthread",
                            "-L/usr/local/cuda/lib64", "-lcudart"],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "cxx host logic ok" in r.stdout
