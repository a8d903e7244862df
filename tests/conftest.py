import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_addoption(parser):
    parser.addoption("--jit-prepare", action="store_true",
                     help="build the generated kernel module of every shape the GPU tests create "
                          "(p2s_shape_prepare, no GPU needed) and skip the tests")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    if config.getoption("--jit-prepare"):
        return
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


_PREPARE = []


@pytest.fixture(autouse=True)
def _jit_prepare(request, monkeypatch):
    """--jit-prepare: every capi.Context a test creates is recorded instead of
    created; at the end of the session the generated modules of all recorded
    shapes are built in parallel (so the module cache ships with the repo)."""
    if not request.config.getoption("--jit-prepare"):
        yield
        return
    from paper_1703_09619_b200 import capi

    def init(self, n_comp, order, kinds, nq, device=0, basis=0, options=None):
        opts = dict(capi.DEFAULT_OPTIONS)
        opts.update(options or {})
        if opts.get("P2S_JIT") != "0" and opts.get("P2S_FORCE_GENERIC") != "1":
            jopts = {k: v for k, v in opts.items() if k.startswith("P2S_JIT_") or k == "P2S_FORCE_JIT"}
            _PREPARE.append((n_comp, tuple(order), [tuple(k) if isinstance(k, (list, tuple)) else k
                                                     for k in kinds], tuple(nq), basis, jopts))
        pytest.skip("jit-prepare")

    monkeypatch.setattr(capi.Context, "__init__", init)
    yield


def pytest_sessionfinish(session, exitstatus):
    if not session.config.getoption("--jit-prepare") or not _PREPARE:
        return
    from paper_1703_09619_b200 import shape_grid
    uniq = {shape_grid.shape_id(c[:5]) + str(sorted(c[5].items())): c for c in _PREPARE}
    res = shape_grid.prepare_all(list(uniq.values()))
    bad = {k: v for k, v in res.items() if v.startswith("ERROR")}
    print(f"\njit-prepare: {len(res)} shapes, {len(bad)} errors")
    for k, v in bad.items():
        print(" ", k, v[:300])
