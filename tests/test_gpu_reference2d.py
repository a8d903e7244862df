"""GPU pinned DIRECTLY to the reference: the 2-D Chebyshev mode of the sm_100a
path (p2s_cheb2d_*) against the numbers the compiled reference produced
(tests/golden/ref2d_elements.npz: compute_kernel_tables + assemble_p2s_element
of /root/reference/proj on its known-answer element and seeded curved
elements, generator tests/golden/make_ref2d_golden.py)."""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1703_09619_b200 import capi

pytestmark = pytest.mark.gpu

E = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref2d_elements.npz"))
TAGS = [str(t) for t in E["tags"]]


def _run(tag, conforming=False):
    g = lambda k: E[f"{tag}__{k}"]
    M, N, nq = int(g("M")), int(g("N")), int(g("nq"))
    ctx = capi.Cheb2dContext(M, N, nq, conforming=conforming)
    grids = np.stack([g("ws"), g("wuu"), g("wuv"), g("wvv")]).reshape(1, -1)
    dg = torch.from_numpy(np.ascontiguousarray(grids)).cuda()
    dt = torch.full((1, ctx.sizes.tables_per_elem), float("nan"), dtype=torch.float64, device="cuda")
    db = torch.full((1, ctx.sizes.blocks_per_elem), float("nan"), dtype=torch.float64, device="cuda")
    ctx.kernel_tables(dg, dt, 1)
    ctx.assemble(dt, db, 1)
    torch.cuda.synchronize()
    return g, ctx.split_tables(dt[0].cpu().numpy()), ctx.split_blocks(db[0].cpu().numpy())


@pytest.mark.parametrize("tag", TAGS)
def test_gpu_reproduces_reference_element(tag):
    g, tables, blocks = _run(tag)
    for k, v in tables.items():
        ok, ij = O.block_close(v, g(k), 1e-12)
        assert ok, (tag, k, ij)
    for k, v in blocks.items():
        ok, ij = O.block_close(v, g("p2s_" + k), 1e-12)
        assert ok, (tag, k, ij)
        # and the reference's direct quadrature (assemble_direct_element)
        ok, ij = O.block_close(v, g("direct_" + k), 1e-10)
        assert ok, (tag, "direct", k, ij)


@pytest.mark.parametrize("tag", TAGS)
def test_gpu_conforming_reproduces_reference_transform(tag):
    """Conforming mode: the reference's apply_conforming_transform (assembly.cpp:
    555-574) of its p2s blocks, folded into the GPU fill."""
    g, _, blocks = _run(tag, conforming=True)
    for k, v in blocks.items():
        ok, ij = O.block_close(v, g("conf_" + k), 1e-12)
        assert ok, (tag, k, ij)


def test_gpu_reference_known_answers():
    # test_assembly.cpp:96-140
    _, t, b = _run("identity_2x2_nq10")
    assert t["Kuu"][0, 0] == 0.0
    assert abs(t["Kuu"][2, 0] + 4.0) <= 4e-13
    assert abs(t["Ks"][2, 2] - 4.0) <= 4e-13
    assert abs(t["Ks"][4, 2] - 16 / 3) <= 16 / 3 * 1e-13
    assert abs(b["Muu"][0, 0] - 4.0) <= 4e-13
    assert abs(b["Suu"][1 * 3 + 1, 1 * 3 + 1] - 16 / 3) <= 16 / 3 * 1e-13
    assert np.array_equal(b["Svu"], b["Suv"].T) or O.block_close(b["Svu"], b["Suv"].T, 1e-14)[0]


REF_DROPIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "oracle", "_ref", "ref_dropin")


@pytest.mark.skipif(not os.path.exists(REF_DROPIN),
                    reason="oracle/_ref/ref_dropin not built (needs /root/reference at build time)")
def test_reference_calls_gpu_fill_through_the_c_abi():
    """The compiled reference fills seeded curved elements through the GPU and
    checks them with its own element_matrices_close (oracle/refbuild/ref_dropin.cpp)."""
    import subprocess
    r = subprocess.run([REF_DROPIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "elements (modal and conforming) pass" in r.stdout
    assert "global systems (assemble_system on GPU) pass" in r.stdout
