"""Drop-in coverage on the GPU: every shape of the coverage grid
(paper_1703_09619_b200/shape_grid.py -- N = 1..18 isotropic, seeded anisotropic
mixed-kind / multi-term / multi-component / conforming shapes, the (12,12,12)
bench shape) through the C-ABI against the CPU oracle at rtol 1e-12 with the
reference comparator (verify.cpp:81-99), per (gi, gj) block; the reference's
fill accepts all of them (assembly.hpp:52-56, 82-83).  Shapes without an
ahead-of-time kernel run their generated module (p2s_jit.cu).  Also checks the
two-stage entry points (p2s_moments + p2s_contract) against the same oracle."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1703_09619_b200 import capi, shape_grid

from helpers import blocks_close, oracle_for

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", shape_grid.ALL, ids=shape_grid.shape_id)
def test_shape_grid_matches_oracle(case):
    nc, order, kinds, nq, basis = case
    assert capi.shape_supported_basis(nc, order, kinds, nq, basis)
    o = oracle_for(nc, order, kinds, nq, basis)
    ctx = capi.Context(nc, order, kinds, nq, basis=basis)
    n = 2
    alpha = o.alpha(O.ALPHA_SINE, 0.5, 3.0, 1703 + sum(order), 0, n)
    st = torch.cuda.current_stream().cuda_stream
    a = torch.from_numpy(alpha).cuda()
    M = torch.full((n, ctx.n_tot, ctx.n_tot), float("nan"), dtype=torch.float64, device="cuda")
    ctx.fill(a, M, ctx.n_tot, n, st)
    I = torch.zeros((n, ctx.moments_per_elem), dtype=torch.float64, device="cuda")
    ctx.moments(a, I, n, st)
    M2 = torch.full_like(M, float("nan"))
    ctx.contract(I, M2, ctx.n_tot, n, st)
    torch.cuda.synchronize()
    Mo = o.fill(alpha, threads=8)
    Nt = order[0] * order[1] * order[2]
    for name, Mg in (("fill", M.cpu().numpy()), ("moments+contract", M2.cpu().numpy())):
        assert np.isfinite(Mg).all(), f"{name}: non-finite entries ({ctx.kernel_path})"
        for e in range(n):
            ok, msg, _ = blocks_close(Mg[e], Mo[e], nc, Nt)
            assert ok, f"{name} element {e}: {msg} ({ctx.kernel_path})"


@pytest.mark.parametrize("case", shape_grid.ALL, ids=shape_grid.shape_id)
def test_large_family_moment_kernels_agree(case):
    # both moment kernels of the large-order family (w-first register tiles, the default
    # where its first pass is wide enough, and the u-first kernel) on every grid shape
    # of the family: same moments to rounding (the sums run in a different order)
    nc, order, kinds, nq, basis = case
    res = []
    for w in ("0", "1"):
        ctx = capi.Context(nc, order, kinds, nq, basis=basis, options={"P2S_LARGE_MOMW": w})
        if not ctx.kernel_path.startswith("large-order"):
            ctx.close()
            pytest.skip("not a large-order shape")
        n = 2
        st = torch.cuda.current_stream().cuda_stream
        a = torch.empty((n, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
        ctx.alpha_generate(O.ALPHA_SINE, 0.5, 3.0, 29 + sum(order), 0, n, a, st)
        I = torch.zeros((n, ctx.moments_per_elem), dtype=torch.float64, device="cuda")
        ctx.moments(a, I, n, st)
        torch.cuda.synchronize()
        res.append(I.cpu().numpy())
        ctx.close()
    scale = np.abs(res[0]).max()
    assert scale > 0 and np.isfinite(res[1]).all()
    assert np.abs(res[0] - res[1]).max() <= 1e-12 * scale
