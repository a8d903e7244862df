"""Fill from element geometry (p2s_geometry_generate / p2s_alpha_from_geometry /
p2s_fill_geometry): alpha sampled on the device from
the hexahedra's trilinear maps and materials (the 3-D analogue of
build_element_quad, assembly.cpp:51-119), bit-identical to the seeded JACOBIAN
alpha the parity tests pin against the oracle, and the chunked fill (alpha of a
chunk produced into an L2-resident double buffer while the fill consumes the
other) bit-identical to the two-step fill."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1703_09619_b200 import capi
from paper_1703_09619_b200.configs import CONFIGS

from helpers import blocks_close, oracle_for

pytestmark = pytest.mark.gpu


def _ctx(name):
    cfg = CONFIGS[name]
    return cfg, capi.Context(**cfg.problem())


def test_alpha_from_geometry_equals_seeded_jacobian_alpha():
    cfg, ctx = _ctx("c2")
    n, seed = 37, 99
    sp = torch.cuda.current_stream().cuda_stream
    geom = torch.empty((n, ctx.GEOM_DOUBLES), dtype=torch.float64, device="cuda")
    ctx.geometry_generate(cfg.alpha_lo, cfg.alpha_hi, seed, 5, n, geom, sp)
    a1 = torch.empty((n, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    a2 = torch.empty_like(a1)
    ctx.alpha_from_geometry(geom, n, a1, sp)
    ctx.alpha_generate(O.ALPHA_JACOBIAN, cfg.alpha_lo, cfg.alpha_hi, seed, 5, n, a2, sp)
    torch.cuda.synchronize()
    # same coupling as the seeded JACOBIAN generator (which rounds like the host;
    # this kernel contracts FMAs and uses one reciprocal per point)
    torch.testing.assert_close(a1, a2, rtol=1e-13, atol=1e-14)
    # and the oracle's host generator (libm vs CUDA sin: ULP-level differences)
    o = oracle_for(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    ah = o.alpha(O.ALPHA_JACOBIAN, cfg.alpha_lo, cfg.alpha_hi, seed, 5, n)
    np.testing.assert_allclose(a1.cpu().numpy(), ah, rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("mode", [2, 1, 0])
def test_fill_geometry_matches_two_step_fill_and_oracle(mode, monkeypatch):
    """P2S_GEO_MODE 0 (default): alpha via the L2 double buffer -- bit-identical to
    p2s_fill(p2s_alpha_from_geometry(...)); 1: each pair's CTA recomputes the
    geometry; 2: one cluster of 9 CTAs per element shares the per-point geometry
    through DSMEM.  All against the oracle on host alpha."""
    monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_GEO_MODE", str(mode))
    chunked = mode == 0
    cfg, ctx = _ctx("c2")
    assert "fused" in ctx.kernel_path
    n = 150  # > 2 chunks of the internal alpha double buffer
    sp = torch.cuda.current_stream().cuda_stream
    geom = torch.empty((n, ctx.GEOM_DOUBLES), dtype=torch.float64, device="cuda")
    ctx.geometry_generate(cfg.alpha_lo, cfg.alpha_hi, 7, 0, n, geom, sp)
    alpha = torch.empty((n, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    ctx.alpha_from_geometry(geom, n, alpha, sp)
    M1 = torch.empty((n, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
    M2 = torch.full_like(M1, float("nan"))
    ctx.fill(alpha, M1, ctx.n_tot, n, sp)
    ctx.fill_geometry(geom, M2, ctx.n_tot, n, sp)
    torch.cuda.synchronize()
    Nt = cfg.order[0] * cfg.order[1] * cfg.order[2]
    if chunked:
        assert torch.equal(M1, M2)
    else:
        for e in (0, 1, 77, 149):
            ok, msg, _ = blocks_close(M2[e].cpu().numpy(), M1[e].cpu().numpy(), cfg.n_comp, Nt)
            assert ok, msg
    o = oracle_for(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    pick = [0, 63, 149]
    ah = o.alpha(O.ALPHA_JACOBIAN, cfg.alpha_lo, cfg.alpha_hi, 7, 0, n)[pick]
    Mo = o.fill(ah, threads=8)
    for i, e in enumerate(pick):
        ok, msg, _ = blocks_close(M2[e].cpu().numpy(), Mo[i], cfg.n_comp, Nt)
        assert ok, msg


def test_fill_geometry_errors():
    cfg, ctx = _ctx("c2")
    with pytest.raises(capi.InvalidArgument):
        ctx.fill_geometry(0, 0, ctx.n_tot - 1, 1)
    ctx.fill_geometry(0, 0, ctx.n_tot, 0)  # empty batch: no-op


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_folded_hexahedron_raises_geometry_error(mode, monkeypatch):
    """A hexahedron folded through itself (two corner layers swapped: det J < 0)
    is the reference's GeometryError (assembly.cpp:95-99) on every geometry
    entry point and mode; valid records still fill afterwards (the flag is reset
    per call)."""
    monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_GEO_MODE", str(mode))
    cfg, ctx = _ctx("c2")
    n = 5
    sp = torch.cuda.current_stream().cuda_stream
    geom = torch.empty((n, ctx.GEOM_DOUBLES), dtype=torch.float64, device="cuda")
    ctx.geometry_generate(cfg.alpha_lo, cfg.alpha_hi, 3, 0, n, geom, sp)
    bad = geom.clone()
    corners = bad[3, :24].view(8, 3).clone()
    bad[3, :24] = corners[[4, 5, 6, 7, 0, 1, 2, 3]].reshape(-1)  # w -> -w: mirrored element
    alpha = torch.empty((n, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    M = torch.empty((n, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
    with pytest.raises(capi.GeometryError):
        ctx.alpha_from_geometry(bad, n, alpha, sp)
    with pytest.raises(capi.GeometryError):
        ctx.fill_geometry(bad, M, ctx.n_tot, n, sp)
    ctx.alpha_from_geometry(geom, n, alpha, sp)
    ctx.fill_geometry(geom, M, ctx.n_tot, n, sp)
    torch.cuda.synchronize()
    assert torch.isfinite(M).all()
