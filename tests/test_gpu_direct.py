"""GPU direct-quadrature fill (p2s_direct_*, the paper's ablation baseline;
reference assemble_direct_element, assembly.cpp:134-274) against the oracle's
direct fill (por_direct) and against the GPU p2s fill: the product-to-sum
identity is exact at the quadrature nodes, so both compute the same discrete
sum and must agree under the reference comparator at rtol 1e-12."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1703_09619_b200 import capi
from paper_1703_09619_b200.capi import DD, DP, PD, PP
from paper_1703_09619_b200.configs import CONFIGS

from helpers import blocks_close, oracle_for

pytestmark = pytest.mark.gpu


def _direct(dctx, alpha, n_tot, ld=None):
    n = alpha.shape[0]
    ld = ld or n_tot
    a = torch.from_numpy(np.ascontiguousarray(alpha)).cuda()
    M = torch.full((n, n_tot, ld), float("nan"), dtype=torch.float64, device="cuda")
    dctx.fill(a, M, ld, n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return M.cpu().numpy()


CASES = [
    (1, (4, 4, 4), [PP], (8, 8, 8), O.ALPHA_SINE, 3),
    (3, (3, 3, 3), [PP, DD], (6, 6, 6), O.ALPHA_JACOBIAN, 3),
    (1, (4, 3, 3), [(DP, PD, PP), (PD, DP, DD)], (9, 5, 7), O.ALPHA_SINE, 2),
    (1, (2, 6, 5), [PP, DD], (4, 9, 8), O.ALPHA_SINE, 2),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}c-{c[1]}-{len(c[2])}t")
def test_direct_matches_oracle_direct(case):
    n_comp, order, kinds, nq, ak, n = case
    o = oracle_for(n_comp, order, kinds, nq)
    dctx = capi.DirectContext(n_comp, order, kinds, nq)
    alpha = o.alpha(ak, 0.5, 3.0, 5, 0, n)
    Mg = _direct(dctx, alpha, o.n_tot, ld=o.n_tot + 3)
    Md = o.direct(alpha, threads=8)
    Nt = order[0] * order[1] * order[2]
    assert np.isnan(Mg[:, :, o.n_tot:]).all()
    for e in range(n):
        ok, msg, _ = blocks_close(Mg[e, :, :o.n_tot], Md[e], n_comp, Nt)
        assert ok, f"element {e}: {msg}"


@pytest.mark.parametrize("name,n", [("c2", 4), ("c3", 3)])
def test_direct_equals_p2s_on_configs(name, n):
    cfg = CONFIGS[name]
    pb = (cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    ctx = capi.Context(*pb)
    dctx = capi.DirectContext(*pb)
    o = oracle_for(*pb)
    alpha = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 9, 0, n)
    a = torch.from_numpy(alpha).cuda()
    Mp = torch.empty((n, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
    ctx.fill(a, Mp, ctx.n_tot, n, torch.cuda.current_stream().cuda_stream)
    Md = _direct(dctx, alpha, ctx.n_tot)
    Mp = Mp.cpu().numpy()
    Nt = cfg.order[0] * cfg.order[1] * cfg.order[2]
    for e in range(n):
        ok, msg, _ = blocks_close(Mp[e], Md[e], cfg.n_comp, Nt)
        assert ok, f"element {e}: {msg}"


def test_direct_errors():
    dctx = capi.DirectContext(1, (2, 2, 2), [PP], (3, 3, 3))
    with pytest.raises(capi.InvalidArgument):
        dctx.fill(0, 0, 4, 1)          # ld_M < n_tot
    with pytest.raises(capi.InvalidArgument):
        capi.DirectContext(1, (2, 2, 2), [PP], (0, 3, 3))
    dctx.fill(0, 0, 8, 0)              # empty batch is a no-op
