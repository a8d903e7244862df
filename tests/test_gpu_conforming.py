"""GPU fill in the conforming basis (P2S_BASIS_CONFORMING; SURVEY.md §8(f)
rank 2): the reference's change of basis folded into the product-to-sum
tables, against the oracle in the same basis (itself pinned to the reference's
conforming_matrix / apply_conforming_transform, tests/test_oracle_conforming.py)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1703_09619_b200 import capi
from paper_1703_09619_b200.capi import BASIS_CONFORMING, DD, DP, PD, PP
from paper_1703_09619_b200.configs import CONFIGS

from helpers import blocks_close, oracle_for

pytestmark = pytest.mark.gpu


def _fill(ctx, alpha):
    n = alpha.shape[0]
    a = torch.from_numpy(np.ascontiguousarray(alpha)).cuda()
    M = torch.full((n, ctx.n_tot, ctx.n_tot), float("nan"), dtype=torch.float64, device="cuda")
    ctx.fill(a, M, ctx.n_tot, n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return M.cpu().numpy()


CASES = [
    # n_comp, order, kinds, nq, env, expected path prefix
    (1, (4, 4, 4), [PP], (8, 8, 8), {}, "fused"),                        # generated module
    (1, (4, 4, 4), [PP], (8, 8, 8), {"P2S_FORCE_GENERIC": "1"}, "two-stage"),
    (1, (4, 4, 4), [PP], (8, 8, 8), {"P2S_NO_FUSED": "1"}, "two-stage: moments_v2_kernel + contract_v2"),
    (1, (4, 3, 3), [(DP, PD, PP), (PD, DP, DD)], (9, 5, 7), {"P2S_FORCE_JIT": "1"}, "fused"),
    (1, (4, 3, 3), [(DP, PD, PP), (PD, DP, DD)], (9, 5, 7), {"P2S_FORCE_JIT": "1", "P2S_JIT_FAMILY": "large"},
     "large-order"),
    (1, (7, 6, 5), [(DP, PD, PP), (PD, DP, DD)], (9, 8, 7), {"P2S_JIT_FAMILY": "large"},
     "large-order"),                                                                  # generated large
    (3, (3, 3, 3), [PP, DD], (6, 6, 6), {}, "two-stage: moments_v2_kernel + contract_v2"),
    (3, (3, 3, 3), [PP, DD], (6, 6, 6), {"P2S_FORCE_GENERIC": "1"}, "two-stage"),
    (1, (4, 3, 3), [(DP, PD, PP), (PD, DP, DD)], (9, 5, 7), {}, "fused"),                    # generated module
    (1, (5, 4, 3), [PP, DD], (8, 8, 6), {}, "large-order"),
    ("c2", None, None, None, {}, "fused"),
    ("c2", None, None, None, {"P2S_NO_FUSED": "1"}, "two-stage: moments_v2_kernel + contract_v2"),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[1]}-{sorted(c[4])}")
def test_conforming_fill_matches_oracle(case, monkeypatch):
    n_comp, order, kinds, nq, env, path = case
    for k, v in env.items():
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, k, v)
    if n_comp == "c2":
        cfg = CONFIGS["c2"]
        n_comp, order, kinds, nq = cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq
        ak, lo, hi, n = cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 3
    else:
        ak, lo, hi, n = O.ALPHA_SINE, 0.5, 3.0, 3
    ctx = capi.Context(n_comp, order, kinds, nq, basis=BASIS_CONFORMING)
    assert ctx.kernel_path.startswith(path), ctx.kernel_path
    o = oracle_for(n_comp, order, kinds, nq, basis=1)
    alpha = o.alpha(ak, lo, hi, 21, 0, n)
    Mg = _fill(ctx, alpha)
    Mo = o.fill(alpha, threads=8)
    Nt = order[0] * order[1] * order[2]
    for e in range(n):
        ok, msg, _ = blocks_close(Mg[e], Mo[e], n_comp, Nt)
        assert ok, f"element {e}: {msg}"


def test_conforming_direct_matches_oracle():
    pb = (3, (3, 3, 3), [PP, DD], (6, 6, 6))
    d = capi.DirectContext(*pb, basis=BASIS_CONFORMING)
    o = oracle_for(*pb, basis=1)
    alpha = o.alpha(O.ALPHA_JACOBIAN, 0.5, 3.0, 4, 0, 2)
    a = torch.from_numpy(alpha).cuda()
    M = torch.empty((2, d.n_tot, d.n_tot), dtype=torch.float64, device="cuda")
    d.fill(a, M, d.n_tot, 2, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    Mo = o.direct(alpha, threads=8)
    for e in range(2):
        ok, msg, _ = blocks_close(M[e].cpu().numpy(), Mo[e], 3, 27)
        assert ok, msg


def test_conforming_errors():
    with pytest.raises(capi.InvalidArgument):
        capi.Context(1, (1, 3, 3), [PP], (4, 4, 4), basis=BASIS_CONFORMING)
    with pytest.raises(capi.InvalidArgument):
        capi.Context(1, (3, 3, 3), [PP], (4, 4, 4), basis=7)
