"""3-D golden fixtures (tests/golden/p2s3d_*.npz, tests/golden/make_3d_golden.py).

CPU: the oracle reproduces its committed fixtures (guards the checker).
GPU: the sm_100a path reproduces the fixtures through the C-ABI.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1703_09619_b200.configs import CONFIGS

from helpers import RTOL, blocks_close

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _g(name):
    return np.load(os.path.join(GOLD, f"p2s3d_{name}.npz"))


def _rows_close(a, b, rtol=RTOL):
    scale = max(np.abs(a).max(), np.abs(b).max())
    return np.all(np.abs(a - b) <= np.maximum(rtol * np.maximum(np.abs(a), np.abs(b)), 1e-12 * scale))


def test_oracle_reproduces_full_fixtures():
    g = _g("c1")
    cfg = CONFIGS["c1"]
    o = O.Oracle(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    a = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, int(g["seed"]), 0, 1)
    assert np.array_equal(a, g["alpha"])
    assert O.block_close(o.fill(a)[0], g["M"][0], RTOL)[0]
    g = _g("vec3")
    o = O.Oracle(3, (3, 3, 3), [O.PP, O.DD], (6, 6, 6))
    M = o.fill(g["alpha"])
    for e in range(2):
        assert blocks_close(M[e], g["M"][e], 3, 27)[0]


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_oracle_reproduces_checksum_fixtures(name):
    g = _g(name)
    cfg = CONFIGS[name]
    o = O.Oracle(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    a = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, int(g["seed"]), int(g["e0"]), 1)
    assert abs(a.sum() - g["alpha_sum"]) <= 1e-12 * abs(g["alpha_abs_sum"])
    M = o.fill(a, threads=8)[0]
    assert _rows_close(np.diag(M), g["diag"])
    assert _rows_close(M[0], g["first_row"])
    assert _rows_close(np.abs(M).sum(axis=1), g["row_abs_sum"])


@pytest.mark.gpu
def test_gpu_matches_full_fixtures():
    import torch
    from paper_1703_09619_b200 import capi
    for name, prob, nc, Nt in [("c1", CONFIGS["c1"].problem(), 1, 64),
                               ("vec3", dict(n_comp=3, order=(3, 3, 3), kinds=[O.PP, O.DD],
                                             nq=(6, 6, 6)), 3, 27)]:
        g = _g(name)
        ctx = capi.Context(**prob)
        a = torch.from_numpy(g["alpha"]).cuda()
        n = a.shape[0]
        M = torch.empty((n, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
        ctx.fill(a, M, ctx.n_tot, n)
        I = torch.empty((n, ctx.moments_per_elem), dtype=torch.float64, device="cuda")
        ctx.moments(a, I, n)
        torch.cuda.synchronize()
        Mg = M.cpu().numpy()
        for e in range(n):
            ok, msg, _ = blocks_close(Mg[e], g["M"][e], nc, Nt)
            assert ok, (name, msg)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_gpu_matches_checksum_fixtures(name):
    import torch
    from paper_1703_09619_b200 import capi
    g = _g(name)
    cfg = CONFIGS[name]
    o = O.Oracle(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    a = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, int(g["seed"]), int(g["e0"]), 1)
    ctx = capi.Context(**cfg.problem())
    M = torch.empty((1, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
    ctx.fill(torch.from_numpy(a).cuda(), M, ctx.n_tot, 1)
    torch.cuda.synchronize()
    Mg = M[0].cpu().numpy()
    assert _rows_close(np.diag(Mg), g["diag"])
    assert _rows_close(Mg[0], g["first_row"])
    assert _rows_close(np.abs(Mg).sum(axis=1), g["row_abs_sum"])
