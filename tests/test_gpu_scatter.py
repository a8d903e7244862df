"""Global scatter-add on the GPU (p2s_scatter_add / p2s_cheb2d_scatter; the
reference's assemble_global, assembly.cpp:594-652) against a numpy restatement
(np.add.at with orientation signs and constrained DOFs dropped), and the full
reference pipeline through tests/test_gpu_reference2d.py's drop-in binary."""
import numpy as np
import pytest
import torch

from paper_1703_09619_b200 import capi

pytestmark = pytest.mark.gpu


def _reference_scatter(E, free, sign, n_free):
    G = np.zeros((n_free, n_free))
    for e in range(E.shape[0]):
        keep = np.nonzero(free[e] >= 0)[0]
        gi = free[e][keep]
        w = np.outer(sign[e][keep], sign[e][keep]) * E[e][np.ix_(keep, keep)]
        np.add.at(G, (gi[:, None], gi[None, :]), w)
    return G


@pytest.mark.parametrize("n_local,n_elem,n_free,ld_pad", [(27, 40, 200, 0), (648, 6, 1500, 3),
                                                         (5, 1, 7, 1)])
def test_scatter_matches_numpy(n_local, n_elem, n_free, ld_pad):
    rng = np.random.default_rng(n_local)
    ld = n_local + ld_pad
    E = rng.standard_normal((n_elem, n_local, ld))
    free = rng.integers(-1, n_free, size=(n_elem, n_local)).astype(np.int32)
    sign = rng.choice([-1.0, 1.0], size=(n_elem, n_local))
    G = torch.zeros((n_free, n_free + 2), dtype=torch.float64, device="cuda")
    dE = torch.from_numpy(E).cuda()
    capi.scatter_add(dE, n_local * ld, ld, n_local, torch.from_numpy(free).cuda(),
                     torch.from_numpy(sign).cuda(), n_elem, G, n_free + 2,
                     torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    want = _reference_scatter(E[:, :, :n_local], free, sign, n_free)
    got = G.cpu().numpy()
    assert np.abs(got[:, :n_free] - want).max() <= 1e-13 * max(1.0, np.abs(want).max())
    assert np.all(got[:, n_free:] == 0.0)


def test_cheb2d_scatter_matches_numpy():
    M, N, nq = 3, 2, 8
    ctx = capi.Cheb2dContext(M, N, nq, conforming=True)
    sz = ctx.sizes
    n_elem, n_local = 5, ctx.sizes.n_eu + ctx.sizes.n_ev
    rng = np.random.default_rng(3)
    blocks = rng.standard_normal((n_elem, sz.blocks_per_elem))
    free = rng.integers(-1, 30, size=(n_elem, n_local)).astype(np.int32)
    sign = rng.choice([-1.0, 1.0], size=(n_elem, n_local))
    S = torch.zeros((30, 30), dtype=torch.float64, device="cuda")
    Mm = torch.zeros((30, 30), dtype=torch.float64, device="cuda")
    ctx.scatter(torch.from_numpy(blocks).cuda(), torch.from_numpy(free).cuda(),
                torch.from_numpy(sign).cuda(), n_elem, S, Mm, 30)
    torch.cuda.synchronize()
    for which, G in (("S", S), ("M", Mm)):
        full = np.zeros((n_elem, n_local, n_local))
        for e in range(n_elem):
            b = ctx.split_blocks(blocks[e])
            p = "S" if which == "S" else "M"
            full[e] = np.block([[b[p + "uu"], b[p + "uv"]], [b[p + "vu"], b[p + "vv"]]])
        want = _reference_scatter(full, free, sign, 30)
        assert np.abs(G.cpu().numpy() - want).max() <= 1e-13 * np.abs(want).max()


def test_scatter_errors():
    with pytest.raises(capi.InvalidArgument):
        capi.scatter_add(0, 10, 2, 3, 0, 0, 1, 0, 3)   # ld_elem < n_local
    capi.scatter_add(0, 9, 3, 3, 0, 0, 0, 0, 3)        # empty batch: no-op
