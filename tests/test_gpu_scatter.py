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


def _serial_reference_order(E, free, sign, n_free):
    """assemble_global's loop order and arithmetic (assembly.cpp:626-641), in
    pure Python floats (IEEE doubles, no FMA): the bitwise target."""
    G = [[0.0] * n_free for _ in range(n_free)]
    for e in range(E.shape[0]):
        for i in range(E.shape[1]):
            gi = int(free[e][i])
            if gi < 0:
                continue
            si = float(sign[e][i])
            for j in range(E.shape[1]):
                gj = int(free[e][j])
                if gj < 0:
                    continue
                w = si * float(sign[e][j])
                G[gi][gj] = G[gi][gj] + w * float(E[e][i][j])
    return np.array(G)


@pytest.mark.parametrize("n_local,n_elem,n_free,ld_pad", [(27, 40, 60, 0), (64, 9, 150, 3), (5, 1, 7, 1)])
def test_ordered_scatter_is_the_reference_sum_bitwise(n_local, n_elem, n_free, ld_pad):
    """p2s_scatter_add_ordered reproduces the reference's serial sum bit for bit
    (elements ascending, then local rows; no FMA), and is run-to-run identical."""
    rng = np.random.default_rng(7 + n_local)
    ld = n_local + ld_pad
    E = rng.standard_normal((n_elem, n_local, ld))
    # each element: distinct free indices (or -1), shared between elements
    free = np.full((n_elem, n_local), -1, dtype=np.int32)
    for e in range(n_elem):
        pick = rng.choice(n_free, size=n_local, replace=False)
        keep = rng.random(n_local) < 0.9
        free[e][keep] = pick[keep]
    sign = rng.choice([-1.0, 1.0], size=(n_elem, n_local))
    plan = capi.ScatterPlan(free, n_free)
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for _ in range(2):
        G = torch.zeros((n_free, n_free + 1), dtype=torch.float64, device="cuda")
        plan.add(torch.from_numpy(E).cuda(), n_local * ld, ld, torch.from_numpy(free).cuda(),
                 torch.from_numpy(sign).cuda(), G, n_free + 1, st)
        torch.cuda.synchronize()
        outs.append(G.cpu().numpy())
    want = _serial_reference_order(E[:, :, :n_local], free, sign, n_free)
    assert np.array_equal(outs[0][:, :n_free], want)
    assert np.array_equal(outs[0], outs[1])
    assert np.all(outs[0][:, n_free:] == 0.0)


def test_cheb2d_ordered_scatter_bitwise():
    M, N, nq = 3, 2, 8
    ctx = capi.Cheb2dContext(M, N, nq, conforming=True)
    sz = ctx.sizes
    n_elem, n_local, n_free = 6, sz.n_eu + sz.n_ev, 40
    rng = np.random.default_rng(11)
    blocks = rng.standard_normal((n_elem, sz.blocks_per_elem))
    free = np.full((n_elem, n_local), -1, dtype=np.int32)
    for e in range(n_elem):
        free[e] = rng.choice(n_free, size=n_local, replace=False)
    free[0][0] = -1
    sign = rng.choice([-1.0, 1.0], size=(n_elem, n_local))
    plan = capi.ScatterPlan(free, n_free)
    S = torch.zeros((n_free, n_free), dtype=torch.float64, device="cuda")
    Mm = torch.zeros((n_free, n_free), dtype=torch.float64, device="cuda")
    ctx.scatter_ordered(plan, torch.from_numpy(blocks).cuda(), torch.from_numpy(free).cuda(),
                        torch.from_numpy(sign).cuda(), S, Mm, n_free)
    torch.cuda.synchronize()
    for which, G in (("S", S), ("M", Mm)):
        full = np.zeros((n_elem, n_local, n_local))
        for e in range(n_elem):
            b = ctx.split_blocks(blocks[e])
            full[e] = np.block([[b[which + "uu"], b[which + "uv"]], [b[which + "vu"], b[which + "vv"]]])
        assert np.array_equal(G.cpu().numpy(), _serial_reference_order(full, free, sign, n_free))
