"""Conforming (hierarchical) basis: SURVEY.md §8(f) rank 2.

Pins the change of basis to the reference: conforming_matrix (assembly.cpp:
476-489) bitwise, and apply_conforming_transform (assembly.cpp:491-574) on the
reference's own element blocks, restated as T_rows^T B T_cols with the
Kronecker structure of its four in-place variants.  Then the 3-D oracle:
M_conforming == T^T M_modal T with T = R (x) R (x) R per component, and p2s ==
direct quadrature in the conforming basis.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from helpers import RTOL, blocks_close, oracle_for

HERE = os.path.dirname(os.path.abspath(__file__))
PP, DD, DP, PD = O.PP, O.DD, O.DP, O.PD


def _golden():
    return np.load(os.path.join(HERE, "golden", "ref2d_elements.npz"))


@pytest.mark.parametrize("n", range(2, 18))
def test_conforming_matrix_matches_reference(n):
    g = _golden()
    assert np.array_equal(O.conforming_matrix(n), g[f"conforming_matrix__{n}"])


def test_conforming_transform_matches_reference_blocks():
    """Every fixture element: the reference's transformed blocks equal
    T_r^T B T_c with R from the oracle (rows/cols 'inner' = I (x) R, 'outer' = R (x) I)."""
    g = _golden()
    for tag in g["tags"]:
        M, N = int(g[f"{tag}__M"]), int(g[f"{tag}__N"])
        if M < 1 or N < 1:
            continue
        inner = np.kron(np.eye(M), O.conforming_matrix(N + 1))   # E_u = m (N+1) + n
        outer = np.kron(O.conforming_matrix(M + 1), np.eye(N))   # E_v = m N + n
        T = {"u": inner, "v": outer}
        for blk in ("Suu", "Suv", "Svv", "Muu", "Muv", "Mvv", "Svu", "Mvu"):
            r, c = blk[1], blk[2]
            B = g[f"{tag}__p2s_{blk}"]
            want = g[f"{tag}__conf_{blk}"]
            got = T[r].T @ B @ T[c]
            scale = max(np.abs(want).max(), 1e-300)
            assert np.abs(got - want).max() <= 1e-14 * scale, (tag, blk)


def _kron3(order):
    return np.kron(np.kron(O.conforming_matrix(order[0]), O.conforming_matrix(order[1])),
                   O.conforming_matrix(order[2]))


CASES = [
    (1, (4, 4, 4), [PP], (8, 8, 8)),
    (3, (3, 3, 3), [PP, DD], (6, 6, 6)),
    (1, (4, 3, 3), [(DP, PD, PP), (PD, DP, DD)], (9, 5, 7)),
    (1, (2, 5, 3), [PP, DD], (5, 8, 6)),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}c-{c[1]}-{len(c[2])}t")
def test_conforming_equals_transformed_modal(case):
    n_comp, order, kinds, nq = case
    om = oracle_for(n_comp, order, kinds, nq, basis=0)
    oc = oracle_for(n_comp, order, kinds, nq, basis=1)
    alpha = om.alpha(O.ALPHA_SINE, 0.5, 3.0, 3, 0, 2)
    Mm = om.fill(alpha, threads=4)
    Mc = oc.fill(alpha, threads=4)
    T = np.kron(np.eye(n_comp), _kron3(order))
    Nt = order[0] * order[1] * order[2]
    for e in range(2):
        ok, msg, _ = blocks_close(Mc[e], T.T @ Mm[e] @ T, n_comp, Nt, rtol=1e-13)
        assert ok, msg


@pytest.mark.parametrize("case", CASES[:3], ids=lambda c: f"{c[0]}c-{c[1]}-{len(c[2])}t")
def test_conforming_p2s_equals_direct(case):
    n_comp, order, kinds, nq = case
    oc = oracle_for(n_comp, order, kinds, nq, basis=1)
    alpha = oc.alpha(O.ALPHA_SINE, 0.5, 3.0, 8, 0, 2)
    Mp = oc.fill(alpha, threads=4)
    Md = oc.direct(alpha, threads=4)
    Nt = order[0] * order[1] * order[2]
    for e in range(2):
        ok, msg, _ = blocks_close(Mp[e], Md[e], n_comp, Nt, rtol=RTOL)
        assert ok, msg


def test_conforming_needs_order_two():
    with pytest.raises(Exception):
        oracle_for(1, (1, 3, 3), [PP], (4, 4, 4), basis=1)
