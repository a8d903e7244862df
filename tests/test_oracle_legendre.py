"""CPU: the 3-D Legendre oracle (no reference test covers 3-D).

Pins: pointwise product-to-sum identities (the role of
test_chebyshev.cpp:131-152), p2s == direct full quadrature on the same alpha
(acceptance.cpp:84-121 / test_assembly.cpp:142-172 pattern), known answers,
scaling laws (test_assembly.cpp:202-237) and thread-count determinism
(test_assembly.cpp:392-403).
"""
import numpy as np
import pytest

from oracle import oracle as O

from helpers import RTOL, blocks_close


@pytest.mark.parametrize("kind", [O.PP, O.DD, O.DP, O.PD])
def test_legendre_identities_pointwise(kind):
    rng = np.random.default_rng(2024)
    pts = [-1.0, 1.0, 0.0] + list(rng.uniform(-1, 1, 60))
    for N in (1, 2, 4, 6, 8, 10, 16):
        C = O.legendre_coef(kind, N)
        K = C.shape[2]
        assert K == O.kernel_count(kind, N)
        for x in pts:
            P, dP = O.legendre_eval(2 * N + 2, x)
            fa = dP if kind in (O.DD, O.DP) else P
            fb = dP if kind in (O.DD, O.PD) else P
            lhs = np.outer(fa[:N], fb[:N])
            rhs = C @ P[:K]
            scale = max(1.0, np.abs(lhs).max())
            assert np.abs(lhs - rhs).max() <= 1e-12 * scale, (kind, N, x)


@pytest.mark.parametrize("kind", [O.PP, O.DD, O.DP, O.PD])
def test_legendre_band_structure(kind):
    # nonzeros only at k = lo, lo+2, .., hi (the bands the kernels hard-code)
    from paper_1703_09619_b200.bands import band_hi, band_lo
    N = 9
    C = O.legendre_coef(kind, N)
    for a in range(N):
        for b in range(N):
            lo, hi = band_lo(kind, a, b), band_hi(kind, a, b)
            nz = set(np.nonzero(C[a, b])[0].tolist())
            assert nz == set(range(lo, hi + 1, 2)) if hi >= lo else nz == set(), (a, b, nz)


def test_pp_known_values():
    C = O.legendre_coef(O.PP, 3)
    # P1 P1 = (2 P2 + P0) / 3 ;  P2 P1 = (3 P3 + 2 P1) / 5
    assert np.allclose(C[1, 1, [0, 2]], [1 / 3, 2 / 3], rtol=1e-15)
    assert np.allclose(C[2, 1, [1, 3]], [2 / 5, 3 / 5], rtol=1e-15)


CASES = [
    (1, (4, 4, 4), [O.PP], (8, 8, 8), O.ALPHA_SINE),
    (3, (3, 3, 3), [O.PP, O.DD], (7, 7, 7), O.ALPHA_JACOBIAN),
    (1, (3, 5, 4), [O.DP, (O.PP, O.PD, O.DD)], (8, 9, 7), O.ALPHA_SINE),
    (1, (4, 3, 2), [O.PP, O.DD], (9, 8, 6), O.ALPHA_EXPSIN),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}c-{c[1]}")
def test_p2s_equals_direct_quadrature(case):
    n_comp, order, kinds, nq, ak = case
    o = O.Oracle(n_comp, order, kinds, nq)
    alpha = o.alpha(ak, 0.5, 3.0, 31, 0, 2)
    M = o.fill(alpha)
    D = o.direct(alpha)
    Nt = order[0] * order[1] * order[2]
    for e in range(2):
        ok, msg, _ = blocks_close(M[e], D[e], n_comp, Nt, RTOL)
        assert ok, msg


def test_constant_alpha_mass_is_diagonal():
    # alpha = 1: the PP block is the Legendre mass matrix prod 2/(2m+1)
    o = O.Oracle(1, (4, 3, 5), [O.PP], (8, 8, 8))
    M = o.fill(np.ones((1, o.alpha_per_elem)))[0]
    d = np.array([8 / ((2 * m + 1) * (2 * n + 1) * (2 * p + 1))
                  for m in range(4) for n in range(3) for p in range(5)])
    assert np.abs(np.diag(M) - d).max() <= 1e-14
    assert np.abs(M - np.diag(np.diag(M))).max() <= 1e-14


def test_scaling_laws_exact():
    o = O.Oracle(1, (3, 3, 3), [O.PP, O.DD], (6, 6, 6))
    a = o.alpha(O.ALPHA_SINE, 0.5, 3.0, 3, 0, 2)
    M1 = o.fill(a)
    M2 = o.fill(2.0 * a)
    assert np.array_equal(M2, 2.0 * M1)   # doubling is exact in IEEE


def test_thread_count_determinism():
    o = O.Oracle(3, (3, 3, 2), [O.PP, O.DD], (6, 5, 4))
    a = o.alpha(O.ALPHA_JACOBIAN, 0.5, 3.0, 4, 0, 9)
    assert np.array_equal(o.fill(a, threads=1), o.fill(a, threads=4))
    assert np.array_equal(o.moments(a, threads=1), o.moments(a, threads=3))


def test_alpha_generator_counter_based():
    o = O.Oracle(3, (2, 2, 2), [O.PP, O.DD], (4, 4, 4))
    full = o.alpha(O.ALPHA_JACOBIAN, 0.5, 3.0, 99, 0, 6)
    part = o.alpha(O.ALPHA_JACOBIAN, 0.5, 3.0, 99, 3, 3)
    assert np.array_equal(full[3:], part)       # any element regenerates independently
    # Jacobian factors: mass term symmetric positive definite per point
    S = 2
    a = full[0].reshape(3, 3, S, -1)
    assert np.allclose(a[:, :, 0], a[:, :, 0].transpose(1, 0, 2))
    assert np.all(np.linalg.eigvalsh(np.moveaxis(a[:, :, 0], 2, 0)) > 0)
