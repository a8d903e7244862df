"""CPU: the oracle pinned against the REFERENCE itself.

Fixtures tests/golden/ref2d_*.npz were produced by the reference library
compiled from /root/reference/proj/src (oracle/refbuild, generator
tests/golden/make_ref2d_golden.py).  The oracle's generic separable engine --
the same moments / banded-contraction / direct code the 3-D Legendre oracle
uses -- is run in the reference's 2-D Chebyshev specialisation and must
reproduce the reference's kernel tables and element matrices.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    return np.load(os.path.join(GOLD, name))


def test_gauss_legendre_bitwise_equal_to_reference():
    # quadrature.cpp:27-53, n = 1..48
    q = _load("ref2d_quadrature.npz")
    for n in range(1, 49):
        x, w = O.gauss_legendre(n)
        assert np.array_equal(x, q[f"nodes_{n}"]), n
        assert np.array_equal(w, q[f"weights_{n}"]), n


def test_gauss_legendre_closed_forms_and_exactness():
    # test_quadrature.cpp:10-65
    x, w = O.gauss_legendre(1)
    assert abs(x[0]) <= 1e-15 and abs(w[0] - 2.0) <= 1e-15
    x, w = O.gauss_legendre(2)
    assert np.allclose(x, [-1 / np.sqrt(3), 1 / np.sqrt(3)], rtol=1e-14)
    x, w = O.gauss_legendre(3)
    assert abs(np.sum(w * x ** 4) - 0.4) <= 1e-14
    rng = np.random.default_rng(5)
    for n in range(1, 13):
        x, w = O.gauss_legendre(n)
        assert abs(w.sum() - 2.0) <= 1e-13
        assert np.all(np.diff(x) > 0) and np.allclose(x, -x[::-1], atol=1e-14)
        for _ in range(5):
            c = rng.uniform(-2, 2, 2 * n)
            exact = sum(2 * c[k] / (k + 1) for k in range(0, 2 * n, 2))
            num = np.sum(w * np.polyval(c[::-1], x))
            assert abs(num - exact) <= 1e-12 * max(1, abs(exact))


def test_family_values_match_reference():
    # eval_T / eval_U / eval_Tns (chebyshev.cpp:23-108), degrees 0..40, incl. u = +-1
    f = _load("ref2d_families.npz")
    pts = f["points"]
    vals = f["values"]
    for fam in range(3):
        for n in range(41):
            mine = np.array([O.cheb_eval(fam, n, u) for u in pts])
            ref = vals[fam, n]
            assert np.allclose(mine, ref, rtol=1e-15, atol=1e-15 * max(1.0, np.abs(ref).max())), (fam, n)


def test_product_to_sum_expansions_match_reference():
    # product_to_sum (chebyshev.cpp:156-178) for T/U, degrees <= 20
    f = _load("ref2d_families.npz")
    rows, nterms = f["p2s"], f["p2s_nterms"]
    for r, nt in zip(rows, nterms):
        fa, a, fb, b = (int(v) for v in r[:4])
        mine = sorted(O.cheb_p2s(fa, a, fb, b))
        ref = sorted((r[4 + 3 * i], int(r[5 + 3 * i]), int(r[6 + 3 * i])) for i in range(nt))
        assert mine == ref, (fa, a, fb, b)


def _cases():
    e = _load("ref2d_elements.npz")
    return e, [str(t) for t in e["tags"]]


E, TAGS = _cases()
BLOCKS = ["Suu", "Suv", "Svu", "Svv", "Muu", "Muv", "Mvu", "Mvv"]


@pytest.mark.parametrize("tag", TAGS)
def test_engine_reproduces_reference_element(tag):
    g = lambda k: E[f"{tag}__{k}"]
    M, N, nq = int(g("M")), int(g("N")), int(g("nq"))
    tables, p2s, direct = O.cheb2d_element(M, N, nq, g("nodes"), g("ws"), g("wuu"), g("wuv"), g("wvv"))
    # kernel tables (compute_kernel_tables, assembly.cpp:276-314)
    for k in ("Ks", "Kuu", "Kuv", "Kvv"):
        ok, ij = O.block_close(tables[k], g(k), 1e-12)
        assert ok, (tag, k, ij)
    # element matrices: p2s (assembly.cpp:375-474) and direct (:142-274)
    for b in BLOCKS:
        ok, ij = O.block_close(p2s[b], g("p2s_" + b), 1e-12)
        assert ok, (tag, "p2s", b, ij)
        ok, ij = O.block_close(direct[b], g("direct_" + b), 1e-12)
        assert ok, (tag, "direct", b, ij)


def test_reference_known_answers():
    # test_assembly.cpp:96-140 on the identity element, orders (2, 2), nq = 10
    g = lambda k: E[f"identity_2x2_nq10__{k}"]
    tables, p2s, _ = O.cheb2d_element(2, 2, 10, g("nodes"), g("ws"), g("wuu"), g("wuv"), g("wvv"))
    assert tables["Kuu"][0, 0] == 0.0
    assert abs(tables["Kuu"][2, 0] - (-4.0)) <= 4e-13
    assert abs(tables["Ks"][2, 2] - 4.0) <= 4e-13
    assert abs(tables["Ks"][4, 2] - 16.0 / 3.0) <= 16 / 3 * 1e-13
    for m in range(5):
        for n in range(5):
            if m < 2 or n < 2:
                assert tables["Ks"][m, n] == 0.0
            if m < 2:
                assert tables["Kuu"][m, n] == 0.0
            if n < 2:
                assert tables["Kvv"][m, n] == 0.0
    eu = lambda m, n: m * 3 + n
    assert abs(p2s["Muu"][eu(0, 0), eu(0, 0)] - 4.0) <= 4e-13
    assert abs(p2s["Suu"][eu(1, 1), eu(1, 1)] - 16.0 / 3.0) <= 16 / 3 * 1e-13
    # counters of the reference for this case
    assert int(g("n_integrals")) == 3 * 25 + 16
    assert int(g("n_mass_uu_integrals")) == 25


def test_comparator_semantics():
    # verify.cpp:81-99: relative OR block-floor
    a = np.array([[1.0, 1e-20], [2.0, 3.0]])
    b = a.copy()
    b[0, 1] = 2e-20           # relative error 1, but below 1e-12 * block max -> pass
    assert O.block_close(a, b, 1e-12)[0]
    b = a.copy()
    b[1, 1] = 3.0 * (1 + 1e-11)
    assert O.block_close(a, b, 1e-12) == (False, (1, 1))
    assert O.block_close(a, b, 1e-10)[0]
