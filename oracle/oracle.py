"""ctypes binding of the CPU ORACLE (liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / reference arm, as the checker.  The product package
(paper_1703_09619_b200) never imports this module.

See p2s_oracle.h for the reference file:line each function restates.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
# the same source built for speed (-ffp-contract=fast, FMA): CPU-baseline timing
# only (bench.py), never the checker
_LIB_FAST_PATH = os.path.join(_HERE, "liboracle_fast.so")

PP, DD, DP, PD = 0, 1, 2, 3
ALPHA_SINE, ALPHA_JACOBIAN, ALPHA_EXPSIN = 0, 1, 2
FAM_T, FAM_U, FAM_TNS = 0, 1, 2
MAX_TERMS = 4


def build(force: bool = False) -> str:
    """Compile liboracle.so (and liboracle_fast.so) with oracle/Makefile (gcc)."""
    if force or not os.path.exists(_LIB_PATH) or not os.path.exists(_LIB_FAST_PATH):
        subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    return _LIB_PATH


class Problem(C.Structure):
    _fields_ = [
        ("n_comp", C.c_int),
        ("order", C.c_int * 3),
        ("n_terms", C.c_int),
        ("kind", (C.c_int * 3) * MAX_TERMS),
        ("nq", C.c_int * 3),
        ("basis", C.c_int),
    ]


_libs = {}


def lib(fast: bool = False):
    if fast not in _libs:
        build()
        L = C.CDLL(_LIB_FAST_PATH if fast else _LIB_PATH)
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        L.por_gauss_legendre.argtypes = [C.c_int, dp, dp]
        L.por_conforming_matrix.argtypes = [C.c_int, dp]
        L.por_conforming_matrix.restype = None
        L.por_legendre_eval.argtypes = [C.c_int, C.c_double, dp, dp]
        L.por_kernel_count.argtypes = [C.c_int, C.c_int]
        L.por_kernel_count.restype = C.c_int
        L.por_legendre_coef.argtypes = [C.c_int, C.c_int, C.c_int, dp]
        L.por_create.argtypes = [C.POINTER(Problem)]
        L.por_create.restype = C.c_void_p
        L.por_destroy.argtypes = [C.c_void_p]
        for f in ("por_alpha_per_elem", "por_moments_per_elem"):
            getattr(L, f).argtypes = [C.c_void_p]
            getattr(L, f).restype = C.c_long
        L.por_n_tot.argtypes = [C.c_void_p]
        L.por_n_tot.restype = C.c_int
        L.por_K.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.por_K.restype = C.c_int
        L.por_moment_offset.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.por_moment_offset.restype = C.c_long
        for f in ("por_nodes", "por_weights"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_int]
            getattr(L, f).restype = dp
        for f in ("por_phi", "por_coef"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_int, C.c_int]
            getattr(L, f).restype = dp
        L.por_alpha_gen.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_uint64,
                                    C.c_int64, C.c_int64, dp]
        L.por_uniform.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int]
        L.por_uniform.restype = C.c_double
        L.por_moments.argtypes = [C.c_void_p, dp, C.c_int64, dp, C.c_int]
        for f in ("por_contract", "por_fill", "por_direct"):
            getattr(L, f).argtypes = [C.c_void_p, dp, C.c_int64, dp, C.c_int64, C.c_int]
        L.por_direct_sample.argtypes = [C.c_void_p, dp, C.c_int, C.c_int, dp, C.c_int64, C.POINTER(C.c_long)]
        L.por_direct_sample.restype = C.c_long
        L.por_block_close.argtypes = [dp, C.c_int64, dp, C.c_int64, C.c_int, C.c_int, C.c_double,
                                      ip, ip]
        L.por_block_close.restype = C.c_int
        L.por_cheb_eval.argtypes = [C.c_int, C.c_int, C.c_double]
        L.por_cheb_eval.restype = C.c_double
        L.por_cheb_p2s.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp, ip, ip]
        L.por_cheb_p2s.restype = C.c_int
        L.por_cheb2d_element.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp, dp, dp, dp, dp, dp, dp]
        _libs[fast] = L
    return _libs[fast]


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---------------------------------------------------------------- 1-D pieces

def gauss_legendre(n: int):
    x = np.zeros(n)
    w = np.zeros(n)
    lib().por_gauss_legendre(n, _dp(x), _dp(w))
    return x, w


def legendre_eval(K: int, x: float):
    P = np.zeros(K)
    dP = np.zeros(K)
    lib().por_legendre_eval(K, float(x), _dp(P), _dp(dP))
    return P, dP


def kernel_count(kind: int, N: int) -> int:
    return lib().por_kernel_count(kind, N)


def legendre_coef(kind: int, N: int) -> np.ndarray:
    K = kernel_count(kind, N)
    Cc = np.zeros((N, N, K))
    lib().por_legendre_coef(kind, N, K, _dp(Cc))
    return Cc


def cheb_eval(fam: int, n: int, u: float) -> float:
    return lib().por_cheb_eval(fam, n, float(u))


def cheb_p2s(fa: int, a: int, fb: int, b: int):
    coeff = (C.c_double * 2)()
    fam = (C.c_int * 2)()
    deg = (C.c_int * 2)()
    n = lib().por_cheb_p2s(fa, a, fb, b, coeff, fam, deg)
    return [(coeff[i], fam[i], deg[i]) for i in range(n)]


def block_close(a: np.ndarray, b: np.ndarray, rtol: float = 1e-12):
    """verify.cpp:81-99 semantics; returns (ok, (i, j) of first failure)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape and a.ndim == 2
    bi = C.c_int(-1)
    bj = C.c_int(-1)
    ok = lib().por_block_close(_dp(a), a.shape[1], _dp(b), b.shape[1], a.shape[0], a.shape[1],
                               rtol, C.byref(bi), C.byref(bj))
    return bool(ok), (bi.value, bj.value)


def cheb2d_element(M: int, N: int, nq: int, nodes, ws, wuu, wuv, wvv):
    """Reference 2-D element on the generic engine.  Returns (tables, p2s, direct)
    as dicts of named blocks."""
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    grids = [np.ascontiguousarray(g, dtype=np.float64).reshape(nq, nq) for g in (ws, wuu, wuv, wvv)]
    neu, nev = M * (N + 1), (M + 1) * N
    tsz = [(2 * M + 1, 2 * N + 1), (2 * M + 1, 2 * N + 1), (2 * M, 2 * N), (2 * M + 1, 2 * N + 1)]
    tables = np.zeros(sum(a * b for a, b in tsz))
    bsz = [(neu, neu), (neu, nev), (nev, neu), (nev, nev)] * 2
    nb = sum(a * b for a, b in bsz)
    p2s = np.zeros(nb)
    direct = np.zeros(nb)
    lib().por_cheb2d_element(M, N, nq, _dp(nodes), *[_dp(g) for g in grids], _dp(tables),
                             _dp(p2s), _dp(direct))
    tnames = ["Ks", "Kuu", "Kuv", "Kvv"]
    bnames = ["Suu", "Suv", "Svu", "Svv", "Muu", "Muv", "Mvu", "Mvv"]
    out_t, off = {}, 0
    for name, (r, c) in zip(tnames, tsz):
        out_t[name] = tables[off:off + r * c].reshape(r, c)
        off += r * c
    out_p, out_d, off = {}, {}, 0
    for name, (r, c) in zip(bnames, bsz):
        out_p[name] = p2s[off:off + r * c].reshape(r, c)
        out_d[name] = direct[off:off + r * c].reshape(r, c)
        off += r * c
    return out_t, out_p, out_d


# ---------------------------------------------------------------- 3-D problem

def conforming_matrix(n):
    """R (n x n) of the reference's conforming_matrix(n-1) (assembly.cpp:476-489):
    column m = modal coefficients of the conforming basis function phi_m."""
    R = np.zeros(n * n)
    lib().por_conforming_matrix(n, _dp(R))
    return R.reshape(n, n)


class Oracle:
    """3-D Legendre p2s problem on the CPU oracle."""

    def __init__(self, n_comp, order, kinds, nq, basis=0, fast=False):
        self._L = lib(fast)
        pb = Problem()
        pb.basis = basis
        pb.n_comp = n_comp
        for d in range(3):
            pb.order[d] = order[d]
            pb.nq[d] = nq[d]
        pb.n_terms = len(kinds)
        for s, k in enumerate(kinds):
            kk = k if isinstance(k, (tuple, list)) else (k, k, k)
            for d in range(3):
                pb.kind[s][d] = kk[d]
        self.problem = pb
        self.n_comp = n_comp
        self.order = tuple(order)
        self.kinds = [tuple(k) if isinstance(k, (tuple, list)) else (k, k, k) for k in kinds]
        self.nq = tuple(nq)
        self.h = self._L.por_create(C.byref(pb))
        if not self.h:
            raise ValueError("oracle: invalid problem")
        L = self._L
        self.alpha_per_elem = L.por_alpha_per_elem(self.h)
        self.moments_per_elem = L.por_moments_per_elem(self.h)
        self.n_tot = L.por_n_tot(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self._L.por_destroy(self.h)
            self.h = None

    def K(self, term, d):
        return self._L.por_K(self.h, term, d)

    def moment_offset(self, pair, term):
        return self._L.por_moment_offset(self.h, pair, term)

    def nodes(self, d):
        return np.ctypeslib.as_array(self._L.por_nodes(self.h, d), shape=(self.nq[d],)).copy()

    def weights(self, d):
        return np.ctypeslib.as_array(self._L.por_weights(self.h, d), shape=(self.nq[d],)).copy()

    def phi(self, term, d):
        K = self.K(term, d)
        return np.ctypeslib.as_array(self._L.por_phi(self.h, term, d), shape=(K, self.nq[d])).copy()

    def coef(self, term, d):
        K, N = self.K(term, d), self.order[d]
        return np.ctypeslib.as_array(self._L.por_coef(self.h, term, d), shape=(N, N, K)).copy()

    def alpha(self, kind, lo, hi, seed, e0, n):
        a = np.zeros(n * self.alpha_per_elem)
        self._L.por_alpha_gen(self.h, kind, lo, hi, seed, e0, n, _dp(a))
        return a.reshape(n, self.alpha_per_elem)

    def moments(self, alpha, threads=1):
        alpha = np.ascontiguousarray(alpha, dtype=np.float64)
        n = alpha.size // self.alpha_per_elem
        out = np.zeros((n, self.moments_per_elem))
        self._L.por_moments(self.h, _dp(alpha), n, _dp(out), threads)
        return out

    def contract(self, I, threads=1):
        I = np.ascontiguousarray(I, dtype=np.float64)
        n = I.size // self.moments_per_elem
        out = np.zeros((n, self.n_tot, self.n_tot))
        self._L.por_contract(self.h, _dp(I), n, _dp(out), self.n_tot, threads)
        return out

    def fill(self, alpha, threads=1, out=None):
        alpha = np.ascontiguousarray(alpha, dtype=np.float64)
        n = alpha.size // self.alpha_per_elem
        if out is None:
            out = np.zeros((n, self.n_tot, self.n_tot))
        self._L.por_fill(self.h, _dp(alpha), n, _dp(out), self.n_tot, threads)
        return out

    def direct(self, alpha, threads=1):
        alpha = np.ascontiguousarray(alpha, dtype=np.float64)
        n = alpha.size // self.alpha_per_elem
        out = np.zeros((n, self.n_tot, self.n_tot))
        self._L.por_direct(self.h, _dp(alpha), n, _dp(out), self.n_tot, threads)
        return out


def direct_sample_seconds(orc, alpha_elem, m1_lo, m1_hi):
    """Time one element's direct fill restricted to u-test indices m1 in
    [m1_lo, m1_hi) (single thread); returns (seconds, covered pairs, all pairs)."""
    import time
    a = np.ascontiguousarray(alpha_elem, dtype=np.float64).reshape(-1)
    M = np.zeros((orc.n_tot, orc.n_tot))
    tot = C.c_long(0)
    t0 = time.perf_counter()
    cov = orc._L.por_direct_sample(orc.h, _dp(a), m1_lo, m1_hi, _dp(M), orc.n_tot, C.byref(tot))
    return time.perf_counter() - t0, cov, tot.value


def uniform(seed, elem, slot, j):
    return lib().por_uniform(seed, elem, slot, j)
