"""ctypes binding of the C-ABI in include/p2s_b200.h (libp2s_b200.so).

The product path: every compute call below launches the sm_100a kernels of
libp2s_b200.so.  There is no CPU fallback -- if the library is missing this
module raises at import of the library, and on a machine without a B200 the
context constructor raises P2SError(P2S_CUDA_ERROR).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libp2s_b200.so")

MAX_TERMS = 4
PP, DD, DP, PD = 0, 1, 2, 3
ALPHA_SINE, ALPHA_JACOBIAN, ALPHA_EXPSIN = 0, 1, 2

OK, INVALID_ARG, CUDA_ERROR, UNSUPPORTED_SHAPE, GEOMETRY_ERROR = 0, 1, 2, 3, 4
_STATUS = {0: "P2S_OK", 1: "P2S_INVALID_ARG", 2: "P2S_CUDA_ERROR", 3: "P2S_UNSUPPORTED_SHAPE",
           4: "P2S_GEOMETRY_ERROR"}

# every symbol include/p2s_b200.h declares
EXPORTS = ("p2s_create", "p2s_destroy", "p2s_get_sizes", "p2s_moments", "p2s_contract",
           "p2s_fill", "p2s_fill_host", "p2s_alpha_generate", "p2s_get_tables",
           "p2s_set_profiling", "p2s_get_stage_times", "p2s_shape_supported", "p2s_last_error",
           "p2s_version", "p2s_kernel_path", "p2s_moments_host", "p2s_contract_host",
           "p2s_cheb2d_create", "p2s_cheb2d_destroy", "p2s_cheb2d_get_sizes",
           "p2s_cheb2d_kernel_tables", "p2s_cheb2d_assemble",
           "p2s_direct_create", "p2s_direct_destroy", "p2s_direct_fill",
           "p2s_scatter_add", "p2s_cheb2d_scatter",
           "p2s_geometry_generate", "p2s_alpha_from_geometry", "p2s_fill_geometry",
           "p2s_create_ex", "p2s_shape_prepare", "p2s_jit_cache_dir", "p2s_problem_sizes",
           "p2s_scatter_plan_create", "p2s_scatter_plan_destroy", "p2s_scatter_add_ordered",
           "p2s_cheb2d_scatter_ordered")


class P2SError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class InvalidArgument(P2SError, ValueError):
    """std::invalid_argument in the reference (assembly.cpp:20, 376-378)."""


class UnsupportedShape(P2SError):
    pass


class GeometryError(P2SError):
    """GeometryError in the reference: non-positive Jacobian (assembly.cpp:95-99)."""


class Problem(C.Structure):
    _fields_ = [
        ("n_comp", C.c_int32),
        ("order", C.c_int32 * 3),
        ("n_terms", C.c_int32),
        ("kind", (C.c_int32 * 3) * MAX_TERMS),
        ("nq", C.c_int32 * 3),
        ("basis", C.c_int32),
    ]


BASIS_MODAL, BASIS_CONFORMING = 0, 1


class Cheb2dProblem(C.Structure):
    _fields_ = [("M", C.c_int32), ("N", C.c_int32), ("nq", C.c_int32), ("conforming", C.c_int32)]


class Cheb2dSizes(C.Structure):
    _fields_ = [
        ("grids_per_elem", C.c_int64), ("tables_per_elem", C.c_int64),
        ("blocks_per_elem", C.c_int64), ("table_offset", C.c_int64 * 4),
        ("block_offset", C.c_int64 * 8), ("table_rows", C.c_int32 * 4),
        ("table_cols", C.c_int32 * 4), ("block_rows", C.c_int32 * 8),
        ("block_cols", C.c_int32 * 8), ("n_eu", C.c_int32), ("n_ev", C.c_int32),
    ]


class Sizes(C.Structure):
    _fields_ = [
        ("alpha_per_elem", C.c_int64),
        ("moments_per_elem", C.c_int64),
        ("moments_per_pair", C.c_int64),
        ("moment_offset", C.c_int64 * MAX_TERMS),
        ("n_tot", C.c_int32),
        ("n_pairs", C.c_int32),
        ("K", (C.c_int32 * 3) * MAX_TERMS),
    ]


def build(force: bool = False) -> str:
    """Compile libp2s_b200.so (nvcc, sm_100a) in-tree."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-C", os.path.join(_HERE, "csrc"), "-s"], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the fill has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i64, dp = C.c_void_p, C.c_int64, C.POINTER(C.c_double)
        L.p2s_create.argtypes = [C.POINTER(Problem), C.c_int, C.POINTER(vp)]
        L.p2s_create_ex.argtypes = [C.POINTER(Problem), C.c_int, C.c_char_p, C.POINTER(vp)]
        L.p2s_shape_prepare.argtypes = [C.POINTER(Problem), C.c_char_p, C.c_char_p, C.c_int]
        L.p2s_jit_cache_dir.restype = C.c_char_p
        L.p2s_destroy.argtypes = [vp]
        L.p2s_destroy.restype = None
        L.p2s_get_sizes.argtypes = [vp, C.POINTER(Sizes)]
        L.p2s_problem_sizes.argtypes = [C.POINTER(Problem), C.POINTER(Sizes)]
        L.p2s_moments.argtypes = [vp, vp, vp, i64, vp]
        L.p2s_contract.argtypes = [vp, vp, vp, i64, i64, vp]
        L.p2s_fill.argtypes = [vp, vp, vp, i64, i64, vp]
        L.p2s_fill_host.argtypes = [vp, vp, vp, i64, i64]
        L.p2s_moments_host.argtypes = [vp, vp, vp, i64]
        L.p2s_contract_host.argtypes = [vp, vp, vp, i64, i64]
        L.p2s_alpha_generate.argtypes = [vp, C.c_int, C.c_double, C.c_double, C.c_uint64, i64, i64,
                                         vp, vp]
        L.p2s_get_tables.argtypes = [vp, C.c_int, C.c_int, dp, dp, dp, dp]
        L.p2s_set_profiling.argtypes = [vp, C.c_int]
        L.p2s_get_stage_times.argtypes = [vp, dp, dp, C.POINTER(i64), C.POINTER(i64)]
        L.p2s_shape_supported.argtypes = [C.POINTER(Problem)]
        L.p2s_shape_supported.restype = C.c_int
        L.p2s_last_error.restype = C.c_char_p
        L.p2s_version.restype = C.c_char_p
        L.p2s_kernel_path.argtypes = [vp]
        L.p2s_kernel_path.restype = C.c_char_p
        L.p2s_cheb2d_create.argtypes = [C.POINTER(Cheb2dProblem), C.c_int, C.POINTER(vp)]
        L.p2s_cheb2d_destroy.argtypes = [vp]
        L.p2s_cheb2d_destroy.restype = None
        L.p2s_cheb2d_get_sizes.argtypes = [vp, C.POINTER(Cheb2dSizes)]
        L.p2s_cheb2d_kernel_tables.argtypes = [vp, vp, vp, i64, vp]
        L.p2s_cheb2d_assemble.argtypes = [vp, vp, vp, i64, vp]
        L.p2s_direct_create.argtypes = [C.POINTER(Problem), C.c_int, C.POINTER(vp)]
        L.p2s_direct_destroy.argtypes = [vp]
        L.p2s_direct_destroy.restype = None
        L.p2s_direct_fill.argtypes = [vp, vp, vp, i64, i64, vp]
        L.p2s_geometry_generate.argtypes = [vp, C.c_double, C.c_double, C.c_uint64, i64, i64, vp, vp]
        L.p2s_alpha_from_geometry.argtypes = [vp, vp, i64, vp, vp]
        L.p2s_fill_geometry.argtypes = [vp, vp, vp, i64, i64, vp]
        L.p2s_scatter_add.argtypes = [vp, i64, i64, C.c_int32, vp, vp, i64, vp, i64, vp]
        L.p2s_cheb2d_scatter.argtypes = [vp, vp, vp, vp, i64, vp, vp, i64, vp]
        L.p2s_scatter_plan_create.argtypes = [vp, i64, C.c_int32, C.c_int32, C.c_int, C.POINTER(vp)]
        L.p2s_scatter_plan_destroy.argtypes = [vp]
        L.p2s_scatter_plan_destroy.restype = None
        L.p2s_scatter_add_ordered.argtypes = [vp, vp, i64, i64, vp, vp, vp, i64, vp]
        L.p2s_cheb2d_scatter_ordered.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, vp]
        for f in EXPORTS:
            if f not in ("p2s_destroy", "p2s_shape_supported", "p2s_last_error", "p2s_version",
                         "p2s_jit_cache_dir", "p2s_scatter_plan_destroy",
                         "p2s_kernel_path", "p2s_cheb2d_destroy", "p2s_direct_destroy"):
                getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _check(status: int):
    if status != OK:
        msg = lib().p2s_last_error().decode()
        if status == INVALID_ARG:
            raise InvalidArgument(status, msg)
        if status == UNSUPPORTED_SHAPE:
            raise UnsupportedShape(status, msg)
        if status == GEOMETRY_ERROR:
            raise GeometryError(status, msg)
        raise P2SError(status, msg)


def make_problem(n_comp, order, kinds, nq, basis=BASIS_MODAL) -> Problem:
    if not 1 <= len(kinds) <= MAX_TERMS:  # the C struct holds MAX_TERMS terms
        raise InvalidArgument(INVALID_ARG, f"n_terms must be 1..{MAX_TERMS}")
    pb = Problem()
    pb.basis = basis
    pb.n_comp = n_comp
    for d in range(3):
        pb.order[d] = order[d]
        pb.nq[d] = nq[d]
    pb.n_terms = len(kinds)
    for s, k in enumerate(kinds):
        kk = tuple(k) if isinstance(k, (tuple, list)) else (k, k, k)
        for d in range(3):
            pb.kind[s][d] = kk[d]
    return pb


def shape_supported(n_comp, order, kinds, nq) -> bool:
    return bool(lib().p2s_shape_supported(C.byref(make_problem(n_comp, order, kinds, nq))))


def shape_supported_basis(n_comp, order, kinds, nq, basis) -> bool:
    return bool(lib().p2s_shape_supported(C.byref(make_problem(n_comp, order, kinds, nq, basis))))


def shape_prepare(n_comp, order, kinds, nq, basis=BASIS_MODAL, options: dict | None = None) -> str:
    """Build (or find) the generated kernel module of a shape without a device
    (p2s_shape_prepare); returns the plan and module path."""
    buf = C.create_string_buffer(1024)
    _check(lib().p2s_shape_prepare(C.byref(make_problem(n_comp, order, kinds, nq, basis)),
                                   options_string(options), buf, 1024))
    return buf.value.decode()


# Test / tuning hooks (p2s_create_ex options) applied to every Context created
# without explicit options -- the tests set them with monkeypatch.setitem; the
# library itself never reads the environment.
DEFAULT_OPTIONS: dict = {}


def problem_sizes(n_comp, order, kinds, nq, basis=BASIS_MODAL) -> Sizes:
    """p2s_problem_sizes: buffer sizes without a context or device."""
    sz = Sizes()
    _check(lib().p2s_problem_sizes(C.byref(make_problem(n_comp, order, kinds, nq, basis)), C.byref(sz)))
    return sz


def jit_cache_dir() -> str:
    """Directory of the generated kernel modules of this library build."""
    return lib().p2s_jit_cache_dir().decode()


def options_string(options) -> bytes | None:
    """{"P2S_NO_FUSED": "1", ...} -> b"P2S_NO_FUSED=1;..." (p2s_create_ex test/tuning hooks)."""
    if not options:
        return None
    return ";".join(f"{k}={v}" for k, v in options.items()).encode()


def _ptr(t) -> int:
    """Raw pointer of a torch tensor / int."""
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    if hasattr(t, "ctypes"):
        return t.ctypes.data
    raise TypeError(type(t))


class Context:
    """One p2s_ctx (tables uploaded once) on one device."""

    def __init__(self, n_comp, order, kinds, nq, device: int = 0, basis: int = BASIS_MODAL,
                 options: dict | None = None):
        self.problem = make_problem(n_comp, order, kinds, nq, basis)
        self.n_comp = n_comp
        self.order = tuple(order)
        self.kinds = [tuple(k) if isinstance(k, (tuple, list)) else (k, k, k) for k in kinds]
        self.nq = tuple(nq)
        self.device = device
        h = C.c_void_p()
        opts = dict(DEFAULT_OPTIONS)
        opts.update(options or {})
        _check(lib().p2s_create_ex(C.byref(self.problem), device, options_string(opts), C.byref(h)))
        self.h = h
        sz = Sizes()
        _check(lib().p2s_get_sizes(self.h, C.byref(sz)))
        self.sizes = sz
        self.alpha_per_elem = sz.alpha_per_elem
        self.moments_per_elem = sz.moments_per_elem
        self.moments_per_pair = sz.moments_per_pair
        self.n_tot = sz.n_tot
        self.n_pairs = sz.n_pairs

    def close(self):
        if getattr(self, "h", None):
            lib().p2s_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def K(self, term, d):
        return self.sizes.K[term][d]

    def moment_offset(self, pair, term):
        return pair * self.moments_per_pair + self.sizes.moment_offset[term]

    # ---- stages (device pointers; stream = raw cudaStream_t or 0)
    def moments(self, d_alpha, d_I, n_elem, stream=0):
        _check(lib().p2s_moments(self.h, _ptr(d_alpha), _ptr(d_I), n_elem, _ptr(stream)))

    def contract(self, d_I, d_M, ld_M, n_elem, stream=0):
        _check(lib().p2s_contract(self.h, _ptr(d_I), _ptr(d_M), ld_M, n_elem, _ptr(stream)))

    def fill(self, d_alpha, d_M, ld_M, n_elem, stream=0):
        _check(lib().p2s_fill(self.h, _ptr(d_alpha), _ptr(d_M), ld_M, n_elem, _ptr(stream)))

    GEOM_DOUBLES = 28

    def geometry_generate(self, lo, hi, seed, e0, n_elem, d_geom, stream=0):
        _check(lib().p2s_geometry_generate(self.h, lo, hi, seed, e0, n_elem, _ptr(d_geom), _ptr(stream)))

    def alpha_from_geometry(self, d_geom, n_elem, d_alpha, stream=0):
        _check(lib().p2s_alpha_from_geometry(self.h, _ptr(d_geom), n_elem, _ptr(d_alpha), _ptr(stream)))

    def fill_geometry(self, d_geom, d_M, ld_M, n_elem, stream=0):
        _check(lib().p2s_fill_geometry(self.h, _ptr(d_geom), _ptr(d_M), ld_M, n_elem, _ptr(stream)))

    def fill_host(self, h_alpha, h_M, ld_M, n_elem):
        _check(lib().p2s_fill_host(self.h, _ptr(h_alpha), _ptr(h_M), ld_M, n_elem))

    def moments_host(self, h_alpha, h_I, n_elem):
        _check(lib().p2s_moments_host(self.h, _ptr(h_alpha), _ptr(h_I), n_elem))

    def contract_host(self, h_I, h_M, ld_M, n_elem):
        _check(lib().p2s_contract_host(self.h, _ptr(h_I), _ptr(h_M), ld_M, n_elem))

    def alpha_generate(self, kind, lo, hi, seed, e0, n_elem, d_alpha, stream=0):
        _check(lib().p2s_alpha_generate(self.h, kind, lo, hi, seed, e0, n_elem, _ptr(d_alpha),
                                        _ptr(stream)))

    def tables(self, term, d):
        import numpy as np
        K, nq, N = self.K(term, d), self.nq[d], self.order[d]
        phi = np.zeros((K, nq))
        coef = np.zeros((N, N, K))
        x = np.zeros(nq)
        w = np.zeros(nq)
        dp = C.POINTER(C.c_double)
        _check(lib().p2s_get_tables(self.h, term, d, phi.ctypes.data_as(dp), coef.ctypes.data_as(dp),
                                    x.ctypes.data_as(dp), w.ctypes.data_as(dp)))
        return phi, coef, x, w

    @property
    def kernel_path(self) -> str:
        return lib().p2s_kernel_path(self.h).decode()

    def set_profiling(self, enable: bool):
        _check(lib().p2s_set_profiling(self.h, int(enable)))

    def stage_times(self):
        a, b = C.c_double(), C.c_double()
        na, nb = C.c_int64(), C.c_int64()
        _check(lib().p2s_get_stage_times(self.h, C.byref(a), C.byref(b), C.byref(na), C.byref(nb)))
        return {"ms_moments": a.value, "ms_contract": b.value, "n_moments": na.value,
                "n_contract": nb.value}


TABLE_NAMES = ("Ks", "Kuu", "Kuv", "Kvv")
BLOCK_NAMES = ("Suu", "Suv", "Svu", "Svv", "Muu", "Muv", "Mvu", "Mvv")


class Cheb2dContext:
    """The reference's 2-D Chebyshev element (chebfem) on the GPU:
    kernel_tables() ~ compute_kernel_tables, assemble() ~ assemble_p2s_element."""

    def __init__(self, M, N, nq, device: int = 0, conforming: bool = False):
        self.M, self.N, self.nq = M, N, nq
        pb = Cheb2dProblem(M, N, nq, 1 if conforming else 0)
        h = C.c_void_p()
        _check(lib().p2s_cheb2d_create(C.byref(pb), device, C.byref(h)))
        self.h = h
        sz = Cheb2dSizes()
        _check(lib().p2s_cheb2d_get_sizes(self.h, C.byref(sz)))
        self.sizes = sz

    def close(self):
        if getattr(self, "h", None):
            lib().p2s_cheb2d_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def kernel_tables(self, d_grids, d_tables, n_elem, stream=0):
        _check(lib().p2s_cheb2d_kernel_tables(self.h, _ptr(d_grids), _ptr(d_tables), n_elem,
                                              _ptr(stream)))

    def assemble(self, d_tables, d_blocks, n_elem, stream=0):
        _check(lib().p2s_cheb2d_assemble(self.h, _ptr(d_tables), _ptr(d_blocks), n_elem,
                                         _ptr(stream)))

    def scatter_ordered(self, plan, d_blocks, d_dof_free, d_dof_sign, d_S, d_M, ld_G, stream=0):
        """p2s_cheb2d_scatter_ordered: the reference's summation order, bit for bit."""
        _check(lib().p2s_cheb2d_scatter_ordered(self.h, plan.h, _ptr(d_blocks), _ptr(d_dof_free),
                                                _ptr(d_dof_sign), _ptr(d_S), _ptr(d_M), ld_G, _ptr(stream)))

    def scatter(self, d_blocks, d_dof_free, d_dof_sign, n_elem, d_S, d_M, ld_G, stream=0):
        """assemble_global (assembly.cpp:594-652) from the eight blocks, on the device."""
        _check(lib().p2s_cheb2d_scatter(self.h, _ptr(d_blocks), _ptr(d_dof_free), _ptr(d_dof_sign),
                                        n_elem, _ptr(d_S), _ptr(d_M), ld_G, _ptr(stream)))

    def split_tables(self, flat):
        sz = self.sizes
        return {n: flat[sz.table_offset[i]:sz.table_offset[i] + sz.table_rows[i] * sz.table_cols[i]]
                .reshape(sz.table_rows[i], sz.table_cols[i]) for i, n in enumerate(TABLE_NAMES)}

    def split_blocks(self, flat):
        sz = self.sizes
        return {n: flat[sz.block_offset[i]:sz.block_offset[i] + sz.block_rows[i] * sz.block_cols[i]]
                .reshape(sz.block_rows[i], sz.block_cols[i]) for i, n in enumerate(BLOCK_NAMES)}


class DirectContext:
    """Direct-quadrature fill (p2s_direct_*): the ablation baseline, reference
    assemble_direct_element (assembly.hpp:50; assembly.cpp:134-274) in 3-D."""

    def __init__(self, n_comp, order, kinds, nq, device: int = 0, basis: int = BASIS_MODAL,
                 options: dict | None = None):
        self.problem = make_problem(n_comp, order, kinds, nq, basis)
        self.n_tot = n_comp * order[0] * order[1] * order[2]
        h = C.c_void_p()
        _check(lib().p2s_direct_create(C.byref(self.problem), device, C.byref(h)))
        self._h = h

    def fill(self, d_alpha, d_M, ld_M: int, n_elem: int, stream=0):
        _check(lib().p2s_direct_fill(self._h, _ptr(d_alpha), _ptr(d_M), ld_M, n_elem, _ptr(stream)))

    def close(self):
        if getattr(self, "_h", None):
            lib().p2s_direct_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def scatter_add(d_elem, elem_stride, ld_elem, n_local, d_dof_free, d_dof_sign, n_elem, d_G, ld_G,
                stream=0):
    """Global scatter-add G[gi][gj] += s_i s_j E[i][j] (reference assemble_global,
    assembly.cpp:594-652) on the device."""
    _check(lib().p2s_scatter_add(_ptr(d_elem), elem_stride, ld_elem, n_local, _ptr(d_dof_free),
                                 _ptr(d_dof_sign), n_elem, _ptr(d_G), ld_G, _ptr(stream)))


class ScatterPlan:
    """p2s_scatter_plan: per global row, the (element, local row) contributions in
    the reference's order (assemble_global, assembly.cpp:626-641), from the host
    free-index map dof_free[n_elem][n_local] (numpy int32)."""

    def __init__(self, dof_free, n_free: int, device: int = 0):
        import numpy as np
        f = np.ascontiguousarray(dof_free, dtype=np.int32)
        self.n_elem, self.n_local = f.shape
        self.n_free = n_free
        h = C.c_void_p()
        _check(lib().p2s_scatter_plan_create(f.ctypes.data, self.n_elem, self.n_local, n_free, device, C.byref(h)))
        self.h = h

    def add(self, d_elem, elem_stride, ld_elem, d_dof_free, d_dof_sign, d_G, ld_G, stream=0):
        _check(lib().p2s_scatter_add_ordered(self.h, _ptr(d_elem), elem_stride, ld_elem, _ptr(d_dof_free),
                                             _ptr(d_dof_sign), _ptr(d_G), ld_G, _ptr(stream)))

    def close(self):
        if getattr(self, "h", None):
            lib().p2s_scatter_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
