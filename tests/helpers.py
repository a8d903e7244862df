"""Shared helpers for the parity tests (GPU path vs CPU oracle)."""
import numpy as np

from oracle import oracle as O

RTOL = 1e-12   # north_star: <= 1e-12 relative, reference comparator semantics (verify.cpp:81-99)


def blocks_close(M_gpu, M_ref, n_comp, Nt, rtol=RTOL):
    """Compare one element matrix per (gi, gj) pair block with block_close.
    Returns (ok, message, worst_rel_to_block_max)."""
    worst = 0.0
    for gi in range(n_comp):
        for gj in range(n_comp):
            a = np.ascontiguousarray(M_gpu[gi * Nt:(gi + 1) * Nt, gj * Nt:(gj + 1) * Nt])
            b = np.ascontiguousarray(M_ref[gi * Nt:(gi + 1) * Nt, gj * Nt:(gj + 1) * Nt])
            scale = max(np.abs(a).max(), np.abs(b).max(), 1e-300)
            worst = max(worst, float(np.abs(a - b).max() / scale))
            ok, (i, j) = O.block_close(a, b, rtol)
            if not ok:
                return False, f"block ({gi},{gj}) entry ({i},{j}): {a[i, j]!r} vs {b[i, j]!r}", worst
    return True, "", worst


def oracle_for(n_comp, order, kinds, nq, basis=0):
    return O.Oracle(n_comp, order, kinds, nq, basis)
