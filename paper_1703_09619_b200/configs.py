"""BASELINE.json configurations (C1..C5) as fill problems.

Each entry: component count, orders (N_u, N_v, N_w), term kinds, Gauss-Legendre
points per direction, element count, and the seeded coupling-factor family.
Decision (i) of SURVEY.md 8(d): the N_s=2 "derivative-product term using
P'.P' pairs" is P'P' in all three directions (term kinds are data, so the
alternative reading is a config change).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .capi import ALPHA_EXPSIN, ALPHA_JACOBIAN, ALPHA_SINE, DD, PP


@dataclass(frozen=True)
class FillConfig:
    name: str
    n_comp: int
    order: tuple
    kinds: tuple
    nq: tuple
    n_elem: int
    alpha_kind: int
    alpha_lo: float
    alpha_hi: float
    note: str = ""

    @property
    def n_tot(self) -> int:
        return self.n_comp * self.order[0] * self.order[1] * self.order[2]

    def problem(self):
        return dict(n_comp=self.n_comp, order=self.order, kinds=list(self.kinds), nq=self.nq)


CONFIGS = {
    "c1": FillConfig("c1", 1, (4, 4, 4), (PP,), (8, 8, 8), 1, ALPHA_SINE, 0.5, 3.0,
                     "single element, scalar, order 4, mass term, 8^3 GL"),
    "c2": FillConfig("c2", 3, (6, 6, 6), (PP, DD), (14, 14, 14), 4096, ALPHA_JACOBIAN, 0.5, 3.0,
                     "3-component, order 6, mass + P'P' term, 9 pairs, trilinear Jacobian, 14^3 GL"),
    "c3": FillConfig("c3", 1, (8, 8, 8), (PP, DD), (20, 20, 20), 65536, ALPHA_EXPSIN, 4.0, 10.0,
                     "scalar, order 8, exp(0.5 sin(f(u+v+w)))(1+0.2uvw), 20^3 GL"),
    "c4": FillConfig("c4", 3, (10, 6, 4), (PP, DD), (16, 16, 16), 262144, ALPHA_SINE, 0.5, 3.0,
                     "3-component, anisotropic (10,6,4), 16^3 GL"),
    "c5": FillConfig("c5", 1, (16, 16, 16), (PP, DD), (36, 36, 36), 32768, ALPHA_SINE, 0.5, 12.0,
                     "scalar, order 16, frequency up to 12, 36^3 GL"),
    # drop-in coverage bench line (no ahead-of-time kernel: generated module)
    "c12": FillConfig("c12", 1, (12, 12, 12), (PP, DD), (18, 18, 18), 8192, ALPHA_SINE, 0.5, 3.0,
                      "scalar, order 12 (PAPER.md Table I M=N=12), 18^3 GL, generated module"),
}


def algorithmic_counts(cfg: FillConfig):
    """Per-element algorithmic bytes / flops of SURVEY.md 8(d).

    Returns dict with bytes_mom, flop_mom, bytes_con, flop_con (per element)."""
    from .capi import PP as _PP, DD as _DD
    P = cfg.n_comp ** 2
    Nu, Nv, Nw = cfg.order
    nqu, nqv, nqw = cfg.nq

    def K(kind, N):
        k = 2 * N - 1 if kind == _PP else (2 * N - 3 if kind == _DD else 2 * N - 2)
        return max(1, k)

    def z(kind, N):
        # average nonzeros per (a, b) of the product-to-sum table
        from .bands import band_count
        return sum(band_count(kind, a, b) for a in range(N) for b in range(N)) / (N * N)

    flop_mom = bytes_i = flop_con = 0.0
    for kd in cfg.kinds:
        kk = kd if isinstance(kd, tuple) else (kd, kd, kd)
        Ku, Kv, Kw = K(kk[0], Nu), K(kk[1], Nv), K(kk[2], Nw)
        flop_mom += 2 * P * (nqu * nqv * nqw * Ku + Ku * nqv * nqw * Kv + Ku * Kv * nqw * Kw)
        bytes_i += 8 * P * Ku * Kv * Kw
        flop_con += 2 * P * (Ku * Kv * Nw * Nw * z(kk[2], Nw) + Ku * Nv * Nv * Nw * Nw * z(kk[1], Nv)
                             + Nu * Nu * Nv * Nv * Nw * Nw * z(kk[0], Nu))
    bytes_alpha = 8 * P * len(cfg.kinds) * nqu * nqv * nqw
    bytes_m = 8 * cfg.n_tot ** 2
    return {"bytes_mom": bytes_alpha + bytes_i, "flop_mom": flop_mom,
            "bytes_con": bytes_m + bytes_i, "flop_con": flop_con,
            "bytes_alpha": bytes_alpha, "bytes_I": bytes_i, "bytes_M": bytes_m}
