"""Reference-shaped host API over the C-ABI (device tensors via torch).

Mirrors the reference's fill interface (include/chebfem/assembly.hpp):

  compute_kernel_tables(ctx, alpha)      ~ compute_kernel_tables(mesh, e, orders, nq)
                                           (assembly.hpp:52), batched over elements
  assemble_p2s_element(ctx, tables)      ~ assemble_p2s_element(kernels, orders)
                                           (assembly.hpp:56); raises InvalidArgument when
                                           the tables were built for other orders
                                           (assembly.cpp:376-378)
  fill_elements(ctx, alpha)              ~ fill_elements(mesh, orders, Backend::p2s, nq)
                                           (assembly.hpp:82-83)

torch supplies device memory and streams only; all arithmetic runs in
libp2s_b200.so.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from .capi import Context, InvalidArgument


@dataclass
class KernelTables:
    """Moment integrals of a batch (reference: KernelTable, assembly.hpp:35-40)."""
    I: torch.Tensor          # [E, moments_per_elem] float64, device
    order: tuple
    kinds: list
    n_comp: int
    n_elem: int
    n_integrals: int         # moment entries computed (counter of assembly.hpp:38)


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _check_alpha(ctx: Context, alpha: torch.Tensor) -> int:
    if alpha.dtype != torch.float64 or not alpha.is_cuda or not alpha.is_contiguous():
        raise InvalidArgument(1, "alpha must be a contiguous float64 CUDA tensor")
    if alpha.numel() % ctx.alpha_per_elem:
        raise InvalidArgument(1, f"alpha size {alpha.numel()} is not a multiple of "
                                 f"{ctx.alpha_per_elem}")
    return alpha.numel() // ctx.alpha_per_elem


def compute_kernel_tables(ctx: Context, alpha: torch.Tensor) -> KernelTables:
    n = _check_alpha(ctx, alpha)
    I = torch.empty((n, ctx.moments_per_elem), dtype=torch.float64, device=alpha.device)
    ctx.moments(alpha, I, n, _stream())
    per = sum(ctx.K(s, 0) * ctx.K(s, 1) * ctx.K(s, 2) for s in range(len(ctx.kinds)))
    return KernelTables(I, ctx.order, ctx.kinds, ctx.n_comp, n, per * ctx.n_pairs * n)


def assemble_p2s_element(ctx: Context, tables: KernelTables, out: torch.Tensor | None = None,
                         ld: int | None = None) -> torch.Tensor:
    if (tables.order != ctx.order or tables.kinds != ctx.kinds or tables.n_comp != ctx.n_comp):
        raise InvalidArgument(1, "assemble_p2s_element: kernel table was built for other orders")
    n = tables.n_elem
    ld = ld or ctx.n_tot
    if out is None:
        out = torch.empty((n, ctx.n_tot, ld), dtype=torch.float64, device=tables.I.device)
    ctx.contract(tables.I, out, ld, n, _stream())
    return out


def fill_elements(ctx: Context, alpha: torch.Tensor, out: torch.Tensor | None = None,
                  ld: int | None = None) -> torch.Tensor:
    n = _check_alpha(ctx, alpha)
    ld = ld or ctx.n_tot
    if out is None:
        out = torch.empty((n, ctx.n_tot, ld), dtype=torch.float64, device=alpha.device)
    ctx.fill(alpha, out, ld, n, _stream())
    return out


def generate_alpha(ctx: Context, kind: int, lo: float, hi: float, seed: int, e0: int, n: int,
                   out: torch.Tensor | None = None) -> torch.Tensor:
    """Seeded synthetic coupling factor on the device (harness input)."""
    if out is None:
        out = torch.empty((n, ctx.alpha_per_elem), dtype=torch.float64,
                          device=torch.device("cuda", ctx.device))
    ctx.alpha_generate(kind, lo, hi, seed, e0, n, out, _stream())
    return out
