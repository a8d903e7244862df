"""Legendre product-to-sum bands (mirror of csrc/p2s_tables.hpp band_lo/hi)."""
from .capi import DD, DP, PP


def band_lo(kind, a, b):
    if kind == PP:
        return abs(a - b)
    if kind == DD:
        return (a + b) % 2
    if kind == DP:
        return b - a + 1 if b >= a else (a + b - 1) % 2
    return a - b + 1 if a >= b else (a + b - 1) % 2


def band_hi(kind, a, b):
    if kind == PP:
        return a + b
    if kind == DD:
        return a + b - 2 if (a >= 1 and b >= 1) else -1
    if kind == DP:
        return a + b - 1 if a >= 1 else -1
    return a + b - 1 if b >= 1 else -1


def band_count(kind, a, b):
    lo, hi = band_lo(kind, a, b), band_hi(kind, a, b)
    return (hi - lo) // 2 + 1 if hi >= lo else 0
