"""The drop-in coverage grid: problem shapes the reference's fill accepts
(any Orders / kinds / nq: assembly.hpp:52-56, 82-83; Table I sweeps
M = N = 3..18) beyond the five BASELINE configs.

  ISOTROPIC   N = 1..18, scalar, mass + P'P' terms, nq = N + 7 (the reference's
              default_quad_points policy max(M, N) + geometric order + 6,
              assembly.cpp:23-25, with a trilinear map)
  RANDOM      seeded anisotropic shapes: orders 1..18 per direction, 1-4 terms
              with per-direction PP / DD / DP / PD kinds, 1-3 components, modal
              or conforming basis, nq from under- to over-integration; the
              matrix dimension is capped so the CPU oracle checks 2 elements in
              seconds
  BENCH       (12, 12, 12), the mid-order bench line (bench.py --config c12)

build() (__graft_entry__) prepares the generated module of every shape ahead of
time; tests/test_gpu_shapes.py checks each against the CPU oracle at 1e-12.
"""
from __future__ import annotations

import random

PP, DD, DP, PD = 0, 1, 2, 3
MODAL, CONFORMING = 0, 1


def _iso(n):
    return (1, (n, n, n), [PP, DD], (n + 7,) * 3, MODAL)


ISOTROPIC = [_iso(n) for n in range(1, 19)]


def _random_shapes(count=24, seed=1703, max_ntot=2200):
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        nc = rng.choice([1, 1, 2, 3])
        order = tuple(rng.randint(1, 18) for _ in range(3))
        if nc * order[0] * order[1] * order[2] > max_ntot:
            continue
        S = rng.randint(1, 4)
        kinds = [tuple(rng.choice([PP, DD, DP, PD]) for _ in range(3)) for _ in range(S)]
        nq = tuple(max(1, min(64, n + rng.randint(-2, 8))) for n in order)
        basis = CONFORMING if min(order) >= 2 and rng.random() < 0.3 else MODAL
        out.append((nc, order, kinds, nq, basis))
    return out


RANDOM = _random_shapes()

BENCH = [(1, (12, 12, 12), [PP, DD], (18, 18, 18), MODAL)]

ALL = ISOTROPIC + RANDOM + BENCH


def shape_id(case) -> str:
    nc, order, kinds, nq, basis = case
    def kc(k):
        return "PDLR"[k] if 0 <= k < 4 else f"[{k}]"

    ks = "".join(kc(k) if isinstance(k, int) else "".join(kc(x) for x in k) for k in kinds)
    return f"{nc}c-{order[0]}x{order[1]}x{order[2]}-{ks}-q{nq[0]}x{nq[1]}x{nq[2]}" + ("-conf" if basis else "")


def prepare_all(cases=None, workers: int = 0):
    """Build the generated module of every grid shape (p2s_shape_prepare, no
    device needed), in parallel; returns {shape_id: plan | error}."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    from . import capi
    cases = ALL if cases is None else cases
    workers = workers or min(16, os.cpu_count() or 1)

    def one(c):
        name = shape_id(c[:5]) + (f" {c[5]}" if len(c) > 5 else "")
        try:
            return name, capi.shape_prepare(*c)
        except Exception as e:  # reported, not raised: the GPU tests name the shape
            return name, f"ERROR {e}"

    with ThreadPoolExecutor(max_workers=workers) as ex:  # ctypes releases the GIL
        return dict(ex.map(one, cases))


def prune_cache():
    """Remove modules built from other versions of the kernel headers from the
    in-tree module cache (paper_1703_09619_b200/jit/<header hash>/)."""
    import os
    import shutil

    from . import capi
    root = os.path.join(os.path.dirname(capi.LIB_PATH), "jit")
    if not os.path.isdir(root):
        return
    current = capi.jit_cache_dir()
    for name in os.listdir(root):
        path = os.path.join(root, name)
        if path != current:
            shutil.rmtree(path, ignore_errors=True) if os.path.isdir(path) else os.remove(path)
