"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

Bar (north_star): <= 1e-12 relative error with the reference comparator
(verify.cpp:81-99: |a-b| <= 1e-12 max(|a|,|b|) or <= 1e-12 max|block|),
applied per (gi, gj) pair block, on byte-identical alpha.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1703_09619_b200 import capi
from paper_1703_09619_b200.capi import DD, DP, PD, PP
from paper_1703_09619_b200.configs import CONFIGS

from helpers import RTOL, blocks_close, oracle_for

pytestmark = pytest.mark.gpu


def _gpu_fill(ctx, alpha_np, ld=None):
    n = alpha_np.shape[0]
    ld = ld or ctx.n_tot
    a = torch.from_numpy(np.ascontiguousarray(alpha_np)).cuda()
    M = torch.full((n, ctx.n_tot, ld), float("nan"), dtype=torch.float64, device="cuda")
    ctx.fill(a, M, ld, n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return M.cpu().numpy()


def _gpu_moments(ctx, alpha_np):
    n = alpha_np.shape[0]
    a = torch.from_numpy(np.ascontiguousarray(alpha_np)).cuda()
    I = torch.zeros((n, ctx.moments_per_elem), dtype=torch.float64, device="cuda")
    ctx.moments(a, I, n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return I.cpu().numpy()


def _check_case(n_comp, order, kinds, nq, alpha_kind, lo, hi, n_elem, seed=11, threads=8):
    o = oracle_for(n_comp, order, kinds, nq)
    ctx = capi.Context(n_comp, order, kinds, nq)
    alpha = o.alpha(alpha_kind, lo, hi, seed, 0, n_elem)
    Mg = _gpu_fill(ctx, alpha)
    Mo = o.fill(alpha, threads=threads)
    assert np.isfinite(Mg).all()
    Nt = order[0] * order[1] * order[2]
    worst = 0.0
    for e in range(n_elem):
        ok, msg, w = blocks_close(Mg[e], Mo[e], n_comp, Nt)
        worst = max(worst, w)
        assert ok, f"element {e}: {msg}"
    return worst


SMALL_CASES = [
    # n_comp, order, kinds, nq, alpha_kind
    (1, (4, 4, 4), [PP], (8, 8, 8), O.ALPHA_SINE),                      # C1 shape
    (1, (2, 3, 4), [PP], (5, 6, 7), O.ALPHA_SINE),                      # anisotropic
    (3, (3, 3, 3), [PP, DD], (6, 6, 6), O.ALPHA_JACOBIAN),              # small C2 analogue
    (1, (3, 5, 2), [DD], (7, 8, 6), O.ALPHA_SINE),
    (1, (3, 4, 3), [DP], (7, 7, 7), O.ALPHA_SINE),
    (1, (3, 2, 4), [PD], (7, 7, 7), O.ALPHA_SINE),
    (1, (4, 3, 3), [(DP, PD, PP), (PD, DP, DD)], (9, 5, 7), O.ALPHA_SINE),
    (3, (4, 2, 3), [PP, (DD, PP, DP), (DP, PD, PD), (PD, DD, PP)], (6, 5, 4), O.ALPHA_SINE),
    (1, (5, 5, 5), [PP, DD], (9, 9, 9), O.ALPHA_EXPSIN),
    (1, (1, 1, 1), [PP], (3, 3, 3), O.ALPHA_SINE),
    (1, (3, 3, 3), [PP, (DP, DD, PD)], (5, 5, 5), O.ALPHA_SINE),
    (1, (2, 6, 5), [PP, DD], (4, 9, 8), O.ALPHA_SINE),
]


@pytest.mark.parametrize("case", SMALL_CASES, ids=lambda c: f"{c[0]}c-{c[1]}-{len(c[2])}t")
def test_small_shapes_match_oracle(case):
    n_comp, order, kinds, nq, ak = case
    _check_case(n_comp, order, kinds, nq, ak, 0.5, 3.0, n_elem=5)


# (round 2: 6 / 4 / 4 elements -> 48 / 32 / 24: several waves of CTAs per kernel; the
# bench additionally checks three elements of every full-size timed batch)
@pytest.mark.parametrize("name,n_elem", [("c1", 1), ("c2", 48), ("c3", 32), ("c4", 24)])
def test_baseline_configs_match_oracle(name, n_elem):
    cfg = CONFIGS[name]
    worst = _check_case(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq, cfg.alpha_kind,
                        cfg.alpha_lo, cfg.alpha_hi, n_elem=n_elem, seed=2024, threads=16)
    assert worst < 1e-12


def test_moments_match_oracle():
    cfg = CONFIGS["c2"]
    o = oracle_for(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    ctx = capi.Context(**cfg.problem())
    alpha = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 5, 0, 3)
    Ig = _gpu_moments(ctx, alpha)
    Io = o.moments(alpha, threads=4)
    for e in range(3):
        for pr in range(ctx.n_pairs):
            for s in range(len(cfg.kinds)):
                K = [ctx.K(s, d) for d in range(3)]
                n = K[0] * K[1] * K[2]
                g = Ig[e, ctx.moment_offset(pr, s):ctx.moment_offset(pr, s) + n].reshape(K[0], -1)
                r = Io[e, o.moment_offset(pr, s):o.moment_offset(pr, s) + n].reshape(K[0], -1)
                ok, (i, j) = O.block_close(g, r, RTOL)
                assert ok, (e, pr, s, i, j, g[i, j], r[i, j])


@pytest.mark.parametrize("name,variant", [("c3", v) for v in range(5)] + [("c4", v) for v in range(3)]
                         + [("c2", v) for v in range(3)] + [("c5", 0), ("c5", "cluster"), ("c5", "grouped"), ("c5", "tiled"), ("c5", "ufirst")])
def test_moment_kernel_variants_match_oracle(name, variant, monkeypatch):
    # every registered moments_v2 thread-count variant (P2S_MV2_VARIANT) and the
    # large-order moment kernel (both modes) reproduce the oracle's moment integrals
    if variant == "cluster":
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_LARGE_MOMCL", "1")
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_LARGE_MOMW", "0")
    elif variant == "grouped":
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_LARGE_MOMG", "1")
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_LARGE_MOMW", "0")
    elif variant == "tiled":
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_LARGE_MOMT", "1")
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_LARGE_MOMW", "0")
    elif variant == "ufirst":
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_LARGE_MOMW", "0")
    else:
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_MV2_VARIANT", str(variant))
    cfg = CONFIGS[name]
    o = oracle_for(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    ctx = capi.Context(**cfg.problem())
    n = 1 if name == "c5" else 2
    alpha = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 23, 0, n)
    Ig = _gpu_moments(ctx, alpha)
    Io = o.moments(alpha, threads=16)
    for e in range(n):
        for pr in range(ctx.n_pairs):
            for s in range(len(cfg.kinds)):
                K = [ctx.K(s, d) for d in range(3)]
                m = K[0] * K[1] * K[2]
                g = Ig[e, ctx.moment_offset(pr, s):ctx.moment_offset(pr, s) + m].reshape(K[0], -1)
                r = Io[e, o.moment_offset(pr, s):o.moment_offset(pr, s) + m].reshape(K[0], -1)
                ok, (i, j) = O.block_close(g, r, RTOL)
                assert ok, (e, pr, s, i, j, g[i, j], r[i, j])


@pytest.mark.parametrize("name,variant", [(c, v) for c in ("c2", "c3", "c4") for v in range(5)])
def test_two_stage_contraction_variants_match_oracle(name, variant, monkeypatch):
    # every registered contract_v2 variant of the benchmark shapes (P2S_V2_VARIANT,
    # two-stage path) gives the oracle's matrices
    monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_NO_FUSED", "1")
    monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_V2_VARIANT", str(variant))
    cfg = CONFIGS[name]
    ctx = capi.Context(**cfg.problem())
    assert ctx.kernel_path.startswith("two-stage"), ctx.kernel_path
    _check_case(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq, cfg.alpha_kind, cfg.alpha_lo,
                cfg.alpha_hi, n_elem=3, seed=29, threads=16)


@pytest.mark.parametrize("name,variant", [(c, v) for c in ("c2", "c3", "c4") for v in range(12)])
def test_every_fused_variant_matches_oracle(name, variant, monkeypatch):
    # every registered fill_fused_kernel variant of the benchmark shapes
    # (P2S_FUSED_VARIANT; indices past the last fall back to the first)
    monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_FUSED_VARIANT", str(variant))
    cfg = CONFIGS[name]
    ctx = capi.Context(**cfg.problem())
    assert ctx.kernel_path.startswith("fused"), ctx.kernel_path
    _check_case(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq, cfg.alpha_kind, cfg.alpha_lo,
                cfg.alpha_hi, n_elem=2, seed=31, threads=16)


def test_tables_match_oracle():
    for kinds, order, nq in [([PP, DD], (6, 8, 10), (14, 9, 20)), ([DP, PD], (4, 5, 3), (7, 8, 9))]:
        o = oracle_for(1, order, kinds, nq)
        ctx = capi.Context(1, order, kinds, nq)
        for s in range(len(kinds)):
            for d in range(3):
                phi, coef, x, w = ctx.tables(s, d)
                np.testing.assert_allclose(x, o.nodes(d), rtol=0, atol=4e-16)
                # the reference rule (double Newton, quadrature.cpp:27-53) is good to ~1e-14
                np.testing.assert_allclose(w, o.weights(d), rtol=2e-14, atol=0)
                np.testing.assert_allclose(phi, o.phi(s, d), rtol=2e-14, atol=1e-15)
                c = o.coef(s, d)
                np.testing.assert_allclose(coef, c, rtol=4e-16, atol=0)
                assert np.array_equal(coef == 0, c == 0)


def test_device_alpha_matches_host_generator():
    for name in ("c1", "c2", "c3", "c4"):
        cfg = CONFIGS[name]
        o = oracle_for(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
        ctx = capi.Context(**cfg.problem())
        n = 3
        d = torch.empty((n, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
        ctx.alpha_generate(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 77, 1000, n, d)
        torch.cuda.synchronize()
        h = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 77, 1000, n)
        np.testing.assert_allclose(d.cpu().numpy(), h, rtol=1e-13, atol=1e-14)


def test_fill_equals_two_stage_and_is_deterministic():
    cfg = CONFIGS["c2"]
    ctx = capi.Context(**cfg.problem())
    n = 300  # > one scheduler chunk
    st = torch.cuda.current_stream().cuda_stream
    a = torch.empty((n, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    ctx.alpha_generate(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 3, 0, n, a, st)
    M1 = torch.empty((n, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
    M2 = torch.empty_like(M1)
    I = torch.empty((n, ctx.moments_per_elem), dtype=torch.float64, device="cuda")
    ctx.fill(a, M1, ctx.n_tot, n, st)
    ctx.moments(a, I, n, st)
    ctx.contract(I, M2, ctx.n_tot, n, st)
    torch.cuda.synchronize()
    assert torch.equal(M1, M2)
    ctx.fill(a, M2, ctx.n_tot, n, st)
    torch.cuda.synchronize()
    assert torch.equal(M1, M2)
    # element matrices are symmetric for symmetric alpha and PP / P'P' terms
    assert torch.equal(M1, M1.transpose(1, 2))


def test_linearity_doubling_is_exact():
    cfg = CONFIGS["c3"]
    ctx = capi.Context(**cfg.problem())
    n = 64
    a = torch.empty((n, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    ctx.alpha_generate(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 9, 0, n, a)
    M1 = torch.empty((n, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
    M2 = torch.empty_like(M1)
    ctx.fill(a, M1, ctx.n_tot, n, 0)
    a2 = a * 2.0
    ctx.fill(a2, M2, ctx.n_tot, n, 0)
    torch.cuda.synchronize()
    assert torch.equal(M2, 2.0 * M1)


def test_leading_dimension_and_host_path():
    cfg = CONFIGS["c2"]
    o = oracle_for(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    ctx = capi.Context(**cfg.problem())
    n = 3
    alpha = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 21, 0, n)
    ld = ctx.n_tot + 5
    Mg = _gpu_fill(ctx, alpha, ld=ld)
    assert np.isnan(Mg[:, :, ctx.n_tot:]).all()  # padding untouched
    Mh = np.full((n, ctx.n_tot, ld), np.nan)
    ctx.fill_host(np.ascontiguousarray(alpha), Mh, ld, n)
    assert np.array_equal(Mh[:, :, :ctx.n_tot], Mg[:, :, :ctx.n_tot])
    Mo = o.fill(alpha, threads=4)
    for e in range(n):
        ok, msg, _ = blocks_close(Mh[e, :, :ctx.n_tot], Mo[e], cfg.n_comp, 216)
        assert ok, msg


def test_error_paths():
    cfg = CONFIGS["c1"]
    ctx = capi.Context(**cfg.problem())
    a = torch.zeros((1, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    M = torch.zeros((1, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
    with pytest.raises(capi.InvalidArgument):
        ctx.fill(a, M, ctx.n_tot - 1, 1)
    with pytest.raises(capi.InvalidArgument):
        ctx.fill(0, M, ctx.n_tot, 1)
    with pytest.raises(capi.UnsupportedShape):  # no ahead-of-time kernel, generated modules off
        capi.Context(1, (7, 3, 3), [DP], (5, 5, 5), options={"P2S_JIT": "0"})
    with pytest.raises(capi.UnsupportedShape):  # a fused-family instantiation cannot hold N = 16
        capi.Context(1, (16, 16, 16), [PP, DD], (20, 20, 20), options={"P2S_JIT_FAMILY": "fused",
                                                                        "P2S_FORCE_JIT": "1"})
    with pytest.raises(capi.InvalidArgument):
        capi.Context(1, (0, 3, 3), [PP], (5, 5, 5))


@pytest.mark.parametrize("n_comp", [1, 3])
def test_large_order_path_small_shape(n_comp):
    # the three-kernel large-order path (p2s_large.cuh) on a registered small shape
    ctx = capi.Context(n_comp, (5, 4, 3), [PP, DD], (8, 8, 6))
    assert ctx.kernel_path.startswith("large-order")
    _check_case(n_comp, (5, 4, 3), [PP, DD], (8, 8, 6),
                O.ALPHA_JACOBIAN if n_comp == 3 else O.ALPHA_SINE, 0.5, 3.0, n_elem=5)


@pytest.mark.parametrize("env", [
    {"P2S_XCHUNK_MB": "1"},                                 # many chunks, two u streams
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_USTREAMS": "1"},      # many chunks, one u stream
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_OVERLAP": "0"},       # serial v/w and u stages
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_PS": "0"},            # u stage without parity split
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_FIB": "2"},           # two u fibers per thread
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_PRIO": "1"},          # high-priority v/w stream
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_UPERSIST": "1"},      # persistent u stage, 1 CTA / SM
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_UPERSIST": "0"},      # one u-stage CTA per tile
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_USMEM": "1"},         # u coefficients in shared memory
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_MOMCL": "1", "P2S_LARGE_MOMW": "0"},  # cluster moments (DSMEM)
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_MOMG": "1", "P2S_LARGE_MOMW": "0"},   # grouped v / w moment passes
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_MOMT": "1", "P2S_LARGE_MOMW": "0"},   # register-tiled moment passes (u first)
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_MOMW": "0"},          # u-first moment kernel, one row per thread
    {"P2S_XCHUNK_MB": "1", "P2S_LARGE_MOMW": "1"},          # w-first register-tiled moment kernel
])
def test_large_order_path_chunk_schedules(env, monkeypatch):
    # the chunked v/w -> u pipeline over many X chunks (double buffer reuse,
    # alternating u streams) gives the oracle's matrices
    for k, v in env.items():
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, k, v)
    ctx = capi.Context(3, (5, 4, 3), [PP, DD], (8, 8, 6))
    assert ctx.kernel_path.startswith("large-order")
    _check_case(3, (5, 4, 3), [PP, DD], (8, 8, 6), O.ALPHA_JACOBIAN, 0.5, 3.0, n_elem=40)


@pytest.mark.parametrize("env", [{"P2S_LARGE_XS": "0"}, {"P2S_LARGE_XS": "1", "P2S_XCHUNK_MB": "20"},
                                 {"P2S_LARGE_XS": "1", "P2S_LARGE_UPERSIST": "0"}])
def test_c5_u_stage_schedules_match_oracle(env, monkeypatch):
    # C5 with the u stage's next parity class staged in shared memory by cp.async
    # (default; across tiles of the persistent CTAs and across X chunks) and with
    # direct L2 loads
    for k, v in env.items():
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, k, v)
    cfg = CONFIGS["c5"]
    worst = _check_case(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq, cfg.alpha_kind,
                        cfg.alpha_lo, cfg.alpha_hi, n_elem=3, seed=7, threads=16)
    assert worst < 1e-12


def test_c5_matches_oracle():
    # BASELINE config 5 (order 16, 36^3 points): 134 MB per element matrix
    cfg = CONFIGS["c5"]
    ctx = capi.Context(**cfg.problem())
    assert ctx.kernel_path.startswith("large-order")
    worst = _check_case(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq, cfg.alpha_kind,
                        cfg.alpha_lo, cfg.alpha_hi, n_elem=2, seed=5, threads=16)
    assert worst < 1e-12


def _select_variant(monkeypatch, problem, env_var, marker):
    """Set env_var (P2S_FUSED_VARIANT / P2S_V2_VARIANT) to the first registered
    variant of `problem` whose kernel_path contains `marker`."""
    for v in range(24):
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, env_var, str(v))
        ctx = capi.Context(*problem)
        if marker in ctx.kernel_path:
            return ctx
    pytest.fail(f"no variant with {marker!r} registered for {problem}")


# (config or small case, two-stage?, stage-C variant marker, elements)
VARIANT_CASES = [
    ("c2", False, "DMMA", 6),
    ("c3", False, "DMMA", 3),
    ("c4", False, "DMMA", 3),
    ("c2", False, "paired", 6),
    ("c3", False, "paired", 3),
    ("c4", False, "paired", 3),
    ("c2", False, "parity split", 6),
    ("c3", False, "parity split, paired", 3),
    ("c4", False, "parity split", 3),
    ("c4", False, "w-last", 3),
    ("c2", False, "32-B stores", 6),
    ("c3", False, "32-B stores", 3),
    ("c3", False, "parity split, 32-B stores", 3),
    ("c4", False, "parity split, 32-B stores", 3),
    ("c2", False, "(n1, n2)-symmetric", 6),
    ("c3", False, "paired 16-B stores, (n1, n2)-symmetric", 3),
    ("c4", False, "parity split, (n1, n2)-symmetric", 3),
    ((3, (3, 3, 3), [PP, DD], (6, 6, 6)), True, "parity split", 4),
    ((1, (4, 3, 3), [(DP, PD, PP), (PD, DP, DD)], (9, 5, 7)), True, "parity split", 4),
    ((3, (3, 3, 3), [PP, DD], (6, 6, 6)), True, "DMMA", 4),
    ((1, (4, 3, 3), [(DP, PD, PP), (PD, DP, DD)], (9, 5, 7)), True, "DMMA", 4),
]


@pytest.mark.parametrize("case,two_stage,marker,n_elem", VARIANT_CASES,
                         ids=lambda c: str(c)[:24])
@pytest.mark.parametrize("odd_ld", [False, True])
def test_stage_c_variants_match_oracle(case, two_stage, marker, n_elem, odd_ld, monkeypatch):
    """Stage-C variants: on the FP64 tensor cores (DMMA, p2s_mma.cuh) and with
    paired 16-B stores -- same bar; even ldM takes the 16-B store path, odd
    ldM the scalar one."""
    if isinstance(case, str):
        cfg = CONFIGS[case]
        n_comp, order, kinds, nq = cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq
        ak, lo, hi = cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi
    else:
        n_comp, order, kinds, nq = case
        ak, lo, hi = O.ALPHA_SINE, 0.5, 3.0
    if two_stage:
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_NO_FUSED", "1")
    ctx = _select_variant(monkeypatch, (n_comp, order, kinds, nq),
                          "P2S_V2_VARIANT" if two_stage else "P2S_FUSED_VARIANT", marker)
    o = oracle_for(n_comp, order, kinds, nq)
    alpha = o.alpha(ak, lo, hi, 77, 0, n_elem)
    ld = ctx.n_tot + (1 if odd_ld else 0)
    Mg = _gpu_fill(ctx, alpha, ld=ld)
    Mo = o.fill(alpha, threads=8)
    assert np.isfinite(Mg[:, :, :ctx.n_tot]).all()
    if odd_ld:
        assert np.isnan(Mg[:, :, ctx.n_tot:]).all()  # padding column untouched
    Nt = order[0] * order[1] * order[2]
    for e in range(n_elem):
        ok, msg, _ = blocks_close(Mg[e, :, :ctx.n_tot], Mo[e], n_comp, Nt)
        assert ok, f"element {e}: {msg}"
