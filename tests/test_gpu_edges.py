"""Edge cases of every entry point (the reference's own tests cover empty
batches, argument validation and thread-count independence):
empty batches are no-ops that touch nothing, ragged batch sizes that straddle
the internal chunkings, grids beyond 65535 CTAs, and the argument limits."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1703_09619_b200 import capi
from paper_1703_09619_b200.capi import BASIS_CONFORMING, DD, PP
from paper_1703_09619_b200.configs import CONFIGS

from helpers import blocks_close, oracle_for

pytestmark = pytest.mark.gpu


def _nan(*shape):
    return torch.full(shape, float("nan"), dtype=torch.float64, device="cuda")


def test_empty_batches_touch_nothing():
    cfg = CONFIGS["c2"]
    ctx = capi.Context(**cfg.problem())
    sp = torch.cuda.current_stream().cuda_stream
    a = _nan(1, ctx.alpha_per_elem)
    I = _nan(1, ctx.moments_per_elem)
    M = _nan(1, ctx.n_tot, ctx.n_tot)
    ctx.fill(a, M, ctx.n_tot, 0, sp)
    ctx.moments(a, I, 0, sp)
    ctx.contract(I, M, ctx.n_tot, 0, sp)
    ctx.alpha_generate(O.ALPHA_JACOBIAN, 0.5, 3.0, 1, 0, 0, a, sp)
    ctx.fill_geometry(a, M, ctx.n_tot, 0, sp)
    ha = np.full((1, ctx.alpha_per_elem), np.nan)
    hM = np.full((1, ctx.n_tot, ctx.n_tot), np.nan)
    ctx.fill_host(ha, hM, ctx.n_tot, 0)
    d = capi.DirectContext(**cfg.problem())
    d.fill(a, M, ctx.n_tot, 0, sp)
    c2d = capi.Cheb2dContext(3, 3, 8)
    c2d.kernel_tables(a, I, 0)
    c2d.assemble(I, M, 0)
    torch.cuda.synchronize()
    assert torch.isnan(M).all() and torch.isnan(I).all() and torch.isnan(a).all()
    assert np.isnan(hM).all()


@pytest.mark.parametrize("path_env", [{}, {"P2S_NO_FUSED": "1"}, {"P2S_FORCE_GENERIC": "1",
                                                                   "P2S_NO_FUSED": "1"}])
@pytest.mark.parametrize("n", [1, 7, 33])
def test_ragged_batches_match_oracle(n, path_env, monkeypatch):
    for k, v in path_env.items():
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, k, v)
    pb = (3, (3, 3, 3), [PP, DD], (6, 6, 6))
    ctx = capi.Context(*pb)
    o = oracle_for(*pb)
    alpha = o.alpha(O.ALPHA_JACOBIAN, 0.5, 3.0, 13, 0, n)
    M = _nan(n, ctx.n_tot, ctx.n_tot)
    ctx.fill(torch.from_numpy(alpha).cuda(), M, ctx.n_tot, n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    Mo = o.fill(alpha, threads=8)
    for e in range(n):
        ok, msg, _ = blocks_close(M[e].cpu().numpy(), Mo[e], 3, 27)
        assert ok, (e, msg)


def test_host_path_across_ring_chunks():
    """p2s_fill_host pipelines 64 MB chunks through a 2-slot ring: 80 C2 elements
    span five chunks (19 per chunk; elements 75 | 76 straddle a boundary) and
    reuse both slots twice."""
    cfg = CONFIGS["c2"]
    ctx = capi.Context(**cfg.problem())
    n = 80
    o = oracle_for(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    alpha = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 3, 0, n)
    hM = np.full((n, ctx.n_tot, ctx.n_tot), np.nan)
    ctx.fill_host(alpha, hM, ctx.n_tot, n)
    d = torch.from_numpy(alpha).cuda()
    M = _nan(n, ctx.n_tot, ctx.n_tot)
    ctx.fill(d, M, ctx.n_tot, n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(hM, M.cpu().numpy())
    Mo = o.fill(alpha[[0, 75, 76, 79]], threads=8)
    for i, e in enumerate([0, 75, 76, 79]):
        ok, msg, _ = blocks_close(hM[e], Mo[i], cfg.n_comp, 216)
        assert ok, (e, msg)


@pytest.mark.parametrize("env", [{}, {"P2S_NO_FUSED": "1"}])
def test_grid_beyond_65535_ctas(env, monkeypatch):
    """70 000 C1 elements: one CTA per (element, pair) unit in the fused kernel,
    70 000 moment CTAs in the two-stage path."""
    for k, v in env.items():
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, k, v)
    cfg = CONFIGS["c1"]
    ctx = capi.Context(**cfg.problem())
    n = 70000
    sp = torch.cuda.current_stream().cuda_stream
    a = torch.empty((n, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    ctx.alpha_generate(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 5, 0, n, a, sp)
    M = _nan(n, ctx.n_tot, ctx.n_tot)
    ctx.fill(a, M, ctx.n_tot, n, sp)
    torch.cuda.synchronize()
    assert not torch.isnan(M).any()
    o = oracle_for(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    pick = [0, 65535, 69999]
    Mo = o.fill(a[pick].cpu().numpy(), threads=4)
    for i, e in enumerate(pick):
        ok, msg, _ = blocks_close(M[e].cpu().numpy(), Mo[i], 1, 64)
        assert ok, (e, msg)


@pytest.mark.parametrize("bad", [
    dict(n_comp=4), dict(n_comp=0), dict(order=(33, 3, 3)), dict(nq=(65, 4, 4)), dict(nq=(4, 0, 4)),
    dict(kinds=[4]), dict(kinds=[PP, DD, PP, DD, PP]), dict(basis=2),
    dict(basis=BASIS_CONFORMING, order=(1, 2, 2)),
])
def test_argument_limits(bad):
    args = dict(n_comp=1, order=(3, 3, 3), kinds=[PP], nq=(4, 4, 4), basis=0)
    args.update(bad)
    with pytest.raises(capi.InvalidArgument):
        capi.Context(args["n_comp"], args["order"], args["kinds"], args["nq"], basis=args["basis"])
    with pytest.raises(capi.InvalidArgument):
        capi.DirectContext(args["n_comp"], args["order"], args["kinds"], args["nq"], basis=args["basis"])


def test_unregistered_orders_need_a_generated_module():
    # valid problem with no ahead-of-time kernel for N_u = 11: accepted through a
    # generated module; with generated modules switched off it is unsupported
    assert capi.shape_supported(1, (11, 3, 3), [PP], (12, 4, 4))
    ctx = capi.Context(1, (11, 3, 3), [PP], (12, 4, 4))
    assert "generated module" in ctx.kernel_path, ctx.kernel_path
    with pytest.raises(capi.UnsupportedShape):
        capi.Context(1, (11, 3, 3), [PP], (12, 4, 4), options={"P2S_JIT": "0"})
    with pytest.raises(capi.InvalidArgument):
        capi.Context(1, (4, 4, 4), [PP], (8, 8, 8), options={"P2S_NO_SUCH_KNOB": "1"})


GUARD = 8192  # doubles of canary on each side of the output matrices


@pytest.mark.parametrize("problem,env", [
    ((3, (6, 6, 6), [PP, DD], (14, 14, 14)), {}),                                    # C2 fused
    ((3, (6, 6, 6), [PP, DD], (14, 14, 14)), {"P2S_FUSED_VARIANT": "1"}),          # paired stores
    ((1, (8, 8, 8), [PP, DD], (20, 20, 20)), {}),                                   # C3 fused
    ((3, (10, 6, 4), [PP, DD], (16, 16, 16)), {}),                                  # C4 fused
    ((3, (5, 4, 3), [PP, DD], (8, 8, 6)), {"P2S_XCHUNK_MB": "1"}),                 # large path
    ((1, (2, 3, 4), [PP], (5, 6, 7)), {"P2S_FORCE_GENERIC": "1"}),                 # generic kernels
    ((1, (2, 3, 4), [PP], (5, 6, 7)), {}),                                          # generated fused
    ((1, (9, 5, 4), [PP, DD], (11, 7, 6)), {"P2S_XCHUNK_MB": "1"}),                # generated large
])
@pytest.mark.parametrize("odd_ld", [False, True])
def test_writes_stay_inside_the_output(problem, env, odd_ld, monkeypatch):
    """Canary zones around M (and the padding columns of ld_M > n_tot) are left
    untouched by every kernel path; compute-sanitizer is unavailable on the pool,
    so out-of-bounds stores are caught by value here."""
    for k, v in env.items():
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, k, v)
    ctx = capi.Context(*problem)
    n = 7
    ld = ctx.n_tot + (1 if odd_ld else 0)
    o = oracle_for(*problem)
    alpha = torch.from_numpy(o.alpha(O.ALPHA_SINE, 0.5, 3.0, 3, 0, n)).cuda()
    canary = -1.2345e300
    buf = torch.full((GUARD + n * ctx.n_tot * ld + GUARD,), canary, dtype=torch.float64, device="cuda")
    M = buf[GUARD:GUARD + n * ctx.n_tot * ld].view(n, ctx.n_tot, ld)
    ctx.fill(alpha, M, ld, n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    b = buf.cpu().numpy()
    assert (b[:GUARD] == canary).all() and (b[-GUARD:] == canary).all()
    Mh = M.cpu().numpy()
    assert np.isfinite(Mh[:, :, :ctx.n_tot]).all() and not (Mh[:, :, :ctx.n_tot] == canary).any()
    if odd_ld:
        assert (Mh[:, :, ctx.n_tot:] == canary).all()


@pytest.mark.parametrize("env", [
    {"P2S_CHUNK_MB": "1"},                                   # C3 default: two-stage, overlapped
    {"P2S_CHUNK_MB": "1", "P2S_TWO_STAGE_OVERLAP": "0"},     # serial chunks
    {"P2S_CHUNK_MB": "1", "P2S_NO_FUSED": "1"},
])
def test_two_stage_chunk_pipeline_matches_oracle(env, monkeypatch):
    """The two-stage fill over many scheduler chunks (double-buffered moment
    scratch, the next chunk's moments on a side stream) gives the oracle's
    matrices; C3 runs this path by default."""
    for k, v in env.items():
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, k, v)
    cfg = CONFIGS["c3"]
    ctx = capi.Context(**cfg.problem())
    assert ctx.kernel_path.startswith("two-stage"), ctx.kernel_path
    n = 61  # 23 elements per 1 MB chunk: three chunks, the last one ragged
    o = oracle_for(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    alpha = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 17, 0, n)
    M = _nan(n, ctx.n_tot, ctx.n_tot)
    ctx.fill(torch.from_numpy(alpha).cuda(), M, ctx.n_tot, n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    Mo = o.fill(alpha, threads=16)
    Mg = M.cpu().numpy()
    for e in range(n):
        ok, msg, _ = blocks_close(Mg[e], Mo[e], 1, ctx.n_tot)
        assert ok, (e, msg)


@pytest.mark.parametrize("problem", [
    (3, (5, 4, 3), [PP, DD], (8, 8, 6)),      # registered large-path test shape
    (1, (9, 5, 4), [PP, DD], (11, 7, 6)),     # generated module of the large family
])
def test_large_path_graph_replay_matches_direct_launches(problem, monkeypatch):
    """A large-path fill that comes back with the same buffers is captured into a
    CUDA graph on its second call and replayed from the third: every call gives the
    oracle's matrices, bitwise equal to a context with graphs off; other buffers
    and other element counts launch directly (and get their own graphs)."""
    monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_XCHUNK_MB", "1")  # several chunks
    if problem[1] == (9, 5, 4):
        monkeypatch.setitem(capi.DEFAULT_OPTIONS, "P2S_JIT_FAMILY", "large")
    n = 23
    o = oracle_for(*problem)
    alpha_np = o.alpha(O.ALPHA_SINE, 0.5, 3.0, 11, 0, n)
    alpha = torch.from_numpy(alpha_np).cuda()
    Mo = o.fill(alpha_np, threads=8)
    st = torch.cuda.current_stream().cuda_stream
    ref_ctx = capi.Context(*problem, options={"P2S_GRAPH": "0"})
    Mref = _nan(n, ref_ctx.n_tot, ref_ctx.n_tot)
    ref_ctx.fill(alpha, Mref, ref_ctx.n_tot, n, st)
    torch.cuda.synchronize()
    ctx = capi.Context(*problem)
    assert ctx.kernel_path.startswith("large-order"), ctx.kernel_path
    M = _nan(n, ctx.n_tot, ctx.n_tot)
    side = torch.cuda.Stream()
    for call in range(5):  # 0 direct, 1 capture + launch, 2.. replay; call 3 on another stream
        M.fill_(float("nan"))
        torch.cuda.synchronize()
        s = side.cuda_stream if call == 3 else st
        ctx.fill(alpha, M, ctx.n_tot, n, s)
        torch.cuda.synchronize()
        assert torch.equal(M, Mref), f"call {call}"
    Nt = problem[1][0] * problem[1][1] * problem[1][2]
    Mg = M.cpu().numpy()
    for e in range(n):
        ok, msg, _ = blocks_close(Mg[e], Mo[e], problem[0], Nt)
        assert ok, (e, msg)
    # a shorter batch and a second output buffer between replays
    M2 = _nan(n, ctx.n_tot, ctx.n_tot)
    for call in range(3):
        ctx.fill(alpha, M2, ctx.n_tot, n - 5, st)
        ctx.fill(alpha, M, ctx.n_tot, n, st)
    torch.cuda.synchronize()
    assert torch.equal(M2[:n - 5], Mref[:n - 5]) and torch.isnan(M2[n - 5:]).all()
    assert torch.equal(M, Mref)


@pytest.mark.parametrize("name,shift", [("c4", 2), ("c4", 4), ("c2", 2)])
def test_alpha_alignment_is_checked(name, shift):
    """alpha rows are read with 32-B loads when nq_u % 4 == 0 (C4: nq 16): an
    alpha 16-B but not 32-B aligned is rejected up front instead of faulting;
    32-B aligned offsets (and 16-B offsets for C2's nq 14) fill correctly."""
    cfg = CONFIGS[name]
    ctx = capi.Context(**cfg.problem())
    n = 2
    o = oracle_for(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    alpha = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 8, 0, n)
    buf = torch.zeros(alpha.size + 8, dtype=torch.float64, device="cuda")
    a = buf[shift:shift + alpha.size]
    a.copy_(torch.from_numpy(alpha.reshape(-1)))
    M = _nan(n, ctx.n_tot, ctx.n_tot)
    st = torch.cuda.current_stream().cuda_stream
    need32 = cfg.nq[0] % 4 == 0
    if need32 and (shift * 8) % 32:
        with pytest.raises(capi.InvalidArgument):
            ctx.fill(a, M, ctx.n_tot, n, st)
        with pytest.raises(capi.InvalidArgument):
            ctx.moments(a, torch.zeros((n, ctx.moments_per_elem), dtype=torch.float64, device="cuda"), n, st)
        return
    ctx.fill(a, M, ctx.n_tot, n, st)
    torch.cuda.synchronize()
    Mo = o.fill(alpha, threads=8)
    Nt = cfg.order[0] * cfg.order[1] * cfg.order[2]
    for e in range(n):
        ok, msg, _ = blocks_close(M[e].cpu().numpy(), Mo[e], cfg.n_comp, Nt)
        assert ok, msg


def test_concurrent_streams_share_context_scratch():
    """Two streams fill through one two-stage (C3) and one large-order context at
    once: the context event orders their use of the moment / intermediate scratch
    (each result equals the single-stream fill bitwise)."""
    for problem, opts in (((1, (8, 8, 8), [PP, DD], (20, 20, 20)), {"P2S_CHUNK_MB": "1"}),
                          ((3, (5, 4, 3), [PP, DD], (8, 8, 6)), {"P2S_XCHUNK_MB": "1"})):
        ctx = capi.Context(*problem, options=opts)
        o = oracle_for(*problem)
        n = 40
        alpha = torch.from_numpy(o.alpha(O.ALPHA_SINE, 0.5, 3.0, 21, 0, n)).cuda()
        ref = _nan(n, ctx.n_tot, ctx.n_tot)
        ctx.fill(alpha, ref, ctx.n_tot, n, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        A, B = _nan(n, ctx.n_tot, ctx.n_tot), _nan(n, ctx.n_tot, ctx.n_tot)
        for _ in range(3):
            ctx.fill(alpha, A, ctx.n_tot, n, s1.cuda_stream)
            ctx.fill(alpha, B, ctx.n_tot, n, s2.cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(A, ref) and torch.equal(B, ref)
