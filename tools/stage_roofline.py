"""Roofline of the separate stage kernels behind p2s_moments / p2s_contract
(two-stage API) next to the fused p2s_fill, per config: CUDA events on the
launching stream, inputs resident, outputs >> L2.

usage: python tools/stage_roofline.py [c2 c3 c4 ...]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1703_09619_b200 import capi  # noqa: E402
from paper_1703_09619_b200.configs import CONFIGS, algorithmic_counts  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.0) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6550.0
for name in sys.argv[1:] or ["c2", "c3", "c4"]:
    cfg = CONFIGS[name]
    ctx = capi.Context(**cfg.problem())
    per = 8 * (ctx.alpha_per_elem + ctx.moments_per_elem + ctx.n_tot ** 2)
    E = min(cfg.n_elem, int(0.4 * torch.cuda.get_device_properties(0).total_memory // per))
    st = torch.cuda.current_stream().cuda_stream
    a = torch.empty((E, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    ctx.alpha_generate(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 7, 0, E, a, st)
    I = torch.empty((E, ctx.moments_per_elem), dtype=torch.float64, device="cuda")
    M = torch.empty((E, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
    c = algorithmic_counts(cfg)
    tm = timed(lambda: ctx.moments(a, I, E, st), 5)
    tc = timed(lambda: ctx.contract(I, M, ctx.n_tot, E, st), 5)
    tf = timed(lambda: ctx.fill(a, M, ctx.n_tot, E, st), 5)
    out = {"config": name, "elements": E, "kernel_path": ctx.kernel_path,
           "moments": {"s": tm, "GB/s": c["bytes_mom"] * E / tm / 1e9, "frac": c["bytes_mom"] * E / tm / 1e9 / peak,
                       "TF/s": c["flop_mom"] * E / tm / 1e12},
           "contract": {"s": tc, "GB/s": c["bytes_con"] * E / tc / 1e9, "frac": c["bytes_con"] * E / tc / 1e9 / peak,
                        "TF/s": c["flop_con"] * E / tc / 1e12},
           "two_stage_elem_per_s": E / (tm + tc), "fused_elem_per_s": E / tf}
    print(json.dumps(out), flush=True)
    ctx.close()
    del a, I, M
    torch.cuda.empty_cache()
