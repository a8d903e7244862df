"""Moment kernel only (a target for ncu): python tools/moments_only.py <config> <elements> [KEY=VALUE options ...]"""
import sys, torch
sys.path.insert(0, '.')
from paper_1703_09619_b200 import capi
from paper_1703_09619_b200.configs import CONFIGS
cfg = CONFIGS[sys.argv[1]]
opts = dict(kv.split("=", 1) for kv in sys.argv[3:])
ctx = capi.Context(**cfg.problem(), options=opts)
E = int(sys.argv[2])
st = torch.cuda.current_stream().cuda_stream
a = torch.empty((E, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
ctx.alpha_generate(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 7, 0, E, a, st)
I = torch.empty((E, ctx.moments_per_elem), dtype=torch.float64, device="cuda")
for _ in range(3): ctx.moments(a, I, E, st)
torch.cuda.synchronize()
