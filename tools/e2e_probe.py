import sys, time, torch
sys.path.insert(0, '.')
from paper_1703_09619_b200 import capi
from paper_1703_09619_b200.configs import CONFIGS
cfg = CONFIGS["c2"]
ctx = capi.Context(**cfg.problem())
E2 = 1024
a = torch.empty((E2, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
ctx.alpha_generate(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 7, 0, E2, a, torch.cuda.current_stream().cuda_stream)
h_alpha = torch.empty((E2, ctx.alpha_per_elem), dtype=torch.float64, pin_memory=True)
h_alpha.copy_(a)
h_M = torch.empty((E2, ctx.n_tot, ctx.n_tot), dtype=torch.float64, pin_memory=True)
ctx.fill_host(h_alpha, h_M, ctx.n_tot, E2)
t = time.perf_counter()
for _ in range(3): ctx.fill_host(h_alpha, h_M, ctx.n_tot, E2)
dt = (time.perf_counter() - t) / 3
print(sys.argv[1], "MB chunks:", round(E2 / dt), "elem/s", round(E2 * ctx.n_tot**2 * 8 / dt / 1e9, 1), "GB/s D2H")
