"""Large-path moment kernel vs its k1 chunk (P2S_JIT_KC) on a config, through generated
modules: python tools/mom_kc_sweep.py prepare|run [c5] [kc ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1703_09619_b200 import capi  # noqa: E402
from paper_1703_09619_b200.configs import CONFIGS, algorithmic_counts  # noqa: E402

mode = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else "c5"
kcs = [int(k) for k in sys.argv[3:]] or [4, 6, 8, 10, 16]
cfg = CONFIGS[name]
pb = cfg.problem()
for kc in kcs:
    opts = {"P2S_FORCE_JIT": "1", "P2S_JIT_FAMILY": "large", "P2S_JIT_KC": str(kc)}
    if mode == "prepare":
        print(kc, capi.shape_prepare(pb["n_comp"], pb["order"], pb["kinds"], pb["nq"], options=opts)[:90], flush=True)
        continue
    import torch
    ctx = capi.Context(**pb, options=opts)
    E = 512
    st = torch.cuda.current_stream().cuda_stream
    a = torch.empty((E, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    ctx.alpha_generate(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 7, 0, E, a, st)
    I = torch.empty((E, ctx.moments_per_elem), dtype=torch.float64, device="cuda")
    for _ in range(2):
        ctx.moments(a, I, E, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ctx.moments(a, I, E, st)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 5 / 1e3
    c = algorithmic_counts(cfg)
    print(name, "kc", kc, "us/elem", round(t / E * 1e6, 3), "TF/s (algorithmic)", round(c["flop_mom"] * E / t / 1e12, 2),
          "checksum", float(I.sum()), flush=True)
    ctx.close()
