"""Large-path moment kernel A/B (P2S_LARGE_MOMG / MSPLIT / MOMCL) on a config:
python tools/mom_ab.py [c5|c12 ...]  -> us per element, algorithmic TF/s, checksum"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1703_09619_b200 import capi  # noqa: E402
from paper_1703_09619_b200.configs import CONFIGS, algorithmic_counts  # noqa: E402

names = sys.argv[1:] or ["c5", "c12"]
W0 = {"P2S_LARGE_MOMW": "0"}
VARIANTS = [{}, W0, {**W0, "P2S_LARGE_MOMG": "1"}, {**W0, "P2S_LARGE_MOMT": "1"}, {**W0, "P2S_LARGE_MSPLIT": "1"}]
for name in names:
    cfg = CONFIGS[name]
    c = algorithmic_counts(cfg)
    # generated modules (c12) hold the default and the u-first kernel only; the grouped / tiled
    # u-first measurement variants exist in ahead-of-time shapes (c5)
    for opts in (VARIANTS if name == "c5" else [v for v in VARIANTS if "P2S_LARGE_MOMG" not in v and "P2S_LARGE_MOMT" not in v]):
        ctx = capi.Context(**cfg.problem(), options=opts)
        E = 512 if name == "c5" else 2048
        st = torch.cuda.current_stream().cuda_stream
        a = torch.empty((E, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
        ctx.alpha_generate(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, 7, 0, E, a, st)
        I = torch.empty((E, ctx.moments_per_elem), dtype=torch.float64, device="cuda")
        for _ in range(3):
            ctx.moments(a, I, E, st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ctx.moments(a, I, E, st)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 10 / 1e3
        print(name, opts, "us/elem", round(t / E * 1e6, 3), "TF/s (algorithmic)",
              round(c["flop_mom"] * E / t / 1e12, 2), "checksum", repr(float(I.double().sum())), flush=True)
        ctx.close()
