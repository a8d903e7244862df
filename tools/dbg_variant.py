"""Run one fill of a registered two-stage variant (P2S_NO_FUSED, P2S_V2_VARIANT) on
constant alpha: python tools/dbg_variant.py <c2|c3|c4|t> <variant> <n_elem>"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_09619_b200 import capi  # noqa: E402
from paper_1703_09619_b200.capi import DD, PP  # noqa: E402
from paper_1703_09619_b200.configs import CONFIGS  # noqa: E402

name, v, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
os.environ["P2S_NO_FUSED"] = "1"
os.environ["P2S_V2_VARIANT"] = v
pb = dict(n_comp=3, order=(3, 3, 3), kinds=[PP, DD], nq=(6, 6, 6)) if name == "t" else CONFIGS[name].problem()
ctx = capi.Context(**pb)
print(ctx.kernel_path)
a = torch.ones((n, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
M = torch.zeros((n, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
ctx.fill(a, M, ctx.n_tot, n, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", float(M.abs().sum()))
