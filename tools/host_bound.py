"""Is a fill host-bound?  Host time of the p2s_fill call (launch code only, no sync)
next to the device time of the same fills.  python tools/host_bound.py c12 [elements]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1703_09619_b200 import capi  # noqa: E402
from paper_1703_09619_b200.configs import CONFIGS  # noqa: E402


def main():
    cfg = CONFIGS[sys.argv[1]]
    opts = dict(kv.split("=") for kv in sys.argv[3].split(";")) if len(sys.argv) > 3 else None
    ctx = capi.Context(**cfg.problem(), options=opts)
    per = 8 * (ctx.alpha_per_elem + ctx.n_tot * ctx.n_tot)
    E = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else int(max(1, min(65536, 40e9 // per)))
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    A = torch.empty((E, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    ctx.alpha_generate(0, 0.5, 3.0, 1, 0, E, A, sp)
    M = torch.empty((E, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
    for _ in range(2):
        ctx.fill(A, M, ctx.n_tot, E, sp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 5
    e0.record(st)
    t0 = time.perf_counter()
    for _ in range(n):
        ctx.fill(A, M, ctx.n_tot, E, sp)
    t1 = time.perf_counter()
    e1.record(st)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dev = e0.elapsed_time(e1) / n
    print(sys.argv[1], "elements", E, "host ms/fill (launch code)", round((t1 - t0) * 1e3 / n, 3),
          "device ms/fill", round(dev, 3), "wall incl. sync", round((t2 - t0) * 1e3 / n, 3),
          "elem/s", round(E / dev * 1e3), ctx.kernel_path[:60])


if __name__ == "__main__":
    main()
