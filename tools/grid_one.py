"""One grid shape (by index into shape_grid.ALL or by shape id), a few fills: a
target for ncu launch lists.  python tools/grid_one.py <index|id> [elements] [fills] ["KEY=VALUE;..."]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1703_09619_b200 import capi, shape_grid  # noqa: E402


def main():
    key = sys.argv[1]
    cases = shape_grid.ALL
    case = cases[int(key)] if key.isdigit() else next(c for c in cases if shape_grid.shape_id(c) == key)
    nc, order, kinds, nq, basis = case
    opts = dict(kv.split("=") for kv in sys.argv[4].split(";")) if len(sys.argv) > 4 and sys.argv[4] else None
    ctx = capi.Context(nc, order, kinds, nq, basis=basis, options=opts)
    per = 8 * (ctx.alpha_per_elem + ctx.n_tot * ctx.n_tot)
    E = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else int(max(1, min(65536, 3e9 // per)))
    fills = int(sys.argv[3]) if len(sys.argv) > 3 and int(sys.argv[3]) > 0 else 5
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    A = torch.empty((E, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    ctx.alpha_generate(0, 0.5, 3.0, 1, 0, E, A, sp)
    M = torch.empty((E, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):  # (the third call of a large-path fill replays its graph)
        ctx.fill(A, M, ctx.n_tot, E, sp)
    e0.record(st)
    for _ in range(fills):
        ctx.fill(A, M, ctx.n_tot, E, sp)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / fills
    print(shape_grid.shape_id(case), "elements", E, "ms/fill", round(ms, 3), "elem/s", round(E / ms * 1e3),
          "GB/s", round(E * per / ms / 1e6, 1), sys.argv[4] if len(sys.argv) > 4 else "", ctx.kernel_path[:50])


if __name__ == "__main__":
    main()
