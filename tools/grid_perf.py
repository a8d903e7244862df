"""Throughput of every drop-in grid shape (paper_1703_09619_b200/shape_grid.py)
on one B200: p2s_fill over a batch of ~2-4 GB of output, alpha resident, CUDA
events around 5 fills after 2 warm-ups; fraction of the HBM roofline on the
whole fill's algorithmic bytes (alpha read + M write: every byte the fill must
move).  One JSON object per shape, one process (modules prepared by build()).

  python tools/grid_perf.py > gpurun_out/grid_perf.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1703_09619_b200 import capi, shape_grid  # noqa: E402


def main():
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    for case in shape_grid.ALL:
        nc, order, kinds, nq, basis = case
        try:
            ctx = capi.Context(nc, order, kinds, nq, basis=basis)
            per = 8 * (ctx.alpha_per_elem + ctx.n_tot * ctx.n_tot)
            E = int(max(1, min(65536, 3e9 // per)))
            A = torch.empty((E, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
            ctx.alpha_generate(0, 0.5, 3.0, 1, 0, E, A, sp)
            M = torch.empty((E, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
            for _ in range(2):
                ctx.fill(A, M, ctx.n_tot, E, sp)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(5):
                ctx.fill(A, M, ctx.n_tot, E, sp)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            gbs = E * per / (ms / 1e3) / 1e9
            out = {"shape": shape_grid.shape_id(case), "elements": E, "elem_per_s": E / (ms / 1e3),
                   "alpha_plus_M_GBs": gbs, "frac": gbs / hbm, "path": ctx.kernel_path}
            del A, M
            ctx.close()
            torch.cuda.empty_cache()
        except Exception as ex:  # report and continue
            out = {"shape": shape_grid.shape_id(case), "error": str(ex)[:300]}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
