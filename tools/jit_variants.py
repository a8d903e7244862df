"""Parity + speed of generated-module variants of one shape (planner overrides,
p2s_create_ex options P2S_JIT_*), each in its own process so a faulting variant
cannot poison the others.

  python tools/jit_variants.py prepare   # build every variant's module (CPU)
  python tools/jit_variants.py run       # on a GPU: parity vs oracle + elem/s
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PP, DD, DP, PD = 0, 1, 2, 3
S7 = (1, (7, 7, 7), [PP, DD], (14, 14, 14), 0)
S793 = (1, (7, 9, 3), [(DD, PD, DP), (PP, DP, DD), (PD, DP, DD), (PD, DP, DP)], (12, 12, 2), 0)
S3 = (1, (3, 3, 3), [PP, DD], (6, 6, 6), 0)
# P2S_JIT_SWEEP=<file.json>: cases from a JSON list of [grid index, {options}] over
# shape_grid.ALL instead of the built-in list (planner sweeps over the drop-in grid)
CASES = [
    # (shape, options)
    (S7, {"P2S_JIT_FLAGS": "0", "P2S_JIT_T": "1", "P2S_JIT_MINB": "1"}),
    (S7, {"P2S_JIT_FLAGS": "1", "P2S_JIT_T": "1", "P2S_JIT_MINB": "1"}),
    (S3, {"P2S_FORCE_JIT": "1", "P2S_JIT_FLAGS": "0", "P2S_JIT_T": "1"}),
    (S3, {"P2S_FORCE_JIT": "1", "P2S_JIT_FLAGS": "0", "P2S_JIT_T": "3"}),
    (S3, {"P2S_FORCE_JIT": "1", "P2S_JIT_FLAGS": "1", "P2S_JIT_T": "1"}),
    (S793, {"P2S_JIT_T": "1", "P2S_JIT_MINB": "1", "P2S_JIT_FLAGS": "1"}),
]


if os.environ.get("P2S_JIT_SWEEP"):
    from paper_1703_09619_b200 import shape_grid as _sg
    CASES = [(_sg.ALL[i][:5], o) for i, o in json.load(open(os.environ["P2S_JIT_SWEEP"]))]


def one(idx):
    import numpy as np
    import torch

    from oracle import oracle as O
    from paper_1703_09619_b200 import capi
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import blocks_close
    (nc, order, kinds, nq, basis), opts = CASES[idx]
    ctx = capi.Context(nc, order, kinds, nq, basis=basis, options=opts)
    o = O.Oracle(nc, order, kinds, nq, basis)
    alpha = o.alpha(O.ALPHA_SINE, 0.5, 3.0, 5, 0, 2)
    a = torch.from_numpy(alpha).cuda()
    M = torch.full((2, ctx.n_tot, ctx.n_tot), float("nan"), dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    I = torch.zeros((2, ctx.moments_per_elem), dtype=torch.float64, device="cuda")
    ctx.moments(a, I, 2, st)
    M2 = torch.full_like(M, float("nan"))
    ctx.contract(I, M2, ctx.n_tot, 2, st)
    torch.cuda.synchronize()
    Mo = o.fill(alpha, threads=4)
    Nt = order[0] * order[1] * order[2]
    res2 = [blocks_close(M2[e].cpu().numpy(), Mo[e], nc, Nt) for e in range(2)]
    print(json.dumps({"case": idx, "two_stage_ok": all(r[0] for r in res2), "msg": res2[0][1]}), flush=True)
    ctx.fill(a, M, ctx.n_tot, 2, st)
    torch.cuda.synchronize()
    res = [blocks_close(M[e].cpu().numpy(), Mo[e], nc, Nt) for e in range(2)]
    # speed: 2000 elements' worth of fills
    E = max(2, min(4096, int(4e9 // (8 * (ctx.n_tot ** 2 + ctx.alpha_per_elem)))))
    A = torch.empty((E, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    ctx.alpha_generate(0, 0.5, 3.0, 1, 0, E, A, st)
    MM = torch.empty((E, ctx.n_tot, ctx.n_tot), dtype=torch.float64, device="cuda")
    for _ in range(2):
        ctx.fill(A, MM, ctx.n_tot, E, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ctx.fill(A, MM, ctx.n_tot, E, st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    gbs = E * 8 * (ctx.n_tot ** 2 + ctx.alpha_per_elem) / (ms / 1e3) / 1e9
    print(json.dumps({"case": idx, "opts": opts, "ok": all(r[0] for r in res), "msg": res[0][1] or res[1][1],
                      "worst": max(r[2] for r in res), "elem_per_s": E / (ms / 1e3), "alpha+M GB/s": gbs,
                      "path": ctx.kernel_path}))


if __name__ == "__main__":
    if sys.argv[1] == "prepare":
        from paper_1703_09619_b200 import shape_grid
        r = shape_grid.prepare_all([c + (o,) for c, o in CASES])
        print(json.dumps(r, indent=1))
    elif sys.argv[1] == "run":
        for i in range(len(CASES)):
            p = subprocess.run([sys.executable, __file__, "one", str(i)], capture_output=True, text=True,
                               timeout=600)
            print(p.stdout.strip() or f"case {i} {CASES[i][1]}: rc {p.returncode} {p.stderr.strip()[-300:]}",
                  flush=True)
    else:
        one(int(sys.argv[2]))
