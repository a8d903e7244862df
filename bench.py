#!/usr/bin/env python
"""Benchmark: product-to-sum element fill, element matrices/s (FP64) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

One step = one pass of the fill (moment kernel + contraction kernel, every
element matrix written to HBM) over one batch of the workload's elements with
alpha already resident in HBM.  Workload: BASELINE.json configs[1] (C2: 4096
elements, 3-component, order 6, N_s = 2, 14^3 points) unless --config says
otherwise.  Under torchrun every rank fills its own element range (weak
scaling, no collective on the data path); the time is the max over ranks.

--impl reference times the CPU oracle port of the reference algorithm
(oracle/, the reference itself only implements the 2-D Chebyshev case) on the
host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n-elem", type=int, default=0, help="override elements per rank")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="seconds of CPU work per CPU-baseline sample / reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--basis", default="modal", choices=["modal", "conforming"],
                    help="element basis (conforming = the reference's conforming change of basis)")
    ap.add_argument("--no-ablation", action="store_true",
                    help="skip the direct-quadrature ablation (p2s_direct_fill, rank 0)")
    ap.add_argument("--seed", type=int, default=20170328)
    return ap.parse_args()


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
                 "clocks.mem",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, pw, mem, reasons = [], [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx.append(float(parts[1]))
                    pw.append(float(parts[2]))
                    if len(parts) > 8:
                        mem.append(float(parts[8]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[4:8]):
                    if v.lower() == "active":
                        reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "sm_mhz_min": min(sm) if sm else None,
                "power_w_median": statistics.median(pw) if pw else None,
                "mem_mhz_median": statistics.median(mem) if mem else None}


# ---------------------------------------------------------------- CPU oracle baseline

def cpu_baseline(cfg, seconds: float, seed: int, threads: int, batch: int = 0, e0: int = 0):
    """Oracle fill (moments + banded contraction, oracle/p2s_oracle.c) over
    consecutive batches of the workload's elements until `seconds` of CPU work
    are done; the output buffer is one batch, reused.  Returns (elem/s,
    elements, seconds)."""
    import numpy as np

    from oracle import oracle as O
    o = O.Oracle(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    batch = batch or max(threads, min(256, int(2e9 // (8 * o.n_tot * o.n_tot))))
    out = np.empty((batch, o.n_tot, o.n_tot))
    done, elapsed = 0, 0.0
    while done == 0 or elapsed < seconds:
        alpha = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, seed, e0 + done, batch)
        t0 = time.perf_counter()
        o.fill(alpha, threads=threads, out=out)
        elapsed += time.perf_counter() - t0
        done += batch
    return done / elapsed, done, elapsed


def run_reference(args, cfg):
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    # bounded: the whole reference run stays within ~2 minutes of CPU work
    secs = min(args.cpu_seconds, 120.0 / max(1, args.steps))
    for _ in range(max(0, args.warmup)):
        cpu_baseline(cfg, 0.0, args.seed, threads)
    n_total, t_total = 0, 0.0
    for i in range(args.steps):
        _, n, dt = cpu_baseline(cfg, secs, args.seed, threads, e0=n_total)
        n_total += n
        t_total += dt
    value = n_total / t_total
    sample = n_total // max(1, args.steps)
    line = {
        "impl": "reference", "metric": "element matrices/s (FP64)", "value": value,
        "unit": "elem/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_total / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded alpha, BASELINE.json shapes)",
        "config": {"workload": cfg.name, "n_comp": cfg.n_comp, "order": list(cfg.order),
                   "n_terms": len(cfg.kinds), "nq": list(cfg.nq), "elements_per_step": sample},
        "cpu_baseline": {"value": value, "unit": "elem/s", "cores": threads, "kind": "port",
                         "sample": f"~{sample} {cfg.name} elements per step (>= {secs:.0f} s of "
                                   f"moments + banded contraction, oracle/p2s_oracle.c, "
                                   f"{threads} threads)"},
        "e2e": {"value": value, "unit": "elem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- B200 arm

def run_b200(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1703_09619_b200 import capi
    from paper_1703_09619_b200.configs import algorithmic_counts

    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    distributed = world > 1
    torch.cuda.set_device(local)
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    basis = capi.BASIS_CONFORMING if args.basis == "conforming" else capi.BASIS_MODAL
    ctx = capi.Context(**cfg.problem(), device=local, basis=basis)
    # C4 / C5 totals (1.1 TB / 4.4 TB of matrices) exceed HBM: a step fills the
    # largest batch whose alpha + M fit in half of the GPU's memory
    per_elem = 8 * (ctx.alpha_per_elem + ctx.n_tot * ctx.n_tot)
    fit = max(1, int(0.5 * torch.cuda.get_device_properties(local).total_memory // per_elem))
    E = args.n_elem or min(cfg.n_elem, fit)
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    n_tot = ctx.n_tot
    alpha = torch.empty((E, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    ctx.alpha_generate(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, args.seed, rank * E, E, alpha, sp)
    M = torch.empty((E, n_tot, n_tot), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()

    def barrier():
        if distributed:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        ctx.fill(alpha, M, n_tot, E, sp)
    torch.cuda.synchronize()

    ctx.set_profiling(True)
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.5)  # nvidia-smi needs a moment before its first sample
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(st)
    for _ in range(args.steps):
        ctx.fill(alpha, M, n_tot, E, sp)
    ev1.record(st)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier()
    ms = ev0.elapsed_time(ev1)
    stages = ctx.stage_times()
    ctx.set_profiling(False)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * E * args.steps / (ms_max / 1e3)

    # checksum outside the timed region (guards against skipped work)
    chk = float(M[:, :8, :8].abs().sum().item())

    # ---- e2e through the host-buffer entry point (pinned buffers)
    e2e = None
    if not args.no_e2e:
        E2 = min(E, 1024)
        h_alpha = torch.empty((E2, ctx.alpha_per_elem), dtype=torch.float64, pin_memory=True)
        h_alpha.copy_(alpha[:E2])
        h_M = torch.empty((E2, n_tot, n_tot), dtype=torch.float64, pin_memory=True)
        ctx.fill_host(h_alpha, h_M, n_tot, E2)  # warm-up
        reps = 3
        barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            ctx.fill_host(h_alpha, h_M, n_tot, E2)
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        if distributed:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        e2e = {"value": world * E2 * reps / dt, "unit": "elem/s",
               "h2d_bytes_per_step": E2 * ctx.alpha_per_elem * 8,
               "d2h_bytes_per_step": E2 * n_tot * n_tot * 8,
               "elements_per_step": E2, "timing": "wall clock around p2s_fill_host (pinned host buffers)"}
        del h_alpha, h_M

    if rank != 0:
        if distributed:
            dist.destroy_process_group()
        return

    # ---- ablation: the direct-quadrature fill the paper's scheme replaces
    # (p2s_direct_fill: one FP64 DGEMM per element, pair and term on the tensor
    # cores), same alpha, outside the timed region
    ablation = None
    if not args.no_ablation:
        dctx = capi.DirectContext(**cfg.problem(), device=local, basis=basis)
        fma_elem = ctx.n_pairs * len(cfg.kinds) * (cfg.nq[0] * cfg.nq[1] * cfg.nq[2]) * \
            (n_tot // cfg.n_comp) ** 2
        NA = int(max(1, min(E, 2.25e12 // fma_elem)))
        dctx.fill(alpha, M, n_tot, NA, sp)  # warm-up (cuBLAS heuristics)
        torch.cuda.synchronize()
        reps = 3
        ev0.record(st)
        for _ in range(reps):
            dctx.fill(alpha, M, n_tot, NA, sp)
        ev1.record(st)
        torch.cuda.synchronize()
        dms = ev0.elapsed_time(ev1) / reps
        drate = NA / (dms / 1e3)
        ablation = {"direct_elem_per_s": drate, "elements": NA, "ms_per_batch": dms,
                    "direct_tflops": 2 * fma_elem * NA / (dms / 1e3) / 1e12,
                    "p2s_over_direct": (value / world) / drate,
                    "method": "p2s_direct_fill: W = diag(w alpha) B_trial, cuBLAS DGEMM "
                              "B_test^T W per (element, pair, term), CUDA events"}
        dctx.close()

    # ---- fill straight from element geometry: alpha produced
    # on the device into an L2-resident double buffer, so HBM carries only the
    # 28-double geometry records and M; reported beside the alpha-resident headline
    geometry = None
    if cfg.alpha_kind == 1 and not args.no_ablation:  # P2S_ALPHA_JACOBIAN
        geom = torch.empty((E, ctx.GEOM_DOUBLES), dtype=torch.float64, device="cuda")
        ctx.geometry_generate(cfg.alpha_lo, cfg.alpha_hi, args.seed, rank * E, E, geom, sp)
        ctx.fill_geometry(geom, M, n_tot, E, sp)
        torch.cuda.synchronize()
        greps = max(3, min(args.steps, 20))
        ev0.record(st)
        for _ in range(greps):
            ctx.fill_geometry(geom, M, n_tot, E, sp)
        ev1.record(st)
        torch.cuda.synchronize()
        gms = ev0.elapsed_time(ev1) / greps
        geometry = {"value": E / (gms / 1e3), "unit": "elem/s", "steps": greps,
                    "hbm_bytes_per_elem": n_tot * n_tot * 8 + ctx.GEOM_DOUBLES * 8,
                    "method": "p2s_fill_geometry: alpha_geometry_kernel -> L2 double buffer -> "
                              "fill_fused_kernel, CUDA events"}
        del geom

    counts = algorithmic_counts(cfg)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)" if "hbm_gbs" in peaks else "fallback 6650 GB/s"
    # dominant kernel: the fused fill kernel (alpha read + M write) when the
    # shape has one, else the contraction kernel (I read + M write)
    fused = stages["n_moments"] == 0 and stages["n_contract"] > 0
    path = ctx.kernel_path
    kname = ("fill_fused_kernel" if fused else
             "large_w_kernel + large_v_kernel + large_u_kernel" if path.startswith("large") else
             "contract_v2_kernel" if "contract_v2" in path else "contract_kernel")
    alg_bytes_elem = (counts["bytes_alpha"] + counts["bytes_M"]) if fused else counts["bytes_con"]
    n_con = max(1, stages["n_contract"])
    con_ms_avg = stages["ms_contract"] / n_con
    elems_total = E * args.steps
    bytes_per_launch = alg_bytes_elem * elems_total / n_con
    achieved = bytes_per_launch / (con_ms_avg / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(f"{cfg.name}:{kname}")
            if tr:
                traffic = tr["dram_bytes_per_elem"] * bytes_per_launch / alg_bytes_elem
    except Exception:
        pass
    fp64_peak = 34.1  # tools/peaks.cu DFMA loop on this pool's B200 (profiles/r1_peaks.json)
    line = {
        "metric": "element matrices/s (FP64)",
        "value": value,
        "unit": "elem/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": ms_max / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded alpha on device, BASELINE.json shapes)",
        "config": {"workload": cfg.name, "n_comp": cfg.n_comp, "order": list(cfg.order),
                   "kinds": ["PP/DD/DP/PD"[3 * k:3 * k + 2] if isinstance(k, int) else str(k)
                             for k in cfg.kinds],
                   "n_terms": len(cfg.kinds), "nq": list(cfg.nq), "elements_per_rank": E,
                   "basis": args.basis,
                   "n_tot": n_tot, "parallelism": f"element-partitioned x{world}, no collective",
                   "l2": f"outputs {E * n_tot * n_tot * 8 / 1e9:.1f} GB per step >> 126 MB L2"},
        "clocks": clk,
        "gpu_launches": stages["n_moments"] + stages["n_contract"],
        "stage_ms_per_step": {"moments": stages["ms_moments"] / args.steps,
                              ("fused_fill" if fused else "contract"): stages["ms_contract"] / args.steps},
        "roofline": {"kernel": kname, "bound": "hbm", "achieved": achieved,
                     "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_elem": alg_bytes_elem,
                     "avg_launch_ms": con_ms_avg, "launches": n_con,
                     "fp64_tflops_executed": (counts["flop_mom"] / 2 + counts["flop_con"]) *
                     elems_total / max(1e-9, (stages["ms_moments"] + stages["ms_contract"]) / 1e3) / 1e12,
                     "fp64_peak_tflops": fp64_peak},
        "kernel_path": ctx.kernel_path,
        "checksum": chk,
    }
    if e2e:
        line["e2e"] = e2e
    if ablation:
        line["ablation"] = ablation
    if geometry:
        line["geometry_fill"] = geometry
    if not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, n, dt = cpu_baseline(cfg, args.cpu_seconds, args.seed, threads)
        line["cpu_baseline"] = {"value": rate, "unit": "elem/s", "cores": threads, "kind": "port",
                                "sample": f"{n} {cfg.name} elements, {dt:.1f} s (moments + banded "
                                          f"contraction, oracle/p2s_oracle.c, {threads} threads)"}
    print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


def main():
    args = parse()
    from paper_1703_09619_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_b200(args, cfg)


if __name__ == "__main__":
    main()
