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
    ap.add_argument("--no-parity", action="store_true", help="skip the timed-batch parity check")
    ap.add_argument("--no-sustained", action="store_true")
    ap.add_argument("--sustained-steps", type=int, default=600)
    ap.add_argument("--no-subconfigs", action="store_true",
                    help="skip the C3 / C4 / C5 / c12 lines of the default (c2) run")
    ap.add_argument("--sub-steps", type=int, default=10)
    ap.add_argument("--options", default="",
                    help="p2s_create_ex test / tuning hooks for every context, 'KEY=VALUE;...' "
                         "(measurement sweeps; not used by the driver's runs)")
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
    # liboracle_fast.so: the oracle's source built with FMA contraction and
    # unrolling (oracle/Makefile FASTFLAGS) -- the checker build stays strict
    o = O.Oracle(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq, fast=True)
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
                         "cpu_model": cpu_model(),
                         "sample": f"~{sample} {cfg.name} elements per step (>= {secs:.0f} s of "
                                   f"moments + banded contraction, oracle/p2s_oracle.c built -O3 -mavx2 "
                                   f"-mfma -ffp-contract=fast, {threads} threads)"},
        "e2e": {"value": value, "unit": "elem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- B200 arm

SUBCONFIGS = ("c3", "c4", "c5", "c12")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def parity_of(ctx, cfg, alpha, M, picks, threads):
    """Timed-batch parity (verify.cpp:81-99 comparator, per (gi, gj) block, rtol
    1e-12): read back the picked elements' alpha and matrices from the device
    after the timed region and check them against the CPU oracle."""
    import numpy as np

    from oracle import oracle as O
    o = O.Oracle(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    a = alpha[picks].cpu().numpy()
    Mg = M[picks].cpu().numpy()
    Mo = o.fill(a, threads=threads)
    Nt = cfg.order[0] * cfg.order[1] * cfg.order[2]
    worst, ok = 0.0, True
    for i in range(len(picks)):
        for gi in range(cfg.n_comp):
            for gj in range(cfg.n_comp):
                blk = np.s_[gi * Nt:(gi + 1) * Nt, gj * Nt:(gj + 1) * Nt]
                ga, ob = np.ascontiguousarray(Mg[i][blk]), np.ascontiguousarray(Mo[i][blk])
                scale = max(np.abs(ga).max(), np.abs(ob).max(), 1e-300)
                worst = max(worst, float(np.abs(ga - ob).max() / scale))
                ok = ok and O.block_close(ga, ob, 1e-12)[0]
    return {"checked": [int(e) for e in picks], "worst_rel_to_block_max": worst, "rtol": 1e-12,
            "ok": bool(ok), "comparator": "block_close per (gi, gj) block vs oracle/p2s_oracle.c"}


def roofline_of(cfg, stages, elems_total, hbm_peak, peak_src, path):
    """Dominant kernel's algorithmic bytes per launch / its CUDA-event launch time."""
    from paper_1703_09619_b200.configs import algorithmic_counts
    counts = algorithmic_counts(cfg)
    fused = stages["n_moments"] == 0 and stages["n_contract"] > 0
    kname = ("fill_fused_kernel" if fused else
             "large_w_kernel + large_v_kernel + large_u_kernel" if path.startswith("large") else
             "contract_v2_kernel" if "contract_v2" in path else "contract_kernel")
    alg_bytes_elem = (counts["bytes_alpha"] + counts["bytes_M"]) if fused else counts["bytes_con"]
    n_con = max(1, stages["n_contract"])
    con_ms_avg = stages["ms_contract"] / n_con
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
    fp64_peak = 34.1  # builder-measured DFMA loop (tools/peaks.cu, profiles/r1_peaks.json)
    return {"kernel": kname, "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved / hbm_peak, "traffic": traffic,
            "traffic_source": ("profiles/ncu_traffic.json (ncu --set full capture of this kernel: DRAM "
                               "bytes per element x elements per launch; not measured in this run)"
                               if traffic is not None else None),
            "peak_source": peak_src, "alg_bytes_per_elem": alg_bytes_elem,
            "avg_launch_ms": con_ms_avg, "launches": n_con,
            "fp64_tflops_algorithmic": (counts["flop_mom"] + counts["flop_con"]) * elems_total /
            max(1e-9, (stages["ms_moments"] + stages["ms_contract"]) / 1e3) / 1e12,
            "fp64_peak_tflops": fp64_peak,
            "fp64_peak_source": "tools/peaks.cu DFMA loop, profiles/r1_peaks.json (MEASURED_PEAKS.json has "
                                "no FP64 entry)"}


def run_config(cfg, local, rank, E, steps, warmup, seed, sp, st, barrier, clocks=True, basis=None):
    """One config's timed fill: alpha resident, CUDA events on the launching
    stream around exactly `steps` fills; returns (ctx, alpha, M, ms, stages, clk)."""
    import torch

    from paper_1703_09619_b200 import capi
    basis = capi.BASIS_MODAL if basis is None else basis
    ctx = capi.Context(**cfg.problem(), device=local, basis=basis)
    n_tot = ctx.n_tot
    alpha = torch.empty((E, ctx.alpha_per_elem), dtype=torch.float64, device="cuda")
    ctx.alpha_generate(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, seed, rank * E, E, alpha, sp)
    M = torch.empty((E, n_tot, n_tot), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(max(3, warmup)):
        ctx.fill(alpha, M, n_tot, E, sp)
    torch.cuda.synchronize()
    ctx.set_profiling(True)
    sampler = ClockSampler(local) if clocks else None
    barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        time.sleep(0.5)  # nvidia-smi needs a moment before its first sample
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(st)
    for _ in range(steps):
        ctx.fill(alpha, M, n_tot, E, sp)
    ev1.record(st)
    torch.cuda.synchronize()
    clk = sampler.stop() if sampler else None
    barrier()
    ms = ev0.elapsed_time(ev1)
    stages = ctx.stage_times()
    ctx.set_profiling(False)
    return ctx, alpha, M, ms, stages, clk


def run_b200(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1703_09619_b200 import capi
    from paper_1703_09619_b200.configs import CONFIGS

    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    distributed = world > 1
    torch.cuda.set_device(local)
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if distributed:
            dist.barrier()

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if distributed:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    basis = capi.BASIS_CONFORMING if args.basis == "conforming" else capi.BASIS_MODAL
    total_mem = torch.cuda.get_device_properties(local).total_memory
    sizes = capi.problem_sizes(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq, basis)
    # C4 / C5 totals (1.1 TB / 4.4 TB of matrices) exceed HBM: a step fills the
    # largest batch whose alpha + M fit in half of the GPU's memory
    per_elem = 8 * (sizes.alpha_per_elem + sizes.n_tot * sizes.n_tot)
    E = args.n_elem or min(cfg.n_elem, max(1, int(0.5 * total_mem // per_elem)))
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    ctx, alpha, M, ms, stages, clk = run_config(cfg, local, rank, E, args.steps, args.warmup, args.seed, sp, st,
                                                barrier, basis=basis)
    n_tot = ctx.n_tot
    ms_max = max_over_ranks(ms)
    value = world * E * args.steps / (ms_max / 1e3)
    threads = os.cpu_count() or 1

    # ---- parity of the timed batch (the last timed step's matrices)
    parity = None
    if not args.no_parity and rank == 0:
        picks = sorted({0, E // 2, E - 1})
        parity = parity_of(ctx, cfg, alpha, M, picks, threads)

    # ---- sustained run: the same fill over >= 600 steps (power-capped clocks)
    sustained = None
    if not args.no_sustained and args.sustained_steps > 0:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        sampler = ClockSampler(local)
        barrier()
        torch.cuda.synchronize()
        sampler.start()
        time.sleep(0.5)
        ev0.record(st)
        for _ in range(args.sustained_steps):
            ctx.fill(alpha, M, n_tot, E, sp)
        ev1.record(st)
        torch.cuda.synchronize()
        sclk = sampler.stop()
        sms = max_over_ranks(ev0.elapsed_time(ev1))
        sustained = {"steps": args.sustained_steps, "value": world * E * args.sustained_steps / (sms / 1e3),
                     "ms_per_step": sms / args.sustained_steps, "clocks": sclk,
                     "note": "same fill, >= 600 back-to-back steps: the 1000 W power cap sets the SM clock"}

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
        dt = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": world * E2 * reps / dt, "unit": "elem/s",
               "h2d_bytes_per_step": E2 * ctx.alpha_per_elem * 8,
               "d2h_bytes_per_step": E2 * n_tot * n_tot * 8,
               "elements_per_step": E2, "timing": "wall clock around p2s_fill_host (pinned host buffers)"}
        del h_alpha, h_M

    if rank != 0:
        del alpha, M
        ctx.close()
        if distributed:
            dist.destroy_process_group()
        return

    # ---- ablation: the direct-quadrature fill the paper's scheme replaces
    ablation = None
    if not args.no_ablation:
        dctx = capi.DirectContext(**cfg.problem(), device=local, basis=basis)
        fma_elem = ctx.n_pairs * len(cfg.kinds) * (cfg.nq[0] * cfg.nq[1] * cfg.nq[2]) * \
            (n_tot // cfg.n_comp) ** 2
        NA = int(max(1, min(E, 2.25e12 // fma_elem)))
        dctx.fill(alpha, M, n_tot, NA, sp)  # warm-up (cuBLAS heuristics)
        torch.cuda.synchronize()
        reps = 3
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
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

    # ---- fill straight from element geometry
    geometry = None
    if cfg.alpha_kind == 1 and not args.no_ablation:  # P2S_ALPHA_JACOBIAN
        geom = torch.empty((E, ctx.GEOM_DOUBLES), dtype=torch.float64, device="cuda")
        ctx.geometry_generate(cfg.alpha_lo, cfg.alpha_hi, args.seed, rank * E, E, geom, sp)
        ctx.fill_geometry(geom, M, n_tot, E, sp)
        torch.cuda.synchronize()
        greps = max(3, min(args.steps, 20))
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(st)
        for _ in range(greps):
            ctx.fill_geometry(geom, M, n_tot, E, sp)
        ev1.record(st)
        torch.cuda.synchronize()
        gms = ev0.elapsed_time(ev1) / greps
        geometry = {"value": E / (gms / 1e3), "unit": "elem/s", "steps": greps,
                    "hbm_bytes_per_elem": n_tot * n_tot * 8 + ctx.GEOM_DOUBLES * 8,
                    "method": "p2s_fill_geometry: alpha_geometry_kernel -> L2 double buffer -> "
                              "fill_fused_kernel, CUDA events (synchronous: Jacobian check)"}
        del geom

    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)" if "hbm_gbs" in peaks else "fallback 6650 GB/s"
    path = ctx.kernel_path
    roof = roofline_of(cfg, stages, E * args.steps, hbm_peak, peak_src, path)
    fused = roof["kernel"] == "fill_fused_kernel"
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
        "roofline": roof,
        "kernel_path": path,
    }
    if parity:
        line["parity"] = parity
    if sustained:
        line["sustained"] = sustained
    if e2e:
        line["e2e"] = e2e
    if ablation:
        line["ablation"] = ablation
    if geometry:
        line["geometry_fill"] = geometry
    del alpha, M
    ctx.close()
    torch.cuda.empty_cache()

    # ---- the other BASELINE configs (and the generated-module c12 shape), each
    # timed the same way on this GPU: value, roofline of its dominant kernel,
    # kernel path and timed-batch parity
    if args.config == "c2" and not args.no_subconfigs:
        subs = {}
        for name in SUBCONFIGS:
            scfg = CONFIGS[name]
            try:
                sz = capi.problem_sizes(scfg.n_comp, scfg.order, list(scfg.kinds), scfg.nq)
                pe = 8 * (sz.alpha_per_elem + sz.n_tot * sz.n_tot)
                Es = min(scfg.n_elem, max(1, int(0.4 * total_mem // pe)))
                sctx, sa, sM, sms, sst, sclk = run_config(scfg, local, 0, Es, args.sub_steps, 3, args.seed, sp, st,
                                                          lambda: None)
                sroof = roofline_of(scfg, sst, Es * args.sub_steps, hbm_peak, peak_src, sctx.kernel_path)
                sub = {"value": Es * args.sub_steps / (sms / 1e3), "unit": "elem/s", "elements_per_step": Es,
                       "steps": args.sub_steps, "ms_per_step": sms / args.sub_steps,
                       "order": list(scfg.order), "n_comp": scfg.n_comp, "nq": list(scfg.nq),
                       "roofline": {k: sroof[k] for k in ("kernel", "achieved", "peak", "frac", "traffic",
                                                          "avg_launch_ms", "launches", "alg_bytes_per_elem",
                                                          "fp64_tflops_algorithmic")},
                       "kernel_path": sctx.kernel_path, "clocks": sclk,
                       "gpu_launches": sst["n_moments"] + sst["n_contract"]}
                if not args.no_parity:
                    picks = sorted({0, Es - 1}) if sz.n_tot >= 2048 else sorted({0, Es // 2, Es - 1})
                    sub["parity"] = parity_of(sctx, scfg, sa, sM, picks, threads)
                del sa, sM
                sctx.close()
            except Exception as e:  # report, keep the headline
                sub = {"error": f"{type(e).__name__}: {e}"[:400]}
            torch.cuda.empty_cache()
            subs[name] = sub
        line["configs"] = subs

    if not args.no_cpu_baseline:
        rate, n, dt = cpu_baseline(cfg, args.cpu_seconds, args.seed, threads)
        rate1, n1, dt1 = cpu_baseline(cfg, max(2.0, args.cpu_seconds / 4), args.seed, 1, batch=4)
        line["cpu_baseline"] = {"value": rate, "unit": "elem/s", "cores": threads, "kind": "port",
                                "cpu_model": cpu_model(), "value_1thread": rate1,
                                "sample": f"{n} {cfg.name} elements, {dt:.1f} s (moments + banded "
                                          f"contraction, oracle/p2s_oracle.c built -O3 -mavx2 -mfma "
                                          f"-ffp-contract=fast, {threads} threads); 1 thread: "
                                          f"{n1} elements, {dt1:.1f} s"}
        if args.config == "c2" and not args.no_subconfigs:
            line["cpu_baseline"]["c5_direct_ablation"] = c5_direct_sample(args.seed)
        ref2d = reference_2d_context(threads)
        if ref2d:
            line["cpu_baseline"]["reference_2d_bench_fill"] = ref2d
    print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


def c5_direct_sample(seed):
    """BASELINE configs[4]'s ablation on the CPU: the reference algorithm's
    direct full 3-D quadrature fill (assemble_direct_element, assembly.cpp:142-274,
    restated in oracle/p2s_oracle.c) on one C5 element, timed on the u-test row
    m1 = N-1 only (1 of the N(N+1)/2 canonical (m1, m2) pairs, same work per pair)
    and extrapolated -- labelled as such."""
    from oracle import oracle as O
    from paper_1703_09619_b200.configs import CONFIGS
    cfg = CONFIGS["c5"]
    o = O.Oracle(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    a = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, seed, 0, 1)
    N = cfg.order[0]
    secs, cov, tot = O.direct_sample_seconds(o, a[0], N - 1, N)
    per = secs * tot / cov
    return {"seconds_per_element_1thread": per, "elem_per_s_1thread": 1.0 / per,
            "extrapolated": True,
            "sample": f"1 element, u-test row m1 = {N - 1}: {cov} of {tot} canonical (m1, m2) pairs in "
                      f"{secs:.2f} s, x {tot / cov:.0f}"}


def reference_2d_context(threads):
    """The reference's own 2-D bench_fill (bench.cpp:75-140) on its Fig.-1 domain
    at M = N = 8 and 16, built from its sources (oracle/refbuild/ref_bench.cpp)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    if not os.path.exists(exe):
        return None
    try:
        r = subprocess.run([exe, str(threads), "3", "8", "16"], capture_output=True, text=True, timeout=120)
        out = json.loads(r.stdout)
        out["note"] = "reference 2-D Chebyshev fill (16 curved order-4 quadrilaterals), context only"
        return out
    except Exception as e:
        return {"error": str(e)[:200]}


def main():
    args = parse()
    if args.options:
        from paper_1703_09619_b200 import capi
        for kv in args.options.split(";"):
            if kv.strip():
                k, _, v = kv.partition("=")
                capi.DEFAULT_OPTIONS[k.strip()] = v.strip() or "1"
    from paper_1703_09619_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_b200(args, cfg)


if __name__ == "__main__":
    main()
