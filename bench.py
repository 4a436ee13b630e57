#!/usr/bin/env python
"""Headline benchmark: Stokes ALM voxel-iterations/s at 256^3 fp64 (BASELINE.json).

Workload (BASELINE cfg 3): one 256^3 random polydisperse sphere packing per GPU
(SURVEY §8d generator, seed = rank // 3), load case g_p = e_{rank % 3}, the
reference's default (adaptive) penalties, eps = 1e-5.  A "step" is one ADMM
iteration of the device loop (stokes.py:375-417).  Multi-GPU is the ensemble
sharding of §8e: one independent cell per rank, no data-path collective
(scaling "weak"); the time is the max over ranks of CUDA-event durations.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--impl reference` times the CPU restatement of the reference (oracle/, the
reference being pure numpy/scipy for 3D) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Stokes ALM voxel-iters/s at 256³ fp64, 1/2/4/8 GPU; % HBM roofline vs CPU ref"
UNIT = "voxel-iter/s"
B_ALG_ITER = 417.0  # canonical algorithmic bytes per Stokes voxel-iteration
FALLBACK_HBM = 6650.0


def peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def headline_config(n, world):
    """The workload both arms print (identical dicts, so the driver can match them)."""
    return {"workload": f"stokes_admm_random_packing_{n}^3", "grid": [n, n, n], "cells": world,
            "load_cases": "e_{rank%3}", "packing_seed": "rank//3",
            "penalties": "reference default (adaptive)", "eps": 1e-5,
            "parallelism": f"ensemble{world} (one independent cell per GPU)",
            "l2": "inputs larger than L2 (~25 x 128 MiB fields per cell), no flush"}


def host_cpu():
    """lscpu model, logical cores and the POREFLOW_THREADS cap."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"lscpu_model": model, "logical_cpus": os.cpu_count(),
            "POREFLOW_THREADS": os.environ.get("POREFLOW_THREADS") or None}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling around the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = Path(tempfile.mkstemp(prefix="clocks_", suffix=".csv")[1])

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def stop(self, t0, t1):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 10:
                continue
            rows.append(parts)
        self.path.unlink(missing_ok=True)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        # keep the samples taken while the timed region ran (by sample order: the
        # sampler started before warm-up; use the last samples covering t1 - t0)
        n_keep = max(1, int((t1 - t0) / 0.1) + 1)
        sel = rows[-(n_keep + 2):-1] if len(rows) > n_keep + 2 else rows
        sm = sorted(float(r[2]) for r in sel if r[2].replace(".", "").isdigit())
        smax = max((float(r[3]) for r in sel if r[3].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in sel for k in range(4) if r[6 + k].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(sel)}


# ---------------------------------------------------------------- reference (CPU) arm
def cpu_stokes_rate(n, seed, g, budget_s, max_iters):
    """Oracle (CPU restatement of the reference, numpy + scipy.fft, all host
    threads) on the same cell: voxel-iters/s over the loop alone."""
    import numpy as np

    from oracle import poreflow_oracle as O
    import paper_2312_15554_b200 as pf

    ind = pf.random_packing_geometry(n, seed=seed)
    tm = {}
    O.solve_stokes(ind.values, g, 1e-5, 1e-5, max_iter=1, timer=tm)  # warm-up + speed estimate
    k = int(max(1, min(max_iters, budget_s / max(tm["loop_s"], 1e-3))))
    tm = {}
    O.solve_stokes(ind.values, g, 1e-5, 1e-5, max_iter=k, timer=tm)
    del np
    return n ** 3 * k / tm["loop_s"], k, tm["loop_s"]


def run_reference(args):
    rank, _, _ = dist_env()
    if rank != 0:
        return 0
    n = args.n
    rate, k, secs = cpu_stokes_rate(n, 0, (1.0, 0.0, 0.0), args.cpu_budget, max(1, args.steps))
    cores = int(os.environ.get("POREFLOW_THREADS") or os.cpu_count())
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": k, "warmup": 1, "ms_per_step": 1e3 * secs / k, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": headline_config(n, args.gpus),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{k} ADMM iteration(s) of the seed-0 e1 {n}^3 cell after 1 warm-up iteration "
                                   f"(loop time only; numpy + scipy.fft workers={cores})", **host_cpu()},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm
STAGES = ("S1_spectral", "Z2D_cufft", "S3_local", "finalize", "S4_form_r", "D2Z_cufft")
FUSED_STAGES = ("PK_axis0_spectral", "MI_axis1_inverse", "RS_rows_local", "finalize", "RSF_rows_fix",
                "MF_axis1_forward")


def stage_bytes(n_real, n_half, d=3):
    """Algorithmic bytes per launch of each stage."""
    w = 8
    return {
        "S1_spectral": n_half * 16 * (1 + d + 1) + n_half * 16 * (d + 1 + 1),  # Q,R,Dprev in; U,Q,D out
        "Z2D_cufft": d * (n_half * 16 + n_real * w),
        "S3_local": n_real * (w * (5 * d) + 1) + n_real * w * (4 * d),  # 5d words + H in; 4d words out
        "finalize": 0,
        "S4_form_r": n_real * w * (2 * d) + n_real * w * d,
        "D2Z_cufft": d * (n_real * w + n_half * 16),
    }


def stage_bytes_fused(n_real, n_half, n_solid=None):
    """Algorithmic bytes per launch of the fused pipeline's passes.
    With solid-only storage (n_solid given) RS streams u (r+w) on every voxel and
    u~, a, lam (r+w) only on solid voxels."""
    hw = n_half * 16  # one half-spectrum component
    rs_state = 24 * 8 * n_real if n_solid is None else 6 * 8 * n_real + 18 * 8 * n_solid
    return {
        "PK_axis0_spectral": 10 * hw,          # Y(3) Q D in; Y(3) Q D out
        "MI_axis1_inverse": 6 * hw,            # Y(3) in; X(3) out
        "RS_rows_local": 6 * hw + rs_state + n_real,  # X(3) in, X(3) out; state; H
        "finalize": 0,
        "RSF_rows_fix": 0,                     # no-op unless residual balancing changed b
        "MF_axis1_forward": 6 * hw,            # X(3) in; Y(3) out
    }


def run_ours(args):
    import ctypes

    import numpy as np
    import torch

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    import paper_2312_15554_b200 as pf
    from paper_2312_15554_b200 import _native as N

    n = args.n
    seed, case = rank // 3, rank % 3
    g = [0.0, 0.0, 0.0]
    g[case] = 1.0
    ind = pf.random_packing_geometry(n, seed=seed)
    cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=tuple(g), max_iter=10**7)
    pen = pf.PenaltyParams()
    prof_iters = 3
    rows = args.warmup + args.steps + prof_iters + 1
    state = pf.DeviceAdmmState.zeros(ind.grid, dev)
    solver = pf.StokesSolver(ind, cfg, pen, state, dev, history_rows=rows, cold=True)
    solver.begin()
    solver.iterate(args.warmup, poll=False)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = ClockSampler(local_rank).start() if rank == 0 else None
    time.sleep(0.3 if clocks else 0.0)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    start.record()
    solver.iterate(args.steps, poll=False)
    stop.record()
    torch.cuda.synchronize()
    t1 = time.time()
    ms = start.elapsed_time(stop)
    if dist:
        dist.barrier()
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clk = clocks.stop(t0, t1) if clocks else None
    # per-stage launch times on the same stream (CUDA events; no graph)
    stage_ms = (ctypes.c_double * 6)()
    N.check(N.load().pf_stokes_profile(solver.plan.handle, prof_iters, stage_ms))
    pipeline = solver.pipeline
    res = solver.end()
    assert not res.converged and res.iterations == args.warmup + args.steps + prof_iters, (
        "bench cell converged inside the timed window; raise the grid size or lower eps")
    value = world * n ** 3 * args.steps / (ms / 1e3)

    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peak, peak_src = peak_hbm()
    n_real, n_half = n ** 3, n * n * (n // 2 + 1)
    fused = pipeline.startswith("fused")
    names = FUSED_STAGES if fused else STAGES
    sb = stage_bytes(n_real, n_half)
    if fused:
        n_solid = int(np.count_nonzero(ind.values))
        sb = stage_bytes_fused(n_real, n_half, n_solid if pipeline == "fused-compact" else None)
    stages = {}
    for k, name in enumerate(names):
        if name == "-":
            continue
        t_ms = float(stage_ms[k])
        stages[name] = {"ms": t_ms, "alg_bytes": sb[name],
                        "GB_s": (sb[name] / (t_ms * 1e-3) / 1e9) if t_ms > 0 and sb[name] else None}
    ours = [s for s in stages if "cufft" not in s and s not in ("finalize", "RSF_rows_fix")]
    dom = max(ours, key=lambda s: stages[s]["ms"])
    traffic, traffic_src = None, None
    tfile = ROOT / "profiles" / "traffic_per_launch.json"
    if tfile.exists():  # the ncu capture this figure comes from is named with its commit
        try:
            ent = json.loads(tfile.read_text()).get(pipeline, {})
            traffic = ent.get(dom)
            traffic_src = f"{ent.get('_capture')} @ {ent.get('_commit')}" if traffic is not None else None
        except Exception:
            traffic = None
    achieved = stages[dom]["GB_s"]
    pipe_b = sum(v for v in sb.values() if v) / n_real
    iter_ms_profile = sum(float(stage_ms[k]) for k in range(6))

    # end-to-end through the public numpy API: the host's bit-packed indicator in
    # (1 bit per voxel, numpy.packbits order, PackedIndicator: the form a micro-CT
    # segmentation is stored in), host state and history out
    e2e_iters = args.steps
    bits_host = np.packbits(np.asarray(ind.values, dtype=np.uint8).ravel())
    # untimed warm-up call (pinned staging buffers, plan cache), like the W warm-up steps
    pf.solve_stokes(pf.PackedIndicator(pf.UnitCellGrid((n, n, n)), bits_host),
                    pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=tuple(g), max_iter=3), pen)
    torch.cuda.synchronize()
    te0 = time.perf_counter()
    e2e_ind = pf.PackedIndicator(pf.UnitCellGrid((n, n, n)), bits_host)  # host bytes in (validated)
    st_h, rep_h = pf.solve_stokes(e2e_ind, pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=tuple(g),
                                                                          max_iter=e2e_iters), pen)
    torch.cuda.synchronize()
    te1 = time.perf_counter()
    assert rep_h.iterations == e2e_iters
    e2e_value = n ** 3 * e2e_iters / (te1 - te0)
    h2d = bits_host.nbytes  # packed indicator (the zero initial state is created on the device)
    d2h = (4 * 3 + 1) * 8 * n ** 3 + e2e_iters * 15 * 8
    del st_h

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rate, k_cpu, secs = cpu_stokes_rate(n, seed, tuple(g), args.cpu_budget, 100)
        cpu = {"value": rate, "unit": UNIT, "cores": int(os.environ.get("POREFLOW_THREADS") or os.cpu_count()),
               "kind": "port",
               "sample": f"{k_cpu} ADMM iteration(s) of the same {n}^3 cell on the host (loop time only, "
                         f"{secs:.1f} s; numpy + scipy.fft, all host threads)", **host_cpu()}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": headline_config(n, world),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "traffic_source": traffic_src, "peak_source": peak_src},
        "iteration_roofline": {"alg_bytes_per_voxel_iter": B_ALG_ITER,
                               "achieved_GB_s": B_ALG_ITER * value / world / 1e9,
                               "frac": B_ALG_ITER * value / world / 1e9 / peak,
                               # bytes this pipeline actually has to move (solid-only storage moves fewer)
                               "pipeline_bytes_per_voxel_iter": pipe_b,
                               "pipeline_frac": pipe_b * value / world / 1e9 / peak},
        "stages": stages, "stage_profile_ms_per_iter": iter_ms_profile,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d / e2e_iters,
                "d2h_bytes_per_step": d2h / e2e_iters, "iterations": e2e_iters,
                "api": "paper_2312_15554_b200.solve_stokes (PackedIndicator host bytes in, numpy AdmmState out)"},
        "pipeline": pipeline,
        "gpu_launches": (6 if fused else 4) * args.steps,
        "library_launches_note": ("none: all transforms are in-kernel" if fused
                                  else "plus 2 cuFFT executions (batch 3) per iteration"),
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_transport_workload(args):
    """Secondary line (not the headline): transport voxel-iters/s, BASELINE cfg-2 cell
    (n^3 sphere array, r = 0.25) under its unit flow; Pe = 10, a0 = 0.55 (cfg 2's
    Pe = 50 trips the reference's divergence guard on this cell) and eps = 1e-12 so
    the timed window never terminates early."""
    import torch

    import paper_2312_15554_b200 as pf

    dev = torch.device("cuda", 0)
    n = args.n
    ind = pf.make_model_geometry(pf.UnitCellGrid((n, n, n)), radius=0.25)
    pen = pf.PenaltyParams(alpha=100.0, beta=100.0, b=100.0, adaptive=False)
    st, _ = pf.solve_stokes_device(ind, pf.StokesConfig.with_tolerance(1e-4, pressure_gradient=(1.0, 0.0, 0.0),
                                                                       max_iter=200), pen)
    z = lambda *s: torch.zeros(s, dtype=torch.float64, device=dev)  # noqa: E731
    C = max(1, args.tcells)
    solvers, streams = [], [torch.cuda.Stream(dev) for _ in range(C)]
    for k in range(C):  # cfg 2's load cases: composition gradients e_1, e_2, e_3 under one flow
        g = [0.0, 0.0, 0.0]
        g[k % 3] = 1.0
        cfg = pf.TransportConfig(pe=10.0, a0=0.55, eps=1e-12, composition_gradient=tuple(g), max_iter=10**6)
        with torch.cuda.stream(streams[k]):
            state = pf.DeviceTransportState(z(n, n, n), z(3, n, n, n))
            s = pf.TransportSolver(ind, st.u, cfg, state, dev, history_rows=args.warmup + args.steps + 4,
                                   plan_slot=k)
            s.begin()
            s.iterate(args.warmup, poll=False)
        solvers.append(s)
    torch.cuda.synchronize()
    main = torch.cuda.current_stream(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for st_k in streams:
        st_k.wait_stream(main)
    done = 0
    while done < args.steps:
        k = min(8, args.steps - done)
        for j, s in enumerate(solvers):
            with torch.cuda.stream(streams[j]):
                s.iterate(k, poll=False)
        done += k
    for st_k in streams:
        main.wait_stream(st_k)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    solver = solvers[0]
    import ctypes

    from paper_2312_15554_b200 import _native as N

    sm = (ctypes.c_double * 5)()
    prof = 3 if solver.pipeline == "fused" else 0  # stage events exist for the fused passes only
    if prof:
        N.check(N.load().pf_transport_profile(solver.plan.handle, prof, sm))
    res = solver.end()
    assert res.iterations == args.warmup + args.steps + prof and not res.diverged and not res.converged
    for j, s in enumerate(solvers[1:], 1):
        with torch.cuda.stream(streams[j]):
            r = s.end()
        assert r.iterations == args.warmup + args.steps and not r.diverged
    peak, _ = peak_hbm()
    value = C * n ** 3 * args.steps / (ms / 1e3)
    print(json.dumps({"metric": "transport voxel-iters/s (secondary)", "value": value, "unit": UNIT,
                      "ms_per_step": ms / args.steps, "steps": args.steps, "warmup": args.warmup,
                      "pipeline": solver.pipeline, "dtype": "f64",
                      "config": {"workload": f"transport_sphere_{n}^3", "pe": 10.0, "a0": 0.55,
                                 "concurrent_solves": C},
                      "roofline_201B": {"alg_bytes_per_voxel_iter": 201, "achieved_GB_s": 201 * value / 1e9,
                                        "frac": 201 * value / 1e9 / peak},
                      "stages_ms": dict(zip(("PK_T", "MI_T", "RS_T", "finalize", "MF_T"), list(sm)))}),
          flush=True)
    return 0


def run_pipeline_workload(args):
    """Secondary line: BASELINE cfg 2 as the reference's ``cli.run`` computes it —
    the n^3 sphere array (r = 0.25): d unit Stokes solves (reference default
    adaptive penalties, eps 1e-5, to convergence), the d transport solves under
    the e_1 flow (Pe = 10, a0 = 0.55 — cfg 2's Pe = 50 trips the reference's own
    divergence guard on this cell — eps 1e-5), K* and D*; host indicator in,
    tensors out, wall clock.  The CPU figure is EXTRAPOLATED: the oracle's
    per-iteration rates on a bounded sample of the same cell times the GPU's
    iteration counts."""
    import torch

    import paper_2312_15554_b200 as pf
    from oracle import poreflow_oracle as O

    n = args.n
    if args.geometry == "packing":  # cfg 3 / 4 geometry (SURVEY §8d generator, seed 0)
        ind = pf.random_packing_geometry(n, seed=0)
    else:
        ind = pf.make_model_geometry(pf.UnitCellGrid((n, n, n)), radius=0.25)
    scfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0.0, 0.0))
    tcfg = pf.TransportConfig(pe=10.0, a0=0.55, eps=1e-5, composition_gradient=(1.0, 0.0, 0.0))
    host = np.array(ind.values)
    pf.effective_tensors(pf.IndicatorField(pf.UnitCellGrid((n, n, n)), host),
                         pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0.0, 0.0), max_iter=3),
                         pf.TransportConfig(pe=10.0, a0=0.55, eps=1e-5, composition_gradient=(1.0, 0.0, 0.0),
                                            max_iter=3))  # warm-up (plans)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if args.stokes_only:  # cfg 3: the three load cases and K* only
        cell = pf.IndicatorField(pf.UnitCellGrid((n, n, n)), host)
        from paper_2312_15554_b200.batch import solve_stokes_many_device

        flows = solve_stokes_many_device([cell] * 3, [pf.StokesConfig.with_tolerance(
            1e-5, pressure_gradient=tuple(float(i == a) for i in range(3))) for a in range(3)])
        K = pf.permeability([st.u for st, _ in flows], cell, "central")
        D = np.full((3, 3), np.nan)
        torch.cuda.synchronize()
        gpu_s = time.perf_counter() - t0
        s_its, t_its = [r.iterations for _, r in flows], []
        conv = all(r.converged for _, r in flows)
        u_flow = flows[0][0].u
    else:
        res = pf.effective_tensors(pf.IndicatorField(pf.UnitCellGrid((n, n, n)), host), scfg, tcfg)
        K, D = np.asarray(res.tensors.permeability), np.asarray(res.tensors.diffusivity)
        torch.cuda.synchronize()
        gpu_s = time.perf_counter() - t0
        s_its = [r.iterations for r in res.flow_reports]
        t_its = [r.iterations for r in res.transport_reports]
        conv = bool(res.converged)
        u_flow = res.u_phys
    vox_it = n ** 3 * (sum(s_its) + sum(t_its))
    # CPU: oracle rates on a bounded sample (loop time only), extrapolated
    tm = {}
    k_s = 2
    O.solve_stokes(ind.values, (1.0, 0.0, 0.0), 1e-5, 1e-5, max_iter=k_s, timer=tm)
    stokes_rate = n ** 3 * k_s / tm["loop_s"]
    transport_rate = None
    cpu_s = n ** 3 * sum(s_its) / stokes_rate
    if t_its:
        u1 = u_flow.cpu().numpy()
        k_t = 2
        t1 = time.perf_counter()
        O.solve_transport(ind.values, u1, (1.0, 0.0, 0.0), pe=10.0, a0=0.55, eps=1e-5, max_iter=k_t)
        transport_rate = n ** 3 * k_t / (time.perf_counter() - t1)
        cpu_s += n ** 3 * sum(t_its) / transport_rate
    what = "cfg-3 three load cases + K*" if args.stokes_only else "cfg-2 cell-to-tensors run (cli.run flow)"
    print(json.dumps({"metric": f"{what} at {n}^3 ({args.geometry}), wall clock (secondary)",
                      "value": gpu_s, "unit": "s", "higher_is_better": False, "dtype": "f64",
                      "voxel_iters_per_s": vox_it / gpu_s, "stokes_iterations": s_its,
                      "transport_iterations": t_its, "converged": conv,
                      "K": K.tolist(), "D": None if args.stokes_only else D.tolist(),
                      "config": {"workload": f"pipeline_{args.geometry}_{n}^3", "stokes": "eps 1e-5, adaptive penalties",
                                 "transport": None if args.stokes_only else "Pe 10, a0 0.55, eps 1e-5"},
                      "cpu_extrapolated": {"seconds": cpu_s, "kind": "port", "cores": os.cpu_count(),
                                           "sample": f"{k_s} Stokes (+ 2 transport) iterations of the same cell "
                                                     f"(numpy + scipy.fft), rate x GPU iteration counts",
                                           "stokes_rate": stokes_rate, "transport_rate": transport_rate},
                      "speedup_vs_cpu_extrapolated": cpu_s / gpu_s}), flush=True)
    return 0


def run_ensemble_workload(args):
    """Secondary line: BASELINE cfg 4 — an ensemble of independent 128^3 random
    packings (seeds rank*C .. rank*C + C-1), C cells resident per GPU, each on its
    own plan / CUDA stream so their passes overlap; aggregate voxel-iters/s, max
    over ranks under torchrun (weak scaling, no collective in the timed region)."""
    import torch

    import paper_2312_15554_b200 as pf

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    n, C = args.n, args.cells
    solvers = []
    # one torch stream per cell: a plan's work stream is ordered after its bound
    # user stream, so cells sharing one user stream would serialise
    streams = [torch.cuda.Stream(dev) for _ in range(C)]
    for k in range(C):
        ind = pf.random_packing_geometry(n, seed=rank * C + k)
        cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0.0, 0.0), max_iter=10**7)
        with torch.cuda.stream(streams[k]):
            st = pf.DeviceAdmmState.zeros(ind.grid, dev)
            s = pf.StokesSolver(ind, cfg, pf.PenaltyParams(), st, dev, history_rows=args.warmup + args.steps + 1,
                                plan_slot=k)
            s.begin()
        solvers.append(s)
    for k, s in enumerate(solvers):
        with torch.cuda.stream(streams[k]):
            s.iterate(args.warmup, poll=False)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    chunk = 8
    done = 0
    main = torch.cuda.current_stream(dev)
    for st_k in streams:
        st_k.wait_stream(main)
    while done < args.steps:
        k = min(chunk, args.steps - done)
        for j, s in enumerate(solvers):
            with torch.cuda.stream(streams[j]):
                s.iterate(k, poll=False)
        done += k
    for st_k in streams:  # join every cell's stream into the timing stream
        main.wait_stream(st_k)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    its = []
    for k, s in enumerate(solvers):
        with torch.cuda.stream(streams[k]):
            r = s.end()
        its.append(int(r.iterations))
    assert all(i == args.warmup + args.steps for i in its), its
    value = world * C * n ** 3 * args.steps / (ms / 1e3)
    peak, _ = peak_hbm()
    if rank == 0:
        print(json.dumps({"metric": f"Stokes ALM voxel-iters/s, ensemble of {n}^3 cells (secondary, cfg 4)",
                          "value": value, "unit": UNIT, "n_gpus": world, "cells_per_gpu": C,
                          "ms_per_step": ms / args.steps, "steps": args.steps, "warmup": args.warmup,
                          "scaling": "weak", "dtype": "f64", "pipeline": solvers[0].pipeline,
                          "config": {"workload": f"ensemble_random_packing_{n}^3", "cells": world * C},
                          "iteration_roofline": {"alg_bytes_per_voxel_iter": B_ALG_ITER,
                                                 "frac": B_ALG_ITER * value / world / 1e9 / peak}}), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def run_slab_workload(args):
    """Secondary line: BASELINE cfg 5 — ONE random-packing cell slab-decomposed over
    the ranks (x-slabs; two exchanges of 3 half-spectrum components and one
    9-double all_reduce per iteration).  The fused slab pipeline where it applies
    (cubic 64/128/256, power-of-two ranks), else the cuFFT one.  Strong scaling:
    total work fixed."""
    import torch

    import paper_2312_15554_b200 as pf
    from paper_2312_15554_b200 import slab as S

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    n = args.n
    from paper_2312_15554_b200.grid import rasterize_packing_slab, random_sphere_packing

    lo, hi = S.slab_range(n, world, rank)
    solid_np = rasterize_packing_slab(random_sphere_packing(0), (n, n, n), lo, hi)  # this rank's planes only
    cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0.0, 0.0),
                                         max_iter=args.warmup + args.steps + 1)
    be = S.DeviceSlabBackend((n, n, n), world, rank, "central", dev)
    be.bind()
    L = (hi - lo) * n * n
    st = {k: torch.zeros(3 * L, dtype=torch.float64, device=dev) for k in ("u", "u_tilde", "a", "lam")}
    st["q"] = torch.zeros(L, dtype=torch.float64, device=dev)
    solid = torch.as_tensor(solid_np).reshape(-1).to(dev)
    fused = be.fused_sizes()[0] > 0 and not args.slab_cufft
    if fused:
        comm = S.SymmetricMemoryExchange() if (args.exchange == "p2p" and world > 1) else None
        sol = S.FusedSlabStokes(be, (n, n, n), cfg, pf.PenaltyParams(), solid, st, comm=comm, exchange=args.exchange)
    else:
        sol = S.SlabStokes(be, (n, n, n), cfg, pf.PenaltyParams(), solid, st)
    sol.begin()
    sol.iterate(args.warmup, poll=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    a.record()
    sol.iterate(args.steps, poll=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    rep = sol.end()
    assert rep.iterations == args.warmup + args.steps and not rep.converged
    value = n ** 3 * args.steps / (ms / 1e3)
    if rank == 0:
        print(json.dumps({"metric": "Stokes ALM voxel-iters/s, one slab-decomposed cell (secondary, cfg 5)",
                          "value": value, "unit": UNIT, "n_gpus": world, "ms_per_step": ms / args.steps,
                          "steps": args.steps, "warmup": args.warmup, "scaling": "strong", "dtype": "f64",
                          "pipeline": (("slab-fused (fused passes; PK / MF store into the owners' Y over P2P)"
                                        if args.exchange == "p2p" else
                                        "slab-fused (fused passes, per-component Y all_to_all overlapped)")
                                       if fused else "slab (cuFFT local transforms + all_to_all)"),
                          "config": {"workload": f"slab_random_packing_{n}^3", "ranks": world}}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def launch_ranks(n_gpus: int) -> int:
    """``python bench.py --gpus N`` without a launcher: start N ranks on this node
    through torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1),
    each re-running this command line, and return their exit status.  Under
    torchrun (WORLD_SIZE set) the existing ranks are used as they are."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n_gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + [
        # torchrun's own parser would take "--n" as an ambiguous prefix of its options
        "--size" if a == "--n" else ("--size=" + a[4:] if a.startswith("--n=") else a) for a in sys.argv[1:]]
    return subprocess.run(cmd, cwd=str(ROOT)).returncode


def run_dry(args):
    """Fan-out probe (no GPU work): each rank joins the group (NCCL when CUDA is
    visible, else gloo), the ranks are gathered, rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist

    rank, local_rank, world = dist_env()
    ranks = [rank]
    if world > 1:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local_rank)
        dist.init_process_group(backend)
        dev = torch.device("cuda", local_rank) if backend == "nccl" else torch.device("cpu")
        t = torch.zeros(world, dtype=torch.int64, device=dev)
        t[rank] = rank + 1
        dist.all_reduce(t)
        ranks = [int(x) - 1 for x in t.cpu().tolist()]
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": ranks, "gpus_requested": args.gpus,
                          "config": headline_config(args.n, world)}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--size", "--n", dest="n", type=int, default=256, help="cell edge N (N^3 voxels)")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="stokes", choices=("stokes", "transport", "ensemble", "slab", "pipeline"),
                    help="stokes = the headline metric; transport / ensemble = secondary lines")
    ap.add_argument("--cells", type=int, default=16, help="cells per GPU for --workload ensemble")
    ap.add_argument("--slab-cufft", action="store_true", help="--workload slab: the cuFFT slab pipeline")
    ap.add_argument("--exchange", default="a2a", choices=("a2a", "p2p"),
                    help="--workload slab: all_to_all exchange or the transpose fused into the passes over P2P")
    ap.add_argument("--geometry", default="spheres", choices=("spheres", "packing"),
                    help="--workload pipeline: cfg 1/2 sphere array or the cfg 3/4 random packing")
    ap.add_argument("--stokes-only", action="store_true", help="--workload pipeline: cfg 3 (load cases + K* only)")
    ap.add_argument("--tcells", type=int, default=1,
                    help="--workload transport: concurrent solves (cfg 2's load cases e_1..e_3), own plan + stream each")
    ap.add_argument("--dry-run", action="store_true",
                    help="rank fan-out probe: every rank joins the process group, rank 0 prints n_gpus and ranks")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args.gpus)
    if args.dry_run:
        return run_dry(args)
    if args.workload == "transport":
        return run_transport_workload(args)
    if args.workload == "ensemble":
        return run_ensemble_workload(args)
    if args.workload == "slab":
        return run_slab_workload(args)
    if args.workload == "pipeline":
        return run_pipeline_workload(args)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
