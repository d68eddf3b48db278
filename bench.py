#!/usr/bin/env python3
"""bench.py -- HEGrid hot path on B200: gridded samples x channels per second.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--impl ours|reference]

One "step" = Eq. 1 for the whole workload (BASELINE.json configs[3] by default: 1M drift-scan
samples x 4096 channels -> 300x300 map): hegrid_grid_device on HBM-resident, plan-ordered
channel-contiguous values (the layout the staging layer delivers), the plan (shared
component, built once per coordinate set) prebuilt and its time reported separately.
Multi-GPU: one process per GPU (torchrun); the workload's channels are sharded across the
ranks (4096 / G each, configs[3] "channel-sharded at 1/2/4/8 GPUs"), no data-path
collective, strong scaling (the total work is fixed).

Also measured in the same run:
  e2e       -- the public host API (plan from host coords + hegrid_grid on pinned host
               [C][N] values -> pinned host maps), H2D/D2H inside the timed region, against
               the pinned H2D bandwidth measured in the same run (the PCIe roof);
  roofline  -- the accumulate kernel (the dominant kernel) timed with CUDA events on its
               launch stream: the north_star's HBM-roofline fraction, plus the tensor view
               (fp32-accurate work against the tensor peak for its mixed tf32 + bf16 MMA
               stream) and the ALU view;
  cpu_baseline -- the fp64 oracle on this host's cores, on a bounded sample of cells.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "gridded samples x channels per second"
UNIT = "samples*channels/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)
        return self.summary()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        pw = [float(r[3]) for r in self.rows if r[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "power_w_max": max(pw) if pw else None,
                "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def plan_layout_values(w, lon, lat, perm, channel_ids, device):
    """Values of the given channels, generated directly in plan order [n_used][C]."""
    C = len(channel_ids)
    out = torch.empty((perm.shape[0], C), dtype=torch.float32, device=device)
    ch = torch.as_tensor(channel_ids, dtype=torch.int64, device=device)
    for c0 in range(0, C, 256):
        blk = synth.values(w, lon, lat, channels=ch[c0:c0 + 256], samples=perm)
        out[:, c0:c0 + blk.shape[0]] = blk.t()
        del blk
    return out


def user_layout_values_pinned(w, lon, lat, channel_ids, device):
    """Values [C][N] in original sample order in pinned host memory (the e2e input)."""
    C, N = len(channel_ids), lon.shape[0]
    host = torch.empty((C, N), dtype=torch.float32, pin_memory=True)
    ch = torch.as_tensor(channel_ids, dtype=torch.int64, device=device)
    for c0 in range(0, C, 256):
        host[c0:c0 + 256].copy_(synth.values(w, lon, lat, channels=ch[c0:c0 + 256]).cpu())
    return host


def pinned_h2d_gbs(dev, mib=1024, reps=3):
    """Pinned host -> device copy bandwidth (GB/s), the PCIe roof of the e2e path."""
    h = torch.empty(mib << 18, dtype=torch.float32, pin_memory=True)
    d = torch.empty(mib << 18, dtype=torch.float32, device=dev)
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize(dev)
    gbs = reps * h.numel() * 4 / (time.perf_counter() - t0) / 1e9
    del h, d
    return gbs


def oracle_sample(w, lon_h, lat_h, vals_h, target_s=15.0, max_cells=None):
    """Time the fp64 oracle (all host cores) on an evenly spaced sample of cells with all
    channels; return (throughput samples*ch/s extrapolated to the whole map, detail)."""
    import oracle
    oracle.build()
    nthreads = oracle.max_threads()
    cells_all = w.cells
    # calibration round: one cell per thread
    k = min(nthreads, cells_all)
    cal = np.linspace(0, cells_all - 1, k).astype(np.int64)
    t0 = time.perf_counter()
    oracle.grid(lon_h, lat_h, vals_h, w.map, w.fwhm_deg, w.support, cells=cal, nthreads=nthreads)
    t_cal = time.perf_counter() - t0
    # calibrate on a larger round (4 cells per thread) so thread start-up does not dominate
    k2 = min(4 * nthreads, cells_all)
    cal2 = np.linspace(0, cells_all - 1, k2).astype(np.int64)
    t0 = time.perf_counter()
    oracle.grid(lon_h, lat_h, vals_h, w.map, w.fwhm_deg, w.support, cells=cal2, nthreads=nthreads)
    t_cal = time.perf_counter() - t0
    n_cells = int(max(k2, min(cells_all, k2 * max(1.0, target_s / max(t_cal, 1e-3)))))
    if max_cells:
        n_cells = min(n_cells, max_cells)
    cells = np.linspace(0, cells_all - 1, n_cells).astype(np.int64)
    t0 = time.perf_counter()
    oracle.grid(lon_h, lat_h, vals_h, w.map, w.fwhm_deg, w.support, cells=cells, nthreads=nthreads)
    t = time.perf_counter() - t0
    thr = w.n * vals_h.shape[0] * (n_cells / cells_all) / t
    return thr, {"cores": nthreads, "cells": n_cells, "seconds": t,
                 "sample": f"{n_cells} of {cells_all} cells (evenly spaced) x all "
                           f"{vals_h.shape[0]} channels x all {w.n} samples, fp64 brute force; "
                           f"throughput scaled by cells_all/{n_cells}"}


def run_reference(args):
    """--impl reference: the oracle as it stands, on this host's cores, same metric/config."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    w = synth.CONFIGS[args.workload]
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    lon, lat = synth.coords(w, device=dev)
    C = w.channels
    vals = torch.empty((C, w.n), dtype=torch.float32)
    ch = torch.arange(C, device=dev)
    for c0 in range(0, C, 256):
        vals[c0:c0 + 256] = synth.values(w, lon, lat, channels=ch[c0:c0 + 256]).cpu()
    lon_h, lat_h, vals_h = lon.cpu().numpy(), lat.cpu().numpy(), vals.numpy()
    budget = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    per = []
    detail = None
    t_run = time.perf_counter()
    for s in range(args.warmup + args.steps):
        thr, detail = oracle_sample(w, lon_h, lat_h, vals_h, target_s=budget)
        if s >= args.warmup:
            per.append(w.n * C / thr)     # seconds for one whole-workload step (extrapolated)
    t_run = time.perf_counter() - t_run
    ms = 1000 * statistics.median(per)
    value = w.n * C / (ms / 1000)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(w, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": detail["cores"],
                             "kind": "oracle", "sample": detail["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            # each "step" is a bounded, evenly spaced cell sample of the workload timed on the
            # host and extrapolated to the whole map: ms_per_step is that extrapolation, not a
            # measured whole-workload time (the run itself took timed_s seconds)
            "extrapolated": True, "timed_s": t_run,
            "step_note": "per step: %s; ms_per_step extrapolated to all cells" % detail["sample"]}
    print(json.dumps(line), flush=True)


def workload_config(w, world):
    from paper_2207_04584_b200.shard import channel_shard
    c0, c1 = channel_shard(w.channels, world, 0)
    return {"workload": w.name, "desc": w.note, "n_samples": w.n, "channels_per_gpu": c1 - c0,
            "global_channels": w.channels, "map": f"{w.nx}x{w.ny}",
            "cell_deg": w.cdelt, "kernel_fwhm_deg": w.fwhm_deg, "support_sigma": w.support,
            "field_deg": [w.field_lon, w.field_lat], "centre_deg": list(w.centre),
            "sampling": w.kind, "parallelism": f"channel-shard x{world} (strong scaling)",
            "input_layout": "plan-ordered [n_used][C] fp32, HBM-resident",
            "l2": "inputs larger than L2 (values %.1f GB vs 126 MB L2)" % (w.n * w.channels * 4 / 1e9)}


def warm_modules(w, dev, local, engine):
    """Grid a tiny slice of the workload once so that lazy CUDA module loading (a per-process
    cost) is not counted in the per-plan prep_ms."""
    from paper_2207_04584_b200 import Plan
    small = w.with_(n=64 * 64, tracks=64, per_track=64, nx=24, ny=24, field_lon=0.4,
                    field_lat=0.4, channels=4)
    lon, lat = synth.coords(small, device=dev)
    with Plan(lon, lat, small.map, small.fwhm_deg, small.support, device=local,
              engine=engine) as p:
        vals = torch.ones((4, small.n), dtype=torch.float32, device=dev)
        p.grid(vals)
        vp = torch.ones((p.info()["n_used"], 512), dtype=torch.float32, device=dev)
        out = torch.empty((512, small.ny, small.nx), dtype=torch.float32, device=dev)
        W = torch.empty((small.ny, small.nx), dtype=torch.float32, device=dev)
        p.grid_plan_layout(vp, 512, out, W)
    torch.cuda.synchronize(dev)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--engine", default="tc", choices=["simt", "tc", "auto"])
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", local)
    from paper_2207_04584_b200 import Plan, abi

    w = synth.CONFIGS[args.workload]
    from paper_2207_04584_b200.shard import channel_shard
    C_global = w.channels
    c0, c1 = channel_shard(C_global, world, rank)              # strong scaling: 1/G of the channels
    C = c1 - c0
    channel_ids = list(range(c0, c1))
    lon, lat = synth.coords(w, device=dev)

    # ---------------------------------------------------------------- plan (once)
    stream = torch.cuda.current_stream(dev)
    warm_modules(w, dev, local, args.engine)
    plan = Plan(lon, lat, w.map, w.fwhm_deg, w.support, device=local, stream=stream,
                engine=args.engine)
    info = plan.info()
    perm = torch.as_tensor(plan.permutation(), device=dev)
    vp = plan_layout_values(w, lon, lat, perm, channel_ids, dev)
    out = torch.empty((C, w.ny, w.nx), dtype=torch.float32, device=dev)
    Wmap = torch.empty((w.ny, w.nx), dtype=torch.float32, device=dev)
    torch.cuda.synchronize(dev)

    def step():
        plan.grid_plan_layout(vp, C, out, Wmap, stream=stream)

    # the first launch also builds the engine's per-plan tables (TC chunk schedule, W per
    # cell, precomputed weight image): a one-time shared component, reported as prep_ms
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    step()
    f1.record(stream)
    torch.cuda.synchronize(dev)
    first_ms = f0.elapsed_time(f1)
    for _ in range(max(args.warmup - 1, 0)):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    plan.profile(True)
    plan.profile_read()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    l0 = abi.hegrid_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = abi.hegrid_launch_count() - l0
    clk = clocks.stop()
    ms_total = e0.elapsed_time(e1)
    k_ms, k_n = plan.profile_read()
    plan.profile(False)
    t = torch.tensor([ms_total], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    units = w.n * C_global
    value = units / (ms_step / 1000)

    # ---------------------------------------------------------------- roofline
    peaks, peak_src = load_peaks()
    k_avg_ms = k_ms / max(k_n, 1)
    cells = w.cells
    alg_bytes = (4 * info["n_used"] * C + 4 * cells * C + 4 * cells + 16 * info["n_used"]
                 + 4 * (info["n_bins"] + 1))
    flops = 2.0 * info["n_pairs"] * C
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    fp32_peak_tflops = 148 * 128 * 2 * sm_max * 1e6 / 1e12
    hbm_achieved = alg_bytes / (k_avg_ms / 1000) / 1e9
    alu_achieved = flops / (k_avg_ms / 1000) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(w.name, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    # The metric BASELINE.json names is the fraction of the HBM roofline: achieved =
    # algorithmic bytes (values read once, map + weight map written once, plan
    # arrays read once) / the accumulate kernel's average launch time, peak = the measured
    # HBM copy bandwidth.  The ALU view (2 flops per (cell, sample, channel) pair against
    # the FP32 CUDA-core peak) is reported beside it.
    kname = "k_accum_tc" if args.engine == "tc" else "k_accum_simt"
    roof = {"bound": "hbm", "achieved": hbm_achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": hbm_achieved / peaks["hbm_gbs"], "traffic": traffic, "kernel": kname,
            "kernel_ms": k_avg_ms, "kernel_share": k_ms / ms_total if ms_total else None,
            "algorithmic_bytes_per_launch": alg_bytes, "peak_source": f"{peak_src} hbm_gbs",
            "step_frac": (alg_bytes / (ms_step / 1000) / 1e9) / peaks["hbm_gbs"]}
    alu_view = {"achieved": alu_achieved, "peak": fp32_peak_tflops, "unit": "TFLOP/s",
                "frac": alu_achieved / fp32_peak_tflops, "algorithmic_flops_per_launch": flops,
                "peak_source": "148 SMs x 128 FP32 lanes x 2 flop x sm_max_mhz (DESIGN.md)"}
    # Tensor view: per 8-sample K-step and in-reach block the engine issues one kind::tf32 MMA
    # (hi * hi) and one kind::f16 bf16 MMA of K = 16 pairing the two correction terms
    # (DESIGN.md section 6): two MMA slots of equal duration, each running at the TF32 rate
    # (tf32 K = 8 and bf16 K = 16 take the same time).  Useful work = 2 P C fp32-accurate
    # flops; the roof for it = the TF32 peak / 2, the TF32 peak being the measured bf16 peak / 2
    # (the nominal bf16 : tf32 ratio).  mma_density = useful pairs / executed (16-cell x
    # 32-sample block slots); executed_tf32_equiv_tflops counts both MMA slots at the tf32 rate.
    info2 = plan.info()
    tf32_peak = peaks["bf16_tflops"] / 2.0
    slots = info2.get("tc_block_slots", 0) or 0
    tensor_view = {"achieved": flops / (k_avg_ms / 1000) / 1e12, "peak": tf32_peak / 2.0,
                   "unit": "TFLOP/s (fp32-accurate; tf32 hi*hi + bf16 correction MMAs)",
                   "frac": flops / (k_avg_ms / 1000) / 1e12 / (tf32_peak / 2.0),
                   "tf32_peak": tf32_peak,
                   "peak_source": f"{peak_src} bf16_tflops / 2 (tf32) / 2 (MMA slots per pair)",
                   "mma_density": info["n_pairs"] / (512.0 * slots) if slots else None,
                   "executed_tf32_equiv_tflops": (2 * 2 * 512.0 * slots * C / (k_avg_ms / 1000) / 1e12)
                   if slots else None} if args.engine == "tc" else None
    one_shot_ms = info["t_plan_ms"] + max(first_ms - ms_step, 0.0) + ms_step

    # ---------------------------------------------------------------- e2e (public host API)
    e2e = None
    host_vals = None
    if not args.no_e2e:
        del vp
        torch.cuda.empty_cache()
        h2d_gbs = pinned_h2d_gbs(dev)
        host_vals = user_layout_values_pinned(w, lon, lat, channel_ids, dev)
        host_out = torch.empty((C, w.ny, w.nx), dtype=torch.float32, pin_memory=True)
        host_w = torch.empty((w.ny, w.nx), dtype=torch.float32, pin_memory=True)
        # the coordinates are inputs of the step too: pinned like the values
        lon_h = lon.cpu().pin_memory().numpy()
        lat_h = lat.cpu().pin_memory().numpy()

        def e2e_step():
            # the whole job through the public API: a plan from the host coordinates
            # (coordinates H2D, index build, engine tables) and hegrid_grid from pinned host
            # [C][N] values to pinned host maps (H2D, permute, accumulate, D2H over streams)
            with Plan(lon_h, lat_h, w.map, w.fwhm_deg, w.support, device=local,
                      engine=args.engine) as p:
                p.grid(host_vals, host_out, host_w)
            return float(host_w[w.ny // 2, w.nx // 2])   # read of the result
        e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        e2e_marks = []
        for _ in range(args.e2e_steps):
            e2e_step()
            e2e_marks.append(time.perf_counter())
        torch.cuda.synchronize(dev)
        te = (time.perf_counter() - t0) / args.e2e_steps
        e2e_step_ms = [round(1000 * (b - a), 2) for a, b in zip([t0] + e2e_marks[:-1], e2e_marks)]
        # the same hegrid_grid call on a plan built once (the coordinates are shared by every
        # channel block of an observation)
        with Plan(lon_h, lat_h, w.map, w.fwhm_deg, w.support, device=local, engine=args.engine) as p:
            p.grid(host_vals, host_out, host_w)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                p.grid(host_vals, host_out, host_w)
            torch.cuda.synchronize(dev)
            tg = (time.perf_counter() - t0) / args.e2e_steps
        tt = torch.tensor([te, tg], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te, tg = float(tt[0].item()), float(tt[1].item())
        h2d_b = C * w.n * 4 + 16 * w.n
        e2e = {"value": units / te, "unit": UNIT, "ms_per_step": te * 1000,
               "h2d_bytes_per_step": h2d_b,
               "d2h_bytes_per_step": C * cells * 4 + cells * 4,
               "api": "Plan(host coords) + hegrid_grid(pinned host [C][N] -> pinned host maps)",
               "step_ms": e2e_step_ms,
               "pinned_h2d_gbs": h2d_gbs,
               "h2d_roof_ms": h2d_b / (h2d_gbs * 1e9) * 1000,
               "frac_of_h2d_roof": (h2d_b / te / 1e9) / h2d_gbs,
               "plan_reused": {"value": units / tg, "ms_per_step": tg * 1000,
                               "frac_of_h2d_roof": ((h2d_b - 16 * w.n) / tg / 1e9) / h2d_gbs,
                               "api": "hegrid_grid on a plan built once"}}

    # ---------------------------------------------------------------- cpu baseline (rank 0, N=1)
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        if host_vals is None:
            host_vals = user_layout_values_pinned(w, lon, lat, channel_ids, dev)
        thr, det = oracle_sample(w, lon.cpu().numpy(), lat.cpu().numpy(), host_vals.numpy())
        cpu = {"value": thr, "unit": UNIT, "cores": det["cores"], "kind": "oracle",
               "sample": det["sample"], "seconds": det["seconds"]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic (seeded drift-scan coords, sky-model values)",
                "config": workload_config(w, world),
                "plan_ms": info["t_plan_ms"],
                "prep_ms": max(first_ms - ms_step, 0.0),
                "one_shot_ms": one_shot_ms,
                "pairs": {"n_pairs": info["n_pairs"], "candidates": info["n_candidate_pairs"],
                          "nbr_mean": info["nbr_mean"]},
                "roofline": roof, "tensor_view": tensor_view, "alu_view": alu_view, "clocks": clk,
                "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
