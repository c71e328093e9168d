#!/usr/bin/env python
"""Benchmark: EM point*component*iterations/s and ms per GMM fit (BASELINE.json).

A step is one full GMM fit of the hot path on one batch of synthetic input:
kinit (k-means++) -> initial M step -> EM to tolerance, for BASELINE cfg2
(one 640x480 synthetic depth frame -> 307,200 4D points, K=512, seed 0,
ll_rel_tol 1e-3, cov_reg 1e-6) on every GPU. With N > 1 GPUs (torchrun) each
rank fits its own frame (cfg3-style replicas: frame r jittered by 2 mm, seed
r): weak scaling, no collective on the data path; the job value is all
ranks' units over the max-over-ranks time.

value  = sum of units (N * K_t per E step) / device time of the fits, inputs
         resident in HBM (CUDA events inside the library around each fit;
         L2 flushed between steps).
e2e    = the same metric through the C ABI call with host (pinned) buffers:
         H2D of the points and D2H of the model inside the timed region.
--impl reference times the reference algorithm on the host CPU (the FP64
oracle port, all host threads; the reference itself cannot be built here).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "EM point*component*iters/sec and ms per GMM fit"
UNIT = "point*component*iter/s"
FLOP_PER_UNIT = {4: 62.0, 3: 42.0}     # 2D^2 + 6D + 6
NOMINAL_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
# DRAM traffic of one fused-E launch at cfg2 K=512 (ncu --set full capture)
TRAFFIC_BYTES = 5.095e6  # 5.095 MB read + 256 B written per launch
TRAFFIC_SRC = "profiles/r1h_estep_ncu.txt"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="gmmb", choices=["gmmb", "reference"])
    ap.add_argument("--k", type=int, default=512)
    ap.add_argument("--tol", type=float, default=1e-3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=20.0)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_points(gm, rank):
    p = gm.synthetic_frame_cloud()          # make_synthetic_frame + image_pair_to_cloud
    if rank > 0:                            # cfg3 frame r: xyz jittered 2 mm, seed r
        p = gm.jitter_cloud(p, 0.002, rank)
    return p


class Clocks:
    """nvidia-smi sampling during the timed region (clocks + throttle reasons)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f".clocks_{os.getpid()}.csv")

    def __enter__(self):
        self.t_start = time.time()
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            # nvidia-smi needs ~0.5 s to start sampling: keep it alive long
            # enough to cover at least 1 s of the (busy) window
            time.sleep(max(0.0, 1.0 - (time.time() - self.t_start)))
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                try:
                    rows.append(parts)
                except ValueError:
                    pass
        try:
            os.remove(self.path)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[4:8]) if v.strip() == "Active"})
        loaded = [v for v in sm if v > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def cpu_fit_rate(points, k, tol, budget_s, steps=None):
    """Times the FP64 oracle port (all host threads) on full cfg fits."""
    import oracle
    oracle.set_num_threads(0)
    threads = oracle.num_threads()
    times, units = [], []
    t_end = time.time() + budget_s
    n = len(points)
    count = 0
    while True:
        t0 = time.perf_counter()
        r = oracle.fit_k(points, k, max_iters=100, ll_rel_tol=tol, cov_reg=1e-6, seed=0)
        dt = time.perf_counter() - t0
        times.append(dt)
        units.append(float(n) * sum([k] * r["em_iterations"]) if r["removed"] == 0 else
                     float(n) * k * r["em_iterations"])
        count += 1
        if steps is not None:
            if count >= steps:
                break
        elif time.time() > t_end or count >= 3:
            break
    return sum(units) / sum(times), threads, times, units


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import paper_2307_00071_b200 as gm
    pts = make_points(gm, 0)
    if args.warmup > 0:
        cpu_fit_rate(pts, args.k, args.tol, 0, steps=args.warmup)
    rate, threads, times, units = cpu_fit_rate(pts, args.k, args.tol, 0, steps=max(args.steps, 1))
    ms = 1e3 * sum(times) / len(times)
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (make_synthetic_frame 640x480 -> 307,200 4D points)",
        "config": {"workload": "cfg2: 4D frame, N=307200, K=%d, k-means++ + EM to tol %g" %
                   (args.k, args.tol), "global_batch": 1, "parallelism": "cpu"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": "%d full fits (kinit + M + EM), FP64 oracle restatement, "
                                   "std::thread fan-out over 4096-point blocks" % len(times)},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def flush_l2(torch, buf):
    buf.add_(1.0)  # 256 MiB write > 126 MB L2


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    rank, world, local = dist_env()
    import torch
    import paper_2307_00071_b200 as gm

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = gm.Context(local)
    sm, cc_major, cc_minor = ctx.device_info()
    pts = make_points(gm, rank)
    n, d = pts.shape
    em = gm.EmParams(100, args.tol, 1e-6, rank)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- value: inputs resident in HBM ------------------------------------
    ctx.upload(pts)
    res = []
    with Clocks(local) as clk:          # sampling spans warm-up + timed region
        for _ in range(max(args.warmup, 3)):
            ctx.fit_k_resident(args.k, em)
        flush_l2(torch, flush)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush_l2(torch, flush)
            torch.cuda.synchronize()
            res.append(ctx.fit_k_resident(args.k, em))
        barrier()
        wall = time.perf_counter() - t0
    clocks = clk.summary()
    dev_ms = sum(r.ms_total for r in res)
    units = sum(r.units for r in res)
    est_ms = sum(r.ms_estep for r in res)
    iters = [r.em_iterations for r in res]
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([dev_ms, units, est_ms], dtype=torch.float64, device="cuda")
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        dev_ms_job, units_job = float(mx[0]), float(t[1])
    else:
        dev_ms_job, units_job = dev_ms, units
    value = units_job / (dev_ms_job * 1e-3)

    # ---- e2e: C ABI call with pinned host buffers --------------------------
    host = torch.empty((d, n), dtype=torch.float64, pin_memory=True)
    host.numpy()[:] = pts.T                      # column-major N x D
    host_pts = host.numpy().T                    # (N, D) Fortran view, pinned
    assert not host_pts.flags["C_CONTIGUOUS"] and host_pts.flags["F_CONTIGUOUS"]
    for _ in range(2):
        gm.fit_k(host_pts, args.k, em, ctx=ctx)
    barrier()
    e2e_units, t_e2e = 0.0, 0.0
    for _ in range(args.steps):
        flush_l2(torch, flush)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        r = gm.fit_k(host_pts, args.k, em, ctx=ctx)
        torch.cuda.synchronize()
        t_e2e += time.perf_counter() - t1
        e2e_units += r.units
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([t_e2e, e2e_units], dtype=torch.float64, device="cuda")
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        t_e2e, e2e_units = float(mx[0]), float(t[1])
    e2e = e2e_units / t_e2e
    kk = args.k
    d2h = 8 * (kk * (1 + d + d * (d + 1) // 2) + 100) + 96

    # ---- roofline of the dominant kernel (fused E step + statistics) ------
    # The EM loop of a fit is one CUDA graph (no per-kernel events inside);
    # the same K fits are repeated in timing mode (chunked launches, CUDA
    # events on the library stream around every fused E kernel; identical
    # kernels and results) to get the kernel's average launch duration.
    ctx.upload(pts)
    ctx.set_timing(True)
    est_ms, est_units, est_launches = 0.0, 0.0, 0
    for _ in range(args.steps):
        flush_l2(torch, flush)
        torch.cuda.synchronize()
        rt = ctx.fit_k_resident(args.k, em)
        est_ms += rt.ms_estep
        est_units += rt.units
        est_launches += rt.em_iterations
    ctx.set_timing(False)
    peak_tf, _ = ctx.ffma_peak(50.0)
    achieved_tf = FLOP_PER_UNIT[d] * est_units / (est_ms * 1e-3) / 1e12

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": dev_ms_job / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (make_synthetic_frame 640x480 -> 307,200 4D points; "
                "rank r>0: 2 mm jitter, seed r)",
        "config": {"workload": "cfg2: 4D frame N=307200, K=%d, k-means++ + EM to tol %g "
                               "(one fit per GPU per step)" % (args.k, args.tol),
                   "global_batch": world, "points_per_fit": n, "k": args.k,
                   "em_iterations": iters, "parallelism": "replicas%d" % world,
                   "l2": "flushed between steps (256 MiB write)"},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": n * d * 8,
                "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * t_e2e / args.steps},
        "gpu_launches": int(sum(r.launches for r in res)),
        "stage_ms": {"layout": statistics.mean(r.ms_layout for r in res),
                     "kinit": statistics.mean(r.ms_kinit for r in res),
                     "mstep0": statistics.mean(r.ms_mstep0 for r in res),
                     "em": statistics.mean(r.ms_em for r in res),
                     "estep_kernel": est_ms / args.steps,
                     "estep_us_per_launch": 1e3 * est_ms / max(est_launches, 1)},
        "em_only_value": units / (sum(r.ms_em for r in res) * 1e-3),
        "roofline": {"bound": "fp32", "kernel": "estep_ws_kernel (warp-specialised fused E "
                     "step + sufficient statistics)", "achieved": achieved_tf, "peak": peak_tf,
                     "unit": "TFLOP/s", "frac": achieved_tf / peak_tf,
                     "flop_per_unit": FLOP_PER_UNIT[d],
                     "timing": "CUDA events around each fused E launch on the library stream, "
                               "%d launches in a timing-mode pass of the same %d fits"
                               % (est_launches, args.steps),
                     "peak_source": "measured packed-FP32 (fma.rn.f32x2) microbenchmark in this "
                                    "run (MEASURED_PEAKS.json has no FP32 figure); nominal %.1f"
                                    % NOMINAL_FP32_TFLOPS,
                     "traffic": TRAFFIC_BYTES,
                     "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, "
                                     "ncu --set full (%s); algorithmic %.0f B (points 16 B each "
                                     "+ FP64 partials)" % (TRAFFIC_SRC, 16 * n)},
        "clocks": clocks,
        "wall_s": wall,
        "device": {"sm_count": sm, "cc": "%d.%d" % (cc_major, cc_minor)},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, threads, times, cunits = cpu_fit_rate(pts, args.k, args.tol, args.cpu_sample_s)
        line["cpu_baseline"] = {
            "value": rate, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": "%d full cfg2 fit(s) (kinit + M + EM, %.1f s) with the FP64 oracle "
                      "restatement on all host threads" % (len(times), sum(times))}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
