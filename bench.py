#!/usr/bin/env python
"""Benchmark: EM point*component*iterations/s and ms per GMM fit (BASELINE.json).

A step is one full GMM fit of the hot path (layout -> kinit (k-means++) ->
initial M step -> EM to tolerance) on one batch of synthetic input.

--config cfg2 (default; BASELINE cfg2): one 640x480 synthetic depth frame ->
    307,200 4D points, K=512, seed 0, ll_rel_tol 1e-3, cov_reg 1e-6. With
    N > 1 GPUs (torchrun) each rank fits its own frame (frame r jittered by
    2 mm, seed r: cfg3-style frame replicas, weak scaling, no collective on
    the data path); the job value is all ranks' units over the max-over-ranks
    time.
--config cfg4 (BASELINE cfg4): the 4M-point 3D map (make_structured_scene x 25
    + (100, -40, 0) m), K=2048, tol 1e-3. With N > 1 the points are sharded
    contiguously over the ranks (one NCCL communicator; per-iteration
    statistics all-reduce; k-means++ seeds the all-gathered cloud): strong
    scaling, value = global units / max-over-ranks time. --vshard G runs the
    same sharded path as G virtual ranks on one GPU (protocol check, not a
    scaling number).

value  = sum of units (N * K_t per E step) / device time of the fits, inputs
         resident in HBM (CUDA events inside the library around each fit;
         L2 flushed between steps).
e2e    = the same metric through the C ABI call with host (pinned) buffers:
         H2D of the points and D2H of the model inside the timed region.
--impl reference times the reference algorithm on the host CPU (the FP64
oracle port, all host threads; the reference itself cannot be built here),
building its inputs with the oracle's restatement of the reference
generators — it never loads libgmmb.
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
# DRAM traffic per launch of the dominant kernel, from ncu --set full
# captures of exactly these configurations and kernels (emitted only when the
# run matches the capture; re-captured on every kernel change).
# (config, K, E-step kind) -> (bytes per E step: the three pruned-E kernels'
# dram__bytes_read.sum + dram__bytes_write.sum, source). ncu replays with
# flushed caches, so the per-(unit, candidate) statistics the reduce reads
# (L2-resident between the kernels in situ) count as DRAM reads here.
TRAFFIC = {
    ("cfg2", 512, "sparse"): (6.3744e4 + 6.002432e6 + 1.6128e4 + 1.67936e7 + 5.12e2,
                              "profiles/r2bc_cfg2_sparse_ncu.txt"),
    ("cfg4", 2048, "sparse"): (2.97728e5 + 1.536e4 + 9.4760192e7 + 1.16638976e8 + 1.63354112e8
                               + 2.7361024e7, "profiles/r2bc_cfg4_sparse_ncu.txt"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="gmmb", choices=["gmmb", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg3", "cfg4"])
    ap.add_argument("--frames", type=int, default=64, help="cfg3: frames per step")
    ap.add_argument("--k", type=int, default=0, help="override K (0: the config's)")
    ap.add_argument("--tol", type=float, default=1e-3)
    ap.add_argument("--max-iters", type=int, default=100,
                    help="EM iteration cap (cfg4 with --tol 0 --max-iters 20: the fixed-20-"
                         "iteration throughput mode of SURVEY.md §8(d))")
    ap.add_argument("--vshard", type=int, default=0,
                    help="cfg4 on one GPU as G virtual ranks (sharded-path check)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=20.0)
    a = ap.parse_args()
    if a.k == 0:
        a.k = {"cfg2": 512, "cfg3": 256, "cfg4": 2048}[a.config]
    return a


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---- inputs: `gen` is the product's host generators (GPU arm) or the
# oracle's restatement of the reference generators (reference arm, which
# must not load libgmmb); the two are bit-identical (tests/test_abi.py) ------
def cfg2_points(gen, rank):
    p = gen.synthetic_frame_cloud()             # make_synthetic_frame + image_pair_to_cloud
    if rank > 0:                                # cfg3 frame r: xyz jittered 2 mm, seed r
        p = gen.jitter_cloud(p, 0.002, rank)
    return p


def cfg4_points(gen):
    s = gen.structured_scene(4_000_000, 4, 0.005)[:, :3]
    return s * 25.0 + np.array([100.0, -40.0, 0.0])


def shard_bounds(n, world):
    q, r = divmod(n, world)
    out, lo = [], 0
    for i in range(world):
        hi = lo + q + (1 if i < r else 0)
        out.append((lo, hi))
        lo = hi
    return out


def config_dict(args, world):
    """Identical for both arms (the driver compares them)."""
    if args.config == "cfg3":
        return {"workload": "cfg3: batch of %d 4D frames (N=307200 each, 2 mm jitter, seed f), "
                            "K=%d each, k-means++ + EM to tol %g, frames sharded over the GPUs "
                            "(f mod N)" % (args.frames, args.k, args.tol),
                "global_batch": args.frames, "points_per_fit": 307200, "k": args.k,
                "parallelism": "frames%d" % world}
    if args.config == "cfg2":
        return {"workload": "cfg2: 4D frame N=307200, K=%d, k-means++ + EM to tol %g "
                            "(one fit per GPU per step)" % (args.k, args.tol),
                "global_batch": world, "points_per_fit": 307200, "k": args.k,
                "parallelism": "replicas%d" % world,
                "l2": "flushed between steps (256 MiB write)"}
    par = "shard%d" % world if world > 1 else ("vshard%d" % args.vshard if args.vshard else "1")
    its = "" if args.max_iters == 100 else ", at most %d iterations" % args.max_iters
    return {"workload": "cfg4: 3D map N=4000000, K=%d, k-means++ + EM to tol %g%s "
                        "(one fit per step, points sharded over the GPUs)" % (args.k, args.tol, its),
            "global_batch": 1, "points_per_fit": 4_000_000, "k": args.k, "parallelism": par,
            "l2": "flushed between steps (256 MiB write); inputs 96 MB > L2"}


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
                rows.append(parts)
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


# ---- CPU reference (oracle port) ---------------------------------------------
def cpu_cfg2_rate(points, k, tol, budget_s, steps=None):
    """Full cfg2 fits with the FP64 oracle port on all host threads."""
    import oracle
    oracle.set_num_threads(0)
    threads = oracle.num_threads()
    times, units = [], []
    t_end = time.time() + budget_s
    n = len(points)
    while True:
        t0 = time.perf_counter()
        r = oracle.fit_k(points, k, max_iters=100, ll_rel_tol=tol, cov_reg=1e-6, seed=0)
        times.append(time.perf_counter() - t0)
        units.append(float(n) * k * r["em_iterations"])
        if steps is not None:
            if len(times) >= steps:
                break
        elif time.time() > t_end or len(times) >= 3:
            break
    sample = ("%d full cfg2 fit(s) (kinit + M + EM, %.1f s), FP64 oracle restatement, "
              "std::thread fan-out over 4096-point blocks" % (len(times), sum(times)))
    return sum(units) / sum(times), threads, times, sample


CFG4_CPU_SAMPLE = 250_000


def cfg4_cpu_init(points, k):
    """Fixed initial model for the CPU cfg4 sample: K evenly strided points,
    equal weights, isotropic 5 cm covariance (iteration cost is independent
    of the model's values)."""
    idx = np.linspace(0, len(points) - 1, k).astype(np.int64)
    mu = points[idx].copy()
    w = np.full(k, 1.0 / k)
    cov = np.zeros((k, 6))
    cov[:, [0, 2, 5]] = 0.05 ** 2
    return w, mu, cov


def cpu_cfg4_rate(points, k, steps):
    """Bounded sample of cfg4 on the CPU: one streaming FP64 EM iteration
    (E + M, sogmm.cpp:488-503 without the N x K matrix) over a contiguous
    250,000-point slice of the map, per step."""
    import oracle
    oracle.set_num_threads(0)
    threads = oracle.num_threads()
    sub = np.ascontiguousarray(points[:CFG4_CPU_SAMPLE])
    w, mu, cov = cfg4_cpu_init(sub, k)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.fit_from(sub, w, mu, cov, max_iters=1, ll_rel_tol=0.0, cov_reg=1e-6,
                        streaming=True)
        times.append(time.perf_counter() - t0)
    units = float(len(sub)) * k * len(times)
    sample = ("%d streaming FP64 EM iteration(s) (E + M) over a contiguous %d-point slice "
              "of the cfg4 map, K=%d (%.1f s), oracle restatement" %
              (len(times), len(sub), k, sum(times)))
    return units / sum(times), threads, times, sample


def cpu_cfg3_rate(gen, k, tol, steps):
    """cfg3 on the CPU: the reference's serial loop of fits over the frames,
    a bounded sample of it per step (frame s of the batch, seed s)."""
    import oracle
    oracle.set_num_threads(0)
    threads = oracle.num_threads()
    base = gen.synthetic_frame_cloud()
    times, units = [], []
    for f in range(steps):
        p = gen.jitter_cloud(base, 0.002, f) if f > 0 else base
        t0 = time.perf_counter()
        r = oracle.fit_k(p, k, max_iters=100, ll_rel_tol=tol, cov_reg=1e-6, seed=f)
        times.append(time.perf_counter() - t0)
        units.append(float(len(p)) * k * r["em_iterations"])
    sample = ("%d frame fit(s) of the cfg3 batch (frames 0..%d, K=%d, kinit + M + EM, %.1f s), "
              "FP64 oracle restatement" % (len(times), len(times) - 1, k, sum(times)))
    return sum(units) / sum(times), threads, times, sample


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    if args.config == "cfg3":
        cpu_cfg3_rate(oracle, args.k, args.tol, 1)
        rate, threads, times, sample = cpu_cfg3_rate(oracle, args.k, args.tol,
                                                     max(args.steps, 1))
    elif args.config == "cfg2":
        pts = cfg2_points(oracle, 0)
        if args.warmup > 0:
            cpu_cfg2_rate(pts, args.k, args.tol, 0, steps=min(args.warmup, 2))
        rate, threads, times, sample = cpu_cfg2_rate(pts, args.k, args.tol, 0,
                                                     steps=max(args.steps, 1))
    else:
        pts = cfg4_points(oracle)
        cpu_cfg4_rate(pts, args.k, 1)
        rate, threads, times, sample = cpu_cfg4_rate(pts, args.k, max(args.steps, 1))
    ms = 1e3 * sum(times) / len(times)
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak" if args.config == "cfg2" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (oracle restatement of the reference generators)",
        "config": config_dict(args, args.gpus),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def flush_l2(buf):
    buf.add_(1.0)  # 256 MiB write > 126 MB L2


# ---- GPU arm --------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    rank, world, local = dist_env()
    import torch
    import paper_2307_00071_b200 as gm

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.config == "cfg3":
        run_cfg3(args, gm, torch, dist, rank, world, local)
        return
    sharded = args.config == "cfg4" and world > 1
    vshard = args.config == "cfg4" and world == 1 and args.vshard > 1
    if sharded:
        ids = [gm.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        ctx = gm.Context(local, rank, world, ids[0])
    else:
        ctx = gm.Context(local)
    sm, cc_major, cc_minor = ctx.device_info()
    if args.config == "cfg2":
        pts = cfg2_points(gm, rank)
        em = gm.EmParams(args.max_iters, args.tol, 1e-6, rank)
        full_n = len(pts)
    else:
        full = cfg4_points(gm)
        full_n = len(full)
        em = gm.EmParams(args.max_iters, args.tol, 1e-6, 0)
        if sharded:
            lo, hi = shard_bounds(full_n, world)[rank]
            pts = np.ascontiguousarray(full[lo:hi])
        else:
            lo, hi = 0, full_n
            pts = full
    n, d = pts.shape
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    vctx = gm.vshard_contexts(args.vshard) if vshard else None

    def fit_resident():
        if vshard:
            rs = gm.fit_k_vsharded(pts, args.k, em, contexts=vctx)
            r0 = rs[0]
            r0.ms_total = max(r.ms_total for r in rs)
            r0.ms_em = max(r.ms_em for r in rs)
            r0.ms_estep = max(r.ms_estep for r in rs)
            r0.launches = sum(r.launches for r in rs)
            return r0
        return ctx.fit_k_resident(args.k, em)

    # ---- value: inputs resident in HBM ------------------------------------
    if not vshard:
        if sharded:
            ctx.upload(pts, lo, full_n)
        else:
            ctx.upload(pts)
    res = []
    with Clocks(local) as clk:          # sampling spans warm-up + timed region
        for _ in range(max(args.warmup, 3)):
            fit_resident()
        flush_l2(flush)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush_l2(flush)
            torch.cuda.synchronize()
            res.append(fit_resident())
        barrier()
        wall = time.perf_counter() - t0
    clocks = clk.summary()
    dev_ms = sum(r.ms_total for r in res)
    em_ms = sum(r.ms_em for r in res)
    units = sum(r.units for r in res)   # units count the GLOBAL N (sharded: every rank the same)
    iters = [r.em_iterations for r in res]
    if world > 1:
        t = torch.tensor([dev_ms, em_ms, units], dtype=torch.float64, device="cuda")
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        dev_ms_job, em_ms_job = float(mx[0]), float(mx[1])
        units_job = float(mx[2]) if sharded else float(t[2])
    else:
        dev_ms_job, em_ms_job, units_job = dev_ms, em_ms, units
    value = units_job / (dev_ms_job * 1e-3)

    # ---- e2e: C ABI call with pinned host buffers --------------------------
    host = torch.empty((d, n), dtype=torch.float64, pin_memory=True)
    host.numpy()[:] = pts.T                      # column-major N x D
    host_pts = host.numpy().T                    # (N, D) Fortran view, pinned
    assert host_pts.flags["F_CONTIGUOUS"]

    def fit_host():
        if vshard:
            return gm.fit_k_vsharded(host_pts, args.k, em, contexts=vctx)[0]
        return gm.fit_k(host_pts, args.k, em, ctx=ctx)

    for _ in range(2):
        fit_host()
    barrier()
    e2e_units, t_e2e = 0.0, 0.0
    for _ in range(args.steps):
        flush_l2(flush)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t1 = time.perf_counter()
        r = fit_host()
        torch.cuda.synchronize()
        t_e2e += time.perf_counter() - t1
        e2e_units += r.units
    if world > 1:
        t = torch.tensor([t_e2e, e2e_units], dtype=torch.float64, device="cuda")
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        t_e2e = float(mx[0])
        e2e_units = float(mx[1]) if sharded else float(t[1])
    e2e = e2e_units / t_e2e
    kk = args.k
    d2h = 8 * (kk * (1 + d + d * (d + 1) // 2) + 100) + 96

    # ---- roofline of the dominant kernel (fused E step + statistics) ------
    # Graph mode has no per-kernel events inside the EM loop: the same fits
    # are repeated in timing mode (chunked launches, CUDA events on the
    # library stream around every fused E kernel; identical kernels and
    # results). Sharded fits always run chunked, so their pass above has them.
    # The E step evaluates only the (point, component) pairs whose FP32
    # density can be non-zero (exact-zero pruning, estep_sparse.cu): the
    # roofline is taken on the pairs it evaluated (units_evaluated); the
    # dense-equivalent rate and the dense kernels' own fraction (same fits,
    # GMMB dense mode) are reported beside it.
    def timed_estep(dense):
        ctx.set_estep_mode(dense)
        ctx.set_timing(True)
        ms, units_, ev, launches = 0.0, 0.0, 0.0, 0
        for _ in range(args.steps if not dense else max(2, args.steps // 4)):
            flush_l2(flush)
            torch.cuda.synchronize()
            rt = ctx.fit_k_resident(args.k, em)
            ms += rt.ms_estep
            units_ += rt.units
            ev += rt.units_evaluated
            launches += rt.em_iterations
        ctx.set_timing(False)
        ctx.set_estep_mode(False)
        return ms, units_, ev, launches

    dense_cmp = None
    if sharded or vshard:
        est_ms = sum(r.ms_estep for r in res)
        est_units = float(n if sharded else -(-full_n // args.vshard)) * kk * sum(iters)
        est_eval = sum(r.units_evaluated for r in res) * (est_units / max(units, 1.0))
        est_launches = sum(iters)
    else:
        ctx.upload(pts)
        est_ms, est_units, est_eval, est_launches = timed_estep(False)
        d_ms, d_units, _, d_launches = timed_estep(True)
        dense_cmp = (d_ms, d_units, d_launches)
    peak_tf, _ = ctx.ffma_peak(50.0)
    pruned = est_eval < est_units
    achieved_tf = FLOP_PER_UNIT[d] * est_eval / (est_ms * 1e-3) / 1e12
    dense_equiv_tf = FLOP_PER_UNIT[d] * est_units / (est_ms * 1e-3) / 1e12
    tr = (TRAFFIC.get((args.config, kk, "sparse" if pruned else "dense"))
          if world == 1 and not vshard else None)
    kernel = ("E step = block_cand_kernel + estep_sparse_kernel (exact-zero-pruned fused E "
              "step + sufficient statistics) + sparse_reduce_kernel" if pruned else
              "estep_ws_kernel (warp-specialised fused E step + sufficient statistics)"
              if kk <= 512 else "fused E step + sufficient statistics (K > 512 path)")

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": dev_ms_job / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.config == "cfg4" else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": ("synthetic (make_synthetic_frame 640x480 -> 307,200 4D points; rank r>0: "
                 "2 mm jitter, seed r)" if args.config == "cfg2" else
                 "synthetic (make_structured_scene 4M x 25 + (100, -40, 0) m, 3D)"),
        "config": config_dict(args, world),
        "em_iterations": iters,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": n * d * 8,
                "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * t_e2e / args.steps},
        "gpu_launches": int(sum(r.launches for r in res)),
        "stage_ms": {"layout": statistics.mean(r.ms_layout for r in res),
                     "kinit": statistics.mean(r.ms_kinit for r in res),
                     "mstep0": statistics.mean(r.ms_mstep0 for r in res),
                     "em": statistics.mean(r.ms_em for r in res),
                     "estep_kernel": est_ms / args.steps,
                     "estep_us_per_launch": 1e3 * est_ms / max(est_launches, 1)},
        "em_only_value": units_job / (em_ms_job * 1e-3),
        "roofline": {"bound": "fp32", "kernel": kernel, "achieved": achieved_tf,
                     "peak": peak_tf, "unit": "TFLOP/s", "frac": achieved_tf / peak_tf,
                     "flop_per_unit": FLOP_PER_UNIT[d],
                     "units_evaluated_fraction": est_eval / max(est_units, 1.0),
                     "achieved_note": ("FLOP of the (point, component) pairs the pruned E step "
                                       "evaluated (the skipped pairs have FP32 density exactly 0) "
                                       "over the E-step time" if pruned else
                                       "FLOP of every (point, component) pair over the E time"),
                     "dense_equivalent_tflops": dense_equiv_tf,
                     "dense_kernels": ({"us_per_iteration": 1e3 * dense_cmp[0] / max(dense_cmp[2], 1),
                                        "tflops": FLOP_PER_UNIT[d] * dense_cmp[1]
                                        / (dense_cmp[0] * 1e-3) / 1e12,
                                        "frac": FLOP_PER_UNIT[d] * dense_cmp[1]
                                        / (dense_cmp[0] * 1e-3) / 1e12 / peak_tf}
                                       if dense_cmp else None),
                     "timing": "CUDA events around each E step (all its kernels) on the library "
                               "stream, %d iterations over %d fits" % (est_launches, args.steps),
                     "bound_note": ("the pruned E step is latency-bound, not FP32-bound: 16 warps "
                                    "per SM (128 registers), issue slots ~40 % active, the per-unit "
                                    "candidate filter and statistics hand-off are memory round trips "
                                    "(profiles/r2bc_cfg2_sparse_ncu.txt, r2au_sparse_source_stalls.txt); "
                                    "it evaluates ~5 % of the pairs and takes less time than the "
                                    "dense kernels would at their 0.60 target"
                                    if pruned else None),
                     "peak_source": "measured packed-FP32 (fma.rn.f32x2) microbenchmark in this "
                                    "run (MEASURED_PEAKS.json has no FP32 figure); nominal %.1f"
                                    % NOMINAL_FP32_TFLOPS,
                     "traffic": tr[0] if tr else None,
                     "traffic_note": ("dram__bytes_read.sum + dram__bytes_write.sum per E step "
                                      "(its three kernels), ncu --set full of this configuration "
                                      "(%s; cold caches: the statistics pool the reduce reads is "
                                      "L2-resident in situ); algorithmic %.0f B (points 16 B each)"
                                      % (tr[1], 16 * n)) if tr else
                                     "no ncu capture of this configuration; algorithmic "
                                     "%.0f B per launch (points 16 B each)" % (16 * n)},
        "clocks": clocks,
        "wall_s": wall,
        "device": {"sm_count": sm, "cc": "%d.%d" % (cc_major, cc_minor)},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.config == "cfg2":
            rate, threads, times, sample = cpu_cfg2_rate(pts, args.k, args.tol, args.cpu_sample_s)
        else:
            rate, threads, times, sample = cpu_cfg4_rate(pts, args.k, 3)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                                "cpu_model": cpu_model(), "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if vctx:
        for c in vctx:
            c.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def run_cfg3(args, gm, torch, dist, rank, world, local):
    """cfg3: a step fits the whole batch of frames; frame f (2 mm jitter,
    seed f) runs on rank f mod N through gmmb_fit_k_batch (the next frame's
    copy overlaps the current fit). value: frames resident in HBM, the batch
    call bracketed by CUDA events on the launching side (includes every
    per-frame host round trip); e2e: the same call with pinned host frames."""
    ctx = gm.Context(local)
    sm, cc_major, cc_minor = ctx.device_info()
    base = gm.synthetic_frame_cloud()
    mine = [f for f in range(args.frames) if f % world == rank]
    host = []
    for f in mine:
        p = gm.jitter_cloud(base, 0.002, f) if f > 0 else base
        t = torch.empty((4, len(p)), dtype=torch.float64, pin_memory=True)
        t.numpy()[:] = p.T
        host.append(t)
    dev = [t.cuda() for t in host]
    host_views = [t.numpy().T for t in host]          # (N, 4) Fortran views, pinned
    em = gm.EmParams(args.max_iters, args.tol, 1e-6, 0)
    seeds = mine
    n = len(base)

    def run_batch(frames_dev):
        # device pointers: call the C ABI directly (the Python wrapper takes host arrays)
        import ctypes
        F = len(frames_dev)
        ptrs = (ctypes.POINTER(ctypes.c_double) * F)(
            *[ctypes.cast(ctypes.c_void_p(t.data_ptr()), ctypes.POINTER(ctypes.c_double))
              for t in frames_dev])
        ns = np.full(F, n, dtype=np.int64)
        sd = np.array(seeds, dtype=np.uint64)
        st = (gm._FitStats * F)()
        gm._check(gm.load().gmmb_fit_k_batch(
            ctx.handle, F, ptrs, ns.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 4, args.k,
            ctypes.byref(em._c()), sd.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
            None, None, None, st))
        return [st[f] for f in range(F)]

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    res, ms = [], 0.0
    with Clocks(local) as clk:
        for _ in range(max(args.warmup, 3) if args.warmup > 0 else 3):
            run_batch(dev)
        barrier()
        steps = args.steps
        for _ in range(steps):
            flush.add_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res.append(run_batch(dev))
            e1.record()
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
        barrier()
    clocks = clk.summary()
    units = sum(s.units for r in res for s in r)
    dev_ms = sum(s.ms_total for r in res for s in r)
    launches = sum(s.launches for r in res for s in r)
    est_ms = 0.0
    # e2e: pinned host frames through the same call
    t_e2e, e2e_units = 0.0, 0.0
    for _ in range(max(1, steps // 2)):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t1 = time.perf_counter()
        rr = gm.fit_k_batch(host_views, args.k, em, seeds=seeds, ctx=ctx)
        torch.cuda.synchronize()
        t_e2e += time.perf_counter() - t1
        e2e_units += sum(r.units for r in rr)
    e2e_steps = max(1, steps // 2)
    # roofline: the fused E kernel per launch in timing mode on one frame
    ctx.upload(host_views[0])
    ctx.set_timing(True)
    tf = [ctx.fit_k_resident(args.k, gm.EmParams(args.max_iters, args.tol, 1e-6, seeds[0])) for _ in range(3)]
    ctx.set_timing(False)
    est_ms = sum(r.ms_estep for r in tf)
    est_units = sum(r.units for r in tf)
    est_eval = sum(r.units_evaluated for r in tf)
    est_launches = sum(r.em_iterations for r in tf)
    if world > 1:
        t = torch.tensor([ms, units, t_e2e, e2e_units, dev_ms], dtype=torch.float64, device="cuda")
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        ms_job, units_job, t_e2e_job, e2e_units_job = float(mx[0]), float(t[1]), float(mx[2]), float(t[3])
    else:
        ms_job, units_job, t_e2e_job, e2e_units_job = ms, units, t_e2e, e2e_units
    peak_tf, _ = ctx.ffma_peak(50.0)
    achieved_tf = FLOP_PER_UNIT[4] * est_eval / (est_ms * 1e-3) / 1e12
    pruned = est_eval < est_units
    line = {
        "metric": METRIC, "value": units_job / (ms_job * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_job / steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (make_synthetic_frame 640x480 -> 307,200 4D points; frame f: 2 mm "
                "jitter, seed f)",
        "config": config_dict(args, world),
        "frames_per_s": args.frames * steps / (ms_job * 1e-3),
        "e2e": {"value": e2e_units_job / t_e2e_job, "unit": UNIT,
                "h2d_bytes_per_step": len(mine) * n * 4 * 8,
                "d2h_bytes_per_step": len(mine) * 8 * args.k * 15,
                "ms_per_step": 1e3 * t_e2e_job / e2e_steps,
                "frames_per_s": args.frames * e2e_steps / t_e2e_job},
        "gpu_launches": int(launches),
        "device_ms_per_step_sum_of_fits": dev_ms / steps,
        "roofline": {"bound": "fp32", "kernel": ("pruned E step (block_cand + estep_sparse + "
                     "sparse_reduce), K=%d" if pruned else "estep_ws_kernel (fused E step + "
                     "statistics, K=%d)") % args.k, "achieved": achieved_tf, "peak": peak_tf,
                     "unit": "TFLOP/s", "frac": achieved_tf / peak_tf,
                     "flop_per_unit": FLOP_PER_UNIT[4],
                     "units_evaluated_fraction": est_eval / max(est_units, 1.0),
                     "dense_equivalent_tflops": FLOP_PER_UNIT[4] * est_units / (est_ms * 1e-3) / 1e12,
                     "timing": "CUDA events around each E step, %d iterations (3 fits of "
                               "frame %d in timing mode)" % (est_launches, seeds[0]),
                     "peak_source": "measured packed-FP32 microbenchmark in this run",
                     "traffic": None,
                     "traffic_note": "no ncu capture of this configuration; algorithmic %.0f B "
                                     "per launch" % (16 * n)},
        "clocks": clocks,
        "device": {"sm_count": sm, "cc": "%d.%d" % (cc_major, cc_minor)},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, threads, times, sample = cpu_cfg3_rate(gm, args.k, args.tol, 2)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                                "cpu_model": cpu_model(), "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
