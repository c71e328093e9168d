"""Every BASELINE configuration on one box: the GPU fit (device time, the
shipped kernels) and the CPU reference port (FP64 oracle, all host threads)
on a bounded sample. One JSON line per configuration; fills BASELINE.md's
result table (profiles/r2_all_configs.jsonl).

  cfg1  3D N=20,000 K=32, fixed init (oracle kinit + hard M step), 50 fixed
        iterations: GPU gmmb_fit_from vs oracle fit_from (full fit, both)
  cfg2  4D frame K=512, k-means++ + EM to tol 1e-3 (full fits, both)
  cfg3  64 frames K=256: GPU gmmb_fit_k_batch of all 64; CPU 2 frame fits
  cfg4  4M 3D map K=2048: GPU full fit to tol 1e-3; CPU 1 streaming EM
        iteration over a 250k-point slice (units/s)
  cfg5  K sweep on the cfg2 frame: GPU full fits; CPU 1 EM iteration from
        the oracle's k-means++ + hard M step (units/s)

usage: python scripts/all_configs.py [--cpu-budget-s 20]
"""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import oracle
import paper_2307_00071_b200 as gm
from bench import CFG4_CPU_SAMPLE, cfg4_cpu_init, cfg4_points, cpu_model

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
oracle.set_num_threads(0)
threads = oracle.num_threads()
ctx = gm.Context(0)


def gpu_fits(pts, k, em, reps=None):
    ctx.upload(pts)
    ctx.fit_k_resident(k, em)
    rs = [ctx.fit_k_resident(k, em) for _ in range(reps or args.reps)]
    return float(np.mean([r.ms_total for r in rs])), rs[-1]


def emit(**kw):
    kw["host_threads"] = threads
    kw["cpu_model"] = cpu_model()
    print(json.dumps(kw), flush=True)


# ---- cfg1 ------------------------------------------------------------------
p1 = gm.structured_scene(20000, 1, 0.005)[:, :3].copy()
lab, _ = oracle.kinit(p1, 32, 0)
w, mu, cov, _ = oracle.m_step_labels(p1, lab, 32, 1e-6)
w, mu, cov = w, mu[:, :3].copy(), cov[:, :6].copy()
em1 = gm.EmParams(50, 0.0, 1e-6, 0)
ctx_f = gm.Context(0)
gm.fit_from(p1, gm.Gmm(w, mu, cov), em1, ctx=ctx_f)
g = [gm.fit_from(p1, gm.Gmm(w, mu, cov), em1, ctx=ctx_f) for _ in range(args.reps)]
g_ms = float(np.mean([r.ms_total for r in g]))
t = time.perf_counter()
ref = oracle.fit_from(p1, w, mu, cov, max_iters=50, ll_rel_tol=0.0, cov_reg=1e-6)
c_ms = 1e3 * (time.perf_counter() - t)
units = 20000 * 32 * 50
emit(cfg="cfg1", gpu_ms_per_fit=g_ms, gpu_units_per_s=units / (g_ms * 1e-3),
     cpu_ms_per_fit=c_ms, cpu_units_per_s=units / (c_ms * 1e-3), speedup=c_ms / g_ms,
     cpu_sample="1 full fit (50 iterations)")

# ---- cfg2 ------------------------------------------------------------------
frame = gm.synthetic_frame_cloud()
em = gm.EmParams(100, 1e-3, 1e-6, 0)
g_ms, r = gpu_fits(frame, 512, em)
units = r.units
t = time.perf_counter()
ref = oracle.fit_k(frame, 512, max_iters=100, ll_rel_tol=1e-3, cov_reg=1e-6, seed=0)
c_ms = 1e3 * (time.perf_counter() - t)
emit(cfg="cfg2", gpu_ms_per_fit=g_ms, gpu_units_per_s=units / (g_ms * 1e-3),
     cpu_ms_per_fit=c_ms, cpu_units_per_s=len(frame) * 512 * ref["em_iterations"] / (c_ms * 1e-3),
     speedup=c_ms / g_ms, iterations=[r.em_iterations, ref["em_iterations"]],
     cpu_sample="1 full fit")

# ---- cfg3 ------------------------------------------------------------------
frames = [frame] + [gm.jitter_cloud(frame, 0.002, f) for f in range(1, 64)]
seeds = list(range(64))
gm.fit_k_batch(frames[:4], 256, em, seeds=seeds[:4], ctx=ctx)
ms = []
for _ in range(2):
    rs = gm.fit_k_batch(frames, 256, em, seeds=seeds, ctx=ctx)
    ms.append(sum(x.ms_total for x in rs))
g_ms = float(np.mean(ms))
g_units = sum(x.units for x in rs)
t = time.perf_counter()
cu = 0.0
for f in range(2):
    rr = oracle.fit_k(frames[f], 256, max_iters=100, ll_rel_tol=1e-3, cov_reg=1e-6, seed=f)
    cu += len(frame) * 256 * rr["em_iterations"]
c_s = time.perf_counter() - t
emit(cfg="cfg3", gpu_ms_per_batch=g_ms, gpu_frames_per_s=64 / (g_ms * 1e-3),
     gpu_units_per_s=g_units / (g_ms * 1e-3), cpu_ms_per_frame=1e3 * c_s / 2,
     cpu_frames_per_s=2 / c_s, cpu_units_per_s=cu / c_s,
     speedup=(64 / (g_ms * 1e-3)) / (2 / c_s), cpu_sample="2 frame fits (frames 0, 1)")

# ---- cfg4 ------------------------------------------------------------------
full = cfg4_points(gm)
g_ms, r = gpu_fits(full, 2048, em, reps=2)
sub = np.ascontiguousarray(full[:CFG4_CPU_SAMPLE])
w, mu, cov = cfg4_cpu_init(sub, 2048)
t = time.perf_counter()
oracle.fit_from(sub, w, mu, cov, max_iters=1, ll_rel_tol=0.0, cov_reg=1e-6, streaming=True)
c_s = time.perf_counter() - t
cpu_rate = len(sub) * 2048 / c_s
emit(cfg="cfg4", gpu_ms_per_fit=g_ms, gpu_units_per_s=r.units / (g_ms * 1e-3),
     gpu_stage_ms={"kinit": r.ms_kinit, "em": r.ms_em}, iterations=r.em_iterations,
     cpu_units_per_s=cpu_rate,
     cpu_ms_per_fit_estimate=r.units / cpu_rate * 1e3,
     speedup=(r.units / (g_ms * 1e-3)) / cpu_rate,
     cpu_sample="1 streaming EM iteration over a %d-point slice (%.1f s); the ms/fit estimate "
                "scales the EM rate to the GPU fit's units (kinit excluded)" % (len(sub), c_s))
del full

# ---- cfg5 ------------------------------------------------------------------
for k in (64, 128, 256, 512, 1024, 2048, 4096):
    g_ms, r = gpu_fits(frame, k, em, reps=2)
    lab, _ = oracle.kinit(frame, k, 0)
    w, mu, cov, _ = oracle.m_step_labels(frame, lab, k, 1e-6)
    t = time.perf_counter()
    oracle.fit_from(frame, w, mu, cov, max_iters=1, ll_rel_tol=0.0, cov_reg=1e-6, streaming=True)
    c_s = time.perf_counter() - t
    cpu_rate = len(frame) * k / c_s
    emit(cfg="cfg5", k=k, gpu_ms_per_fit=g_ms, gpu_units_per_s=r.units / (g_ms * 1e-3),
         iterations=r.em_iterations, cpu_units_per_s=cpu_rate,
         speedup=(r.units / (g_ms * 1e-3)) / cpu_rate,
         cpu_sample="1 streaming EM iteration from the oracle's k-means++ + hard M step (%.1f s)" % c_s)
