"""cfg5 K sweep (K = 64 ... 4096 on the cfg2 frame, k-means++ + EM to tol
1e-3) and cfg4 (4M-point 3D map, K = 2048): per-stage times and the fused
E kernel's roofline fraction (timing mode: CUDA events around every E
launch). One JSON line per configuration.

usage: python scripts/ksweep.py [--ks 64,128,...] [--cfg4]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2307_00071_b200 as gm
from bench import Clocks

FLOP = {4: 62.0, 3: 42.0}
ap = argparse.ArgumentParser()
ap.add_argument("--ks", default="64,128,256,512,1024,2048,4096")
ap.add_argument("--cfg4", action="store_true")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
ctx = gm.Context(0)
peak, _ = ctx.ffma_peak(50.0)


def run(name, pts, k, em):
    ctx.upload(pts)
    ctx.set_timing(False)
    ctx.fit_k_resident(k, em)                      # warm-up (graph build)
    with Clocks(0) as clk:                         # nvidia-smi clocks during the timed fits
        gr = [ctx.fit_k_resident(k, em) for _ in range(args.reps)]
        ctx.set_timing(True)
        tr = [ctx.fit_k_resident(k, em) for _ in range(args.reps)]
        ctx.set_timing(False)
    d = pts.shape[1]
    r = gr[-1]
    est = sum(t.ms_estep for t in tr)
    units = sum(t.units for t in tr)
    it = sum(t.em_iterations for t in tr)
    ach = FLOP[d] * units / (est * 1e-3) / 1e12
    print(json.dumps({
        "config": name, "n": len(pts), "d": d, "k": k, "em_iterations": r.em_iterations,
        "ms_fit": round(float(np.mean([g.ms_total for g in gr])), 3),
        "ms_kinit": round(r.ms_kinit, 3), "ms_mstep0": round(r.ms_mstep0, 3),
        "ms_em": round(r.ms_em, 3), "estep_us_per_iter": round(1e3 * est / it, 1),
        "units_per_s": units / (sum(g.ms_total for g in gr) * 1e-3) * len(gr) / len(tr),
        "estep_tflops": round(ach, 2), "roofline_frac": round(ach / peak, 3),
        "peak_tflops": round(peak, 1), "clocks": clk.summary()}), flush=True)


frame = gm.synthetic_frame_cloud()
for k in [int(x) for x in args.ks.split(",") if x]:
    run("cfg5", frame, k, gm.EmParams(100, 1e-3, 1e-6, 0))
if args.cfg4:
    s = gm.structured_scene(4_000_000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
    run("cfg4 (20 fixed iterations)", s, 2048, gm.EmParams(20, 0.0, 1e-6, 0))
