"""Runs cfg-style fits on the resident cloud (for ncu / timing)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00071_b200 as gm

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=512)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--tol", type=float, default=1e-3)
args = ap.parse_args()
ctx = gm.Context(0)
if os.environ.get("GMMB_TIMING", "0") == "1":
    ctx.set_timing(True)
p = gm.synthetic_frame_cloud()
ctx.upload(p)
for _ in range(args.reps):
    r = ctx.fit_k_resident(args.k, gm.EmParams(100, args.tol, 1e-6, 0))
    print(f"iters {r.em_iterations} kinit {r.ms_kinit:.3f} m0 {r.ms_mstep0:.3f} em {r.ms_em:.3f} "
          f"estep {r.ms_estep:.3f} ms ({r.ms_estep / max(r.em_iterations, 1) * 1e3:.1f} us/iter) "
          f"total {r.ms_total:.3f}", flush=True)
