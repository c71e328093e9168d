"""Times the fused E kernel (cfg2 frame, K given) for alternative builds of
libgmmb.so (GMMB_LIB=...): timing-mode fits, CUDA events around every E
launch. Prints one JSON line per library.

usage: python scripts/estep_variants.py lib1.so lib2.so ... [--k 512]
"""
import argparse, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--k", type=int, default=512)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--child", action="store_true")
args = ap.parse_args()

if args.child:
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_2307_00071_b200 as gm
    ctx = gm.Context(0)
    peak, _ = ctx.ffma_peak(30.0)
    p = gm.synthetic_frame_cloud()
    ctx.upload(p)
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    ctx.fit_k_resident(args.k, em)
    g = [ctx.fit_k_resident(args.k, em) for _ in range(args.reps)]
    ctx.set_timing(True)
    t = [ctx.fit_k_resident(args.k, em) for _ in range(args.reps)]
    est = sum(r.ms_estep for r in t)
    it = sum(r.em_iterations for r in t)
    units = sum(r.units for r in t)
    ach = 62.0 * units / (est * 1e-3) / 1e12
    print(json.dumps({"lib": args.libs[0], "k": args.k, "iters": t[-1].em_iterations,
                      "ll": t[-1].final_log_likelihood,
                      "ms_fit": float(np.mean([r.ms_total for r in g])),
                      "ms_em": float(np.mean([r.ms_em for r in g])),
                      "estep_us": 1e3 * est / it, "frac": ach / peak, "peak": peak}), flush=True)
else:
    for lib in args.libs:
        env = dict(os.environ, GMMB_LIB=os.path.abspath(lib))
        subprocess.run([sys.executable, __file__, lib, "--k", str(args.k), "--reps",
                        str(args.reps), "--child"], env=env)
