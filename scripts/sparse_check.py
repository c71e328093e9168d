"""Pruned vs dense E step on the same fit: iterations, ll and parameter
differences, E-step time per iteration (timing mode), evaluated fraction.

usage: python scripts/sparse_check.py [--ks 64,512,2048,4096] [--cfg4]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2307_00071_b200 as gm

ap = argparse.ArgumentParser()
ap.add_argument("--ks", default="64,256,512,1024,2048,4096")
ap.add_argument("--cfg4", action="store_true")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
ctx = gm.Context(0)


def fit(pts, k, em, dense, timing):
    ctx.set_estep_mode(dense)
    ctx.set_timing(timing)
    return ctx.fit_k_resident(k, em)


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-12)))


def run(name, pts, k, em):
    ctx.upload(pts)
    out = {"config": name, "n": len(pts), "k": k}
    res = {}
    for dense in (True, False):
        fit(pts, k, em, dense, False)
        g = [fit(pts, k, em, dense, False) for _ in range(args.reps)]
        t = [fit(pts, k, em, dense, True) for _ in range(args.reps)]
        r = g[-1]
        tag = "dense" if dense else "sparse"
        res[tag] = r
        out[tag] = {"iters": r.em_iterations, "ms_fit": round(float(np.mean([x.ms_total for x in g])), 3),
                    "ms_em": round(float(np.mean([x.ms_em for x in g])), 3),
                    "estep_us_per_iter": round(1e3 * sum(x.ms_estep for x in t) /
                                               max(1, sum(x.em_iterations for x in t)), 1),
                    "evaluated_frac": round(r.units_evaluated / max(r.units, 1.0), 4)}
    a, b = res["sparse"], res["dense"]
    out["same_iters"] = a.em_iterations == b.em_iterations
    out["ll_rel"] = abs(a.final_log_likelihood - b.final_log_likelihood) / abs(b.final_log_likelihood)
    if a.model.weights.shape == b.model.weights.shape:
        out["w_rel"] = rel(a.model.weights, b.model.weights)
        out["mu_rel"] = rel(a.model.means, b.model.means)
        out["cov_rel"] = rel(a.model.covariances, b.model.covariances)
    print(json.dumps(out), flush=True)


frame = gm.synthetic_frame_cloud()
for k in [int(x) for x in args.ks.split(",") if x]:
    run("cfg5", frame, k, gm.EmParams(100, 1e-3, 1e-6, 0))
if args.cfg4:
    s = gm.structured_scene(4_000_000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
    run("cfg4", s, 2048, gm.EmParams(100, 1e-3, 1e-6, 0))
