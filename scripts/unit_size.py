"""Pruned E step per work-unit size (GMMB_SPARSE_U, child processes): fit
and E-step time on the cfg2 frame (K = 512, 2048) and cfg4."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = """
import json, numpy as np, paper_2307_00071_b200 as gm
ctx = gm.Context(0)
out = {}
f = gm.synthetic_frame_cloud()
for k in (512, 2048):
    ctx.upload(f)
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    ctx.fit_k_resident(k, em)
    g = [ctx.fit_k_resident(k, em) for _ in range(3)]
    ctx.set_timing(True)
    t = [ctx.fit_k_resident(k, em) for _ in range(2)]
    ctx.set_timing(False)
    out[k] = (float(np.mean([x.ms_total for x in g])), float(np.mean([x.ms_em for x in g])),
              1e3 * sum(x.ms_estep for x in t) / sum(x.em_iterations for x in t))
print(json.dumps(out))
"""
for u in ("1", "2", "4"):
    r = subprocess.run([sys.executable, "-c", CODE], env=dict(os.environ, GMMB_SPARSE_U=u), cwd=ROOT,
                       capture_output=True, text=True)
    print("U", u, r.stdout.strip()[-300:], r.stderr[-300:], flush=True)
