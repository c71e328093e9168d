"""A/B of library builds on full fits (graph mode): cfg2 K=512, the cfg2 frame
at K=2048, cfg4 (4M 3D points, K=2048). usage: python scripts/ab_fits.py
lib1.so [lib2.so ...] (each in a child process, GMMB_LIB)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r"""
import os, sys, numpy as np
sys.path.insert(0, %r)
import paper_2307_00071_b200 as gm
ctx = gm.Context(0)
out = []
for name in os.environ.get("AB_CONFIGS", "cfg2,k2048,cfg4").split(","):
    if name == "cfg4":
        p = gm.structured_scene(4_000_000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
        k = 2048
    else:
        p = gm.synthetic_frame_cloud()
        k = 512 if name == "cfg2" else int(name[1:])
    ctx.upload(p)
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    ctx.fit_k_resident(k, em)
    rs = [ctx.fit_k_resident(k, em) for _ in range(3)]
    out.append("%%s em %%.3f ms (%%d it, %%.1f us/it) total %%.3f" %% (
        name, np.mean([r.ms_em for r in rs]), rs[0].em_iterations,
        1e3 * np.mean([r.ms_em for r in rs]) / rs[0].em_iterations, np.mean([r.ms_total for r in rs])))
print(" | ".join(out), flush=True)
""" % ROOT
for lib in sys.argv[1:]:
    env = dict(os.environ)
    if lib != "cur":
        env["GMMB_LIB"] = lib
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), r.stdout.strip() or r.stderr[-500:], flush=True)
