"""k-means++ time per fit (ms_kinit) of library builds on the cfg2 frame
(K = 512, 2048) and a 20k-point cloud (K = 32); each build in a child
process (GMMB_LIB). usage: python scripts/kinit_lib_ab.py cur lib2.so ..."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2307_00071_b200 as gm
ctx = gm.Context(0)
out = []
for name, pts, k in (("frame K=512", gm.synthetic_frame_cloud(), 512),
                     ("frame K=2048", gm.synthetic_frame_cloud(), 2048),
                     ("20k K=32", gm.structured_scene(20000, 1, 0.005), 32),
                     ("dups K=8", np.repeat(np.array([[0, 0, 0, .1], [1, 0, 0, .2], [0, 1, 0, .3], [0, 0, 1, .4], [1, 1, 1, .5]]), 40, axis=0), 8),
                     ("300k K=64", gm.structured_scene(300000, 2, 0.005), 64)):
    ctx.upload(pts)
    ms = [ctx.fit_k_resident(k, gm.EmParams(1, 0.0, 1e-6, 0)).ms_kinit for _ in range(6)][1:]
    lab, cen = gm.kinit(pts, k, 0, ctx=ctx)
    lh = int(np.sum(lab.astype(np.int64) * (np.arange(len(lab)) %% 1000003)))
    out.append("%%s %%.3f ms (cen %%d lab %%d)" %% (name, float(np.median(ms)), int(np.sum(cen * 7 %% 1000003)), lh))
print(" | ".join(out))
""" % ROOT
for lib in sys.argv[1:]:
    env = dict(os.environ)
    if lib.startswith("env:"):  # env:NAME=VALUE (the current build)
        kv = lib[4:].split("=", 1)
        env[kv[0]] = kv[1]
    elif lib != "cur":
        env["GMMB_LIB"] = lib
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), r.stdout.strip() or r.stderr[-500:], flush=True)
