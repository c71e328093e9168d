import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2307_00071_b200 as gm
ctx = gm.Context(0)
p = gm.synthetic_frame_cloud()
for n in [2000, 20000, 100000, 307200]:
    q = p[:n]
    ctx.upload(q)
    for rep in range(2):
        r = ctx.fit_k_resident(512, gm.EmParams(1, 1e-3, 1e-6, 0))
    print(f"n={n} kinit {r.ms_kinit:.3f} ms  per round {r.ms_kinit/512*1000:.2f} us", flush=True)
