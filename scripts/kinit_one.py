import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00071_b200 as gm
n = int(sys.argv[1]) if len(sys.argv) > 1 else 307200
ctx = gm.Context(0)
p = gm.synthetic_frame_cloud()[:n]
ctx.upload(p)
r = ctx.fit_k_resident(512, gm.EmParams(1, 1e-3, 1e-6, 0))
print(f"n={n} kinit {r.ms_kinit:.3f} ms")
