"""One kinit (k-means++ seeding) on a prefix of the cfg2 frame (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00071_b200 as gm
n = int(sys.argv[1]) if len(sys.argv) > 1 else 307200
k = int(sys.argv[2]) if len(sys.argv) > 2 else 512
ctx = gm.Context(0)
p = gm.synthetic_frame_cloud()[:n]
lab, cen = gm.kinit(p, k, 0, ctx=ctx)
print("kinit ok", n, k, cen[:4])
