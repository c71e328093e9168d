import time, sys, os
sys.path.insert(0, '.')
import paper_2307_00071_b200 as gm
ctx = gm.Context(0); p = gm.synthetic_frame_cloud()
for _ in range(4):
    t0 = time.perf_counter(); gm.kinit(p, 512, 0, ctx=ctx); print(f"plain kinit wall {1e3*(time.perf_counter()-t0):.2f} ms")
