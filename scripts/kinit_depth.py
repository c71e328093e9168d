"""kinit device time (timing mode) for several cloud sizes / K (depth A/B)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00071_b200 as gm
ctx = gm.Context(0)
ctx.set_timing(True)
frame = gm.synthetic_frame_cloud()
for n, k in [(20000, 512), (100000, 512), (307200, 512), (307200, 2048)]:
    ctx.upload(frame[:n])
    ts = []
    for _ in range(3):
        r = ctx.fit_k_resident(k, gm.EmParams(1, 1e-3, 1e-6, 0))
        ts.append(r.ms_kinit)
    print(f"n={n} k={k} kinit {min(ts):.3f} ms", flush=True)
