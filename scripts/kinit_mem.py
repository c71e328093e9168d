"""Memory-resident kinit (N beyond the shared-memory kernel): per-round time vs N."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00071_b200 as gm
ctx = gm.Context(0)
ctx.set_timing(True)
big = gm.structured_scene(4000000, 4, 0.005)[:, :3] * 25.0
for n in (400000, 1000000, 2000000, 4000000):
    ctx.upload(big[:n])
    ts = [ctx.fit_k_resident(256, gm.EmParams(1, 1e-3, 1e-6, 0)).ms_kinit for _ in range(2)]
    print(f"n={n} k=256 kinit {min(ts):.3f} ms = {1e3 * min(ts) / 256:.1f} us/round", flush=True)
