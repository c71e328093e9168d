"""Per-kernel CUDA-event times of the pruned E step in situ (timing mode,
plain launches): block_cand, estep_sparse, sparse_reduce per iteration.

usage: GMMB_SP_EVENTS=1 python scripts/sp_events.py [--k 512] [--cfg4]
"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2307_00071_b200 as gm

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=512)
ap.add_argument("--cfg4", action="store_true")
args = ap.parse_args()
lib = gm.load()
lib.gmmb_debug_sp_events.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_int]
ctx = gm.Context(0)
ctx.set_timing(True)
if args.cfg4:
    p = gm.structured_scene(4_000_000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
else:
    p = gm.synthetic_frame_cloud()
ctx.upload(p)
buf = (ctypes.c_float * (3 * 256))()
for rep in range(3):
    lib.gmmb_debug_sp_events(buf, 256)
    r = ctx.fit_k_resident(args.k, gm.EmParams(100, 1e-3, 1e-6, 0))
    n = lib.gmmb_debug_sp_events(buf, 256)
    a = np.array(buf[:3 * n]).reshape(n, 3) * 1e3
    print("rep %d iters %d: us per E step (mean over %d): block_cand %.1f main %.1f reduce %.1f; "
          "ms_em %.3f ms_estep %.3f" % (rep, r.em_iterations, n, *a.mean(0), r.ms_em, r.ms_estep),
          flush=True)
    if rep == 2:
        for i, row in enumerate(a):
            print("  call %2d: %.1f %.1f %.1f" % (i, *row))
