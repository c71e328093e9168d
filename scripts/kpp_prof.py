"""Per-epoch phase breakdown of kpp_seed_kernel (build with -DGMMB_KPP_PROF).

  make -C paper_2307_00071_b200/csrc BUILD=build_prof OUT=build_prof/libgmmb.so EXTRA=-DGMMB_KPP_PROF
  GMMB_LIB=paper_2307_00071_b200/csrc/build_prof/libgmmb.so python scripts/kpp_prof.py
"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00071_b200 as gm

E, S, B = 320, 12, 160
ctx = gm.Context(0)
p = gm.synthetic_frame_cloud()
import time
for _ in range(3):
    t0 = time.perf_counter()
    gm.kinit(p, 512, 0, ctx=ctx)
    print(f"kinit wall {1e3 * (time.perf_counter() - t0):.2f} ms")
lib = gm.load()
buf = np.zeros(B * E * S, dtype=np.int64)
lib.gmmb_debug_kpp_prof(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(buf.size))
a = buf.reshape(B, E, S).astype(np.float64)
nb = 148
a = a[:nb]
ep = np.arange(5, 250)  # steady state
d = lambda i, j: (a[:, ep, j] - a[:, ep, i])
names = [("compute (fold+clocks+warp reduce), warp 0", 0, 1), ("-> barrier 1 (comm sees it)", 1, 2),
         ("CTA reduce + publish", 2, 3), ("gather (wait for all CTAs)", 3, 4), ("decide (coords)", 4, 5),
         ("draws, warp 0 (from barrier 1)", 2, 6), ("barrier 2 (from decide)", 5, 7),
         ("commit", 7, 8), ("epoch (0 -> 8)", 0, 8)]
print(f"{'phase':45s} {'median':>8s} {'p90':>8s} {'max':>8s}  cycles (all CTAs, epochs 5-249)")
for nm, i, j in names:
    x = d(i, j)
    print(f"{nm:45s} {np.median(x):8.0f} {np.percentile(x, 90):8.0f} {x.max():8.0f}")
nxt = a[:, ep + 1, 0] - a[:, ep, 8]
print(f"{'loop back (8 -> next 0)':45s} {np.median(nxt):8.0f}")
g_pub = a[:, ep, 9]
g_got = a[:, ep, 10]
skew = g_pub.max(0) - g_pub.min(0)
lat = g_got - g_pub.max(0)[None, :]
print(f"publish skew across CTAs (ns): median {np.median(skew):.0f} p90 {np.percentile(skew, 90):.0f}")
print(f"gather done after last publish (ns): median {np.median(lat):.0f} p90 {np.percentile(lat, 90):.0f}")
last = np.argmax(g_pub, axis=0)
print("last-publishing CTA histogram (top 8):", np.bincount(last, minlength=nb).argsort()[::-1][:8],
      np.sort(np.bincount(last, minlength=nb))[::-1][:8])
np.save(os.path.join("gpurun_out", "kpp_prof.npy"), buf.reshape(B, E, S)[:nb])
