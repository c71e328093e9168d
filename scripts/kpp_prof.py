"""Per-epoch phase breakdown of kpp_seed_kernel (build with -DGMMB_KPP_PROF).

  make -C paper_2307_00071_b200/csrc BUILD=build_prof OUT=build_prof/libgmmb.so EXTRA=-DGMMB_KPP_PROF
  GMMB_LIB=paper_2307_00071_b200/csrc/build_prof/libgmmb.so python scripts/kpp_prof.py
"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00071_b200 as gm

E, S, B = 300, 9, 160
ctx = gm.Context(0)
p = gm.synthetic_frame_cloud()[: int(os.environ.get("KPP_N", "307200"))]
import time
for _ in range(3):
    t0 = time.perf_counter()
    gm.kinit(p, 512, 0, ctx=ctx)
    print(f"kinit wall {1e3 * (time.perf_counter() - t0):.2f} ms")
lib = gm.load()
buf = np.zeros(B * E * S, dtype=np.int64)
lib.gmmb_debug_kpp_prof(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(buf.size))
nb = 148
a = buf.reshape(B, E, S)[:nb].astype(np.float64)
np.save(os.path.join("gpurun_out", "kpp_prof.npy"), a)
ep = np.arange(5, 240)  # steady state
f = 1.0  # cycles
def iv(i, j, de=0):
    return a[:, ep + de, j] - a[:, ep, i]
rows = [("tid 0: fold loop (pre_ok epochs)", 0, 1, 0), ("tid 0: vote + recompute/copy + warp top-2s", 1, 2, 0),
        ("tid 0: barrier 1 + precompute", 2, 3, 0), ("tid 0: barrier 2 + commit", 3, 4, 0),
        ("tid 0: epoch", 0, 0, 1),
        ("comm: gather (after own publish)", 5, 6, 0), ("comm: decide", 6, 7, 0),
        ("comm: decide -> next publish", 7, 5, 1)]
nep = int((a[0, :, 0] != 0).sum())
print(f"epochs used (CTA 0): {nep}")
print(f"{'interval (cycles, same warp)':48s} {'median':>8s} {'p10':>8s} {'p90':>8s}")
for nm, i, j, de in rows:
    x = iv(i, j, de)
    x = x[(x > 0) & (x < 1e6)]
    print(f"{nm:48s} {np.median(x):8.0f} {np.percentile(x, 10):8.0f} {np.percentile(x, 90):8.0f}")
