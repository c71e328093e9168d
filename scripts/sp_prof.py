"""Per-tile timeline of the pruned E kernel (build with -DGMMB_SP_PROF, run
with GMMB_LIB pointing at it): span, per-SM busy fraction, tail, cost vs
candidate count, for the last E launch of a cfg2 fit."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2307_00071_b200 as gm
k = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ctx = gm.Context(0)
p = gm.synthetic_frame_cloud()
ctx.upload(p)
r = ctx.fit_k_resident(k, gm.EmParams(3, 0.0, 1e-6, 0))
nt = 4 * ((len(p) + 127) // 128)  # 32-point work items
buf = (ctypes.c_ulonglong * (4 * nt))()
gm.load().gmmb_debug_sp_prof(buf, 4 * nt)
a = np.frombuffer(buf, dtype=np.uint64).reshape(nt, 4).astype(np.int64)
t0, t1 = a[:, 0], a[:, 1]
sm = (a[:, 2] >> 32) & 0xffff
C = a[:, 2] & 0xffffffff
fused = a[:, 3] & 1
xs = (a[:, 3] >> 1) & 1
base = t0.min()
span = t1.max() - base
dur = t1 - t0
print(f"K={k} tiles {nt} span {span/1e3:.1f} us; tile us: mean {dur.mean()/1e3:.2f} p50 {np.median(dur)/1e3:.2f} "
      f"p99 {np.percentile(dur,99)/1e3:.2f} max {dur.max()/1e3:.2f}; fused {fused.mean():.2f} exact-fallback {xs.sum()}")
print("C: mean %.1f p50 %d p90 %d p99 %d max %d" % (C.mean(), np.median(C), np.percentile(C, 90), np.percentile(C, 99), C.max()))
for lo, hi in [(0, 16), (16, 32), (32, 64), (64, 128), (128, 100000)]:
    m = (C > lo) & (C <= hi)
    if m.any():
        print(f"  C in ({lo},{hi}]: {m.sum()} tiles, mean {dur[m].mean()/1e3:.2f} us, sum {dur[m].sum()/1e6:.3f} ms-warp")
ends = np.array([t1[sm == s].max() - base for s in np.unique(sm)])
starts = np.array([t0[sm == s].min() - base for s in np.unique(sm)])
print(f"per-SM first start {starts.max()/1e3:.1f} us max; last end min {ends.min()/1e3:.1f} p50 {np.median(ends)/1e3:.1f} max {ends.max()/1e3:.1f} us")
# warp-time accounting: sum of tile durations / (span * warps)
print(f"busy warp-time fraction {dur.sum() / (span * 148 * 16):.2f} (16 warps/SM)")

ph = (ctypes.c_uint * (6 * nt))()
gm.load().gmmb_debug_sp_ph(ph, 6 * nt)
b = np.frombuffer(ph, dtype=np.uint32).reshape(nt, 6).astype(np.float64)[:, :5]
names = ["load+box", "candidates", "passes", "slots+mask", "pass2/out"]
tot = b.sum(1)
print("phase cycles per unit (mean): " + ", ".join(f"{n} {b[:, i].mean():.0f}" for i, n in enumerate(names)) + f"; total {tot.mean():.0f}")
for lo, hi in [(0, 32), (32, 64), (64, 100000)]:
    m = (C > lo) & (C <= hi)
    if m.any():
        print(f"  C in ({lo},{hi}]: " + ", ".join(f"{n} {b[m, i].mean():.0f}" for i, n in enumerate(names)))
order = np.argsort(-dur)[:8]
print("longest units (us, C, start us, end us): " + "; ".join(
    f"{dur[i]/1e3:.1f} C={C[i]} @{(t0[i]-base)/1e3:.1f}-{(t1[i]-base)/1e3:.1f}" for i in order))
