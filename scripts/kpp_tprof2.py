"""Exchange timeline (two-round kernel: one row per exchange, i.e. per epoch) of the warp-specialised tile k-means++ (build with
-DGMMB_KPP_TPROF, run with GMMB_LIB pointing at it): per exchange the
publish skew across CTAs, the exchange completion, the kept-draw end."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2307_00071_b200 as gm
s = gm.structured_scene(4_000_000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
ctx = gm.Context(0)
gm.kinit(s, 2048, 0, ctx=ctx)
buf = (ctypes.c_ulonglong * (6 * 4096 * 160))()
gm.load().gmmb_debug_kpp_tprof(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(6, 4096, 160).astype(np.int64)[:, :, :148]
NX = int((a[0, :, 0] > 0).sum())  # exchanges recorded
print("exchanges", NX)
pub, seen, draw = a[0, :NX], a[1, :NX], a[2, :NX]
rng = slice(10, NX - 10)
p, q, d = pub[rng], seen[rng], draw[rng]
per_round = np.diff(q.min(1))
print(f"round period: mean {per_round.mean()/1e3:.2f} us, p50 {np.median(per_round)/1e3:.2f}")
print(f"publish skew (max - min over CTAs): mean {(p.max(1) - p.min(1)).mean()/1e3:.2f} us")
print(f"exchange (last publish -> all seen, per CTA mean): {(q - p.max(1)[:, None]).mean()/1e3:.2f} us")
print(f"own publish -> all seen: {(q - p).mean()/1e3:.2f} us")
# which CTA publishes last most often
last = p.argmax(1)
u, c = np.unique(last, return_counts=True)
print("most frequent last CTA:", list(zip(u[np.argsort(-c)][:5], np.sort(c)[::-1][:5])))
# draw end relative to seen (negative: draw finished before the exchange)
dr = d[:-1] - q[:-1]   # kept draw of round r+1 happens during exchange r
print(f"draw end - exchange end: mean {dr.mean()/1e3:.2f} us, p90 {np.percentile(dr, 90)/1e3:.2f}")
# time from exchange end (round r) to own publish of round r+1
nxt = p[1:] - q[:-1]
print(f"exchange end -> next publish: mean {nxt.mean()/1e3:.2f} us (fold + eval + publish)")

start, foldend, nfold = a[3, :NX][rng], a[4, :NX][rng], a[5, :NX][rng]
print(f"round start skew (max-min): {(start.max(1) - start.min(1)).mean()/1e3:.2f} us")
print(f"fold time: mean {(foldend - start).mean()/1e3:.2f} us, max-per-round mean {(foldend - start).max(1).mean()/1e3:.2f} us")
print(f"folded tiles per CTA: mean {nfold.mean():.2f}, max per round mean {nfold.max(1).mean():.1f}, total per round {nfold.sum(1).mean():.1f}")
print(f"fold end -> publish: mean {(p - foldend).mean()/1e3:.2f} us, max {(p - foldend).max(1).mean()/1e3:.2f}")
lastc = p.argmax(1)
print(f"last publisher's nfold mean {nfold[np.arange(len(lastc)), lastc].mean():.2f}; its fold time {(foldend - start)[np.arange(len(lastc)), lastc].mean()/1e3:.2f} us; its start lag {(start[np.arange(len(lastc)), lastc] - start.min(1)).mean()/1e3:.2f} us")
# kept-draw duration: from the CTA's publish of round r to its draw end (round r+1 kept)
dd = d[:-1] - p[:-1]
print(f"kept draw (publish -> draw end): mean {dd.mean()/1e3:.2f} us, max-per-round mean {dd.max(1).mean()/1e3:.2f} us")
