"""Phase timestamps (clock64, thread 0) of the last commit kernel of a cfg2 fit
(build with -DGMMB_COMMIT_PROF)."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00071_b200 as gm
ctx = gm.Context(0)
p = gm.synthetic_frame_cloud()
ctx.upload(p)
for _ in range(2):
    ctx.fit_k_resident(512, gm.EmParams(100, 1e-3, 1e-6, 0))
lib = gm.load()
buf = np.zeros(64 * 8, dtype=np.int64)
lib.gmmb_debug_commit_prof(buf.ctypes.data_as(ctypes.c_void_p))
a = buf.reshape(64, 8)
names = ["state read", "ll + bookkeeping", "keep scans", "SPD check", "compaction copy", "end"]
rows = [r for r in a if r[0] != 0 and r[3] > r[0] and r[6] > r[5] > r[3]]
d = np.array([[r[i + 1] - r[i] for i in range(6)] for r in rows])
print(f"{len(rows)} full commits")
for n, v in zip(names, np.median(d, axis=0)):
    print(f"{n:20s} {v:8.0f} cycles")
