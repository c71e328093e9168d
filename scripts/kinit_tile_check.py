"""Tile-pruned k-means++ (kinit_tile.cu) against the memory-resident kernel
(GMMB_KINIT=mem, in a child process): centres and labels identical; ms."""
import os, subprocess, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2307_00071_b200 as gm

def cases():
    s = gm.structured_scene(4_000_000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
    yield "cfg4", s, 2048
    f = gm.synthetic_frame_cloud()
    big = np.vstack([f, gm.jitter_cloud(f, 0.002, 1)])  # 614k 4D points
    yield "2frames", big, 512
    dup = np.repeat(big[:200000], 2, axis=0)             # exact duplicates
    yield "dups", dup, 300

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    out = {}
    ctx = gm.Context(0)
    for name, p, k in cases():
        gm.kinit(p, k, 0, ctx=ctx)
        t = time.perf_counter()
        lab, cen = gm.kinit(p, k, 0, ctx=ctx)
        out[name] = (time.perf_counter() - t, lab, cen)
    np.savez(sys.argv[2], **{f"{n}_{w}": v for n, (tt, l, c) in out.items()
                             for w, v in (("t", tt), ("lab", l), ("cen", c))})
    sys.exit(0)

for mode in ("tile", "mem"):
    env = dict(os.environ)
    if mode == "mem":
        env["GMMB_KINIT"] = "mem"
    subprocess.run([sys.executable, __file__, "--child", f"/tmp/kinit_{mode}.npz"], env=env, check=True)
a, b = np.load("/tmp/kinit_tile.npz"), np.load("/tmp/kinit_mem.npz")
for name in ("cfg4", "2frames", "dups"):
    print(json.dumps({"case": name, "tile_s": float(a[f"{name}_t"]), "mem_s": float(b[f"{name}_t"]),
                      "centres_equal": bool(np.array_equal(a[f"{name}_cen"], b[f"{name}_cen"])),
                      "labels_equal": bool(np.array_equal(a[f"{name}_lab"], b[f"{name}_lab"]))}), flush=True)
