"""k-means++ on the cfg2 frame: the shared-memory-resident kernel vs the
tile-pruned one (GMMB_KINIT=tile, child process): ms and identical output."""
import os, subprocess, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2307_00071_b200 as gm
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    ctx = gm.Context(0)
    p = gm.synthetic_frame_cloud()
    ctx.upload(p)
    r = [ctx.fit_k_resident(int(sys.argv[3]), gm.EmParams(1, 0.0, 1e-6, 0), want_labels=True)
         for _ in range(4)][-1]
    np.savez(sys.argv[2], lab=r.labels, cen=r.centers, ms=r.ms_kinit)
    sys.exit(0)
for k in (64, 512, 2048):
    out = {}
    for mode in ("resident", "tile"):
        env = dict(os.environ)
        if mode == "tile":
            env["GMMB_KINIT"] = "tile"
        f = f"/tmp/kab_{mode}.npz"
        subprocess.run([sys.executable, __file__, "--child", f, str(k)], env=env, check=True)
        out[mode] = np.load(f)
    a, b = out["resident"], out["tile"]
    print(json.dumps({"k": k, "resident_ms": float(a["ms"]), "tile_ms": float(b["ms"]),
                      "centres_equal": bool(np.array_equal(a["cen"], b["cen"])),
                      "labels_equal": bool(np.array_equal(a["lab"], b["lab"]))}), flush=True)
