"""cfg4-size k-means++ with the tile kernel variants (GMMB_KPP_TILE = ws1 /
default two-round / sync): time per kinit and identical centres + labels.
usage: python scripts/kinit_variant_ab.py [n] [k]"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
CODE = r"""
import json, sys, time, numpy as np
sys.path.insert(0, %r)
import paper_2307_00071_b200 as gm
s = gm.structured_scene(%d, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
ctx = gm.Context(0)
ctx.upload(s)
ts = []
for _ in range(4):
    r = ctx.fit_k_resident(%d, gm.EmParams(1, 0.0, 1e-6, 0))
    ts.append(r.ms_kinit)
ts = ts[1:]
lab, cen = gm.kinit(s, %d, 0, ctx=ctx)
h = int(np.sum(lab.astype(np.int64) * (np.arange(len(lab)) %% 1000003)) %% 2147483647)
print(json.dumps({"ms": ts, "cen": cen.tolist(), "lab": h}))
""" % (ROOT, n, k, k)
res = {}
for v in [x for x in os.environ.get("VARIANTS", "ws1,,sync").split(",")]:
    env = dict(os.environ)
    if v:
        env["GMMB_KPP_TILE"] = v
    else:
        env.pop("GMMB_KPP_TILE", None)
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    if out.returncode != 0:
        print(v or "ws2", "FAILED", out.stderr[-1500:])
        continue
    d = json.loads(out.stdout.strip().splitlines()[-1])
    res[v or "ws2"] = d
    print(v or "ws2", "kinit ms", ["%.2f" % x for x in d["ms"]], flush=True)
names = list(res)
for a in names[1:]:
    print(a, "vs", names[0], "centres equal:", res[a]["cen"] == res[names[0]]["cen"],
          "labels equal:", res[a]["lab"] == res[names[0]]["lab"])
