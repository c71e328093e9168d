"""Precision experiment: GPU variants vs the oracle (teacher-forced + end-to-end)."""
import json, os, pickle, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
import paper_2307_00071_b200 as gm
from parity import model_err, ll_err

REF = "/tmp/prec_refs.pkl"
frame = gm.synthetic_frame_cloud()
f3 = gm.jitter_cloud(frame, 0.002, 3)
s1 = gm.structured_scene(20000, 1, 0.005)[:, :3]
if not os.path.exists(REF):
    refs = {}
    lab, _ = oracle.kinit(frame, 512, 0)
    w, mu, cov, _ = oracle.m_step_labels(frame, lab, 512, 1e-6)
    lg, ll = oracle.e_step(frame, w, mu, cov)
    refs["tf_in"] = (w, mu, cov)
    refs["tf_out"] = oracle.m_step(frame, lg, 1e-6)[:3] + (ll,)
    refs["cfg2"] = oracle.fit_k(frame, 512, 100, 1e-3, 1e-6, 0)
    refs["cfg3"] = oracle.fit_k(f3, 256, 100, 1e-3, 1e-6, 3)
    lab1, _ = oracle.kinit(s1, 32, 0)
    w1, mu1, cov1, _ = oracle.m_step_labels(s1, lab1, 32, 1e-6)
    refs["cfg1_in"] = (w1, mu1[:, :3].copy(), cov1[:, :6].copy())
    refs["cfg1"] = oracle.fit_from(s1, *refs["cfg1_in"], 50, 0.0, 1e-6)
    pickle.dump(refs, open(REF, "wb"))
refs = pickle.load(open(REF, "rb"))
ctx = gm.Context(0)
out = {"lib": os.environ.get("GMMB_LIB", "default")}
w, mu, cov = refs["tf_in"]
ll, m1, _ = gm.em_step(frame, gm.Gmm(w, mu, cov), 1e-6, ctx=ctx)
rw, rmu, rcov, rll = refs["tf_out"]
out["tf"] = model_err(m1.weights, m1.means, m1.covariances, rw, rmu, rcov) + (abs(ll - rll) / abs(rll),)
for name, pts, k, seed in [("cfg2", frame, 512, 0), ("cfg3", f3, 256, 3)]:
    r = gm.fit_k(pts, k, gm.EmParams(100, 1e-3, 1e-6, seed), ctx=ctx)
    ref = refs[name]
    e = model_err(r.model.weights, r.model.means, r.model.covariances, ref["w"], ref["mu"], ref["cov"]) \
        if len(r.model.weights) == len(ref["w"]) else ("K differs",)
    out[name] = e + (r.em_iterations, ref["em_iterations"], ll_err(r.ll_trace, ref["ll_trace"]) if r.em_iterations == ref["em_iterations"] else -1, r.ms_em)
r = gm.fit_from(s1, gm.Gmm(*refs["cfg1_in"]), gm.EmParams(50, 0.0, 1e-6), ctx=ctx)
ref = refs["cfg1"]
out["cfg1"] = model_err(r.model.weights, r.model.means, r.model.covariances, ref["w"], ref["mu"], ref["cov"]) + (ll_err(r.ll_trace, ref["ll_trace"]),)
print(json.dumps(out), flush=True)
