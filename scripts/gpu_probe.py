"""Scratch GPU probe: parity + timing of the first CUDA path (not a test)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_2307_00071_b200 as gm


def relerr_model(g, r, d):
    w_err = np.max(np.abs(g.weights - r["w"]) / r["w"])
    sig = np.sqrt(np.stack([gm.unpack_symmetric(c, d).diagonal() for c in r["cov"]]))
    mu_err = np.max(np.abs(g.means - r["mu"]) / np.maximum(np.abs(r["mu"]), sig))
    ce = 0.0
    for a, b in zip(g.covariances, r["cov"]):
        A, B = gm.unpack_symmetric(a, d), gm.unpack_symmetric(b, d)
        s = np.sqrt(np.outer(B.diagonal(), B.diagonal()))
        ce = max(ce, np.max(np.abs(A - B) / s))
    return w_err, mu_err, ce


ctx = gm.Context(0)
print("device", ctx.device_info(), flush=True)
import __graft_entry__
__graft_entry__.smoke()

# cfg1: fixed init, 50 iterations
s = gm.structured_scene(20000, 1, 0.005)[:, :3]
lab, cen = oracle.kinit(s, 32, 0)
w, mu, cov, rm = oracle.m_step_labels(s, lab, 32, 1e-6)
init = gm.Gmm(w, mu[:, :3].copy(), cov[:, :6].copy())
t = time.time(); ref = oracle.fit_from(s, init.weights, init.means, init.covariances, 50, 0.0, 1e-6); tc = time.time() - t
res = gm.fit_from(s, init, gm.EmParams(50, 0.0, 1e-6), ctx=ctx)
llrel = np.max(np.abs(res.ll_trace - ref["ll_trace"]) / np.abs(ref["ll_trace"]))
print(f"cfg1: iters {res.em_iterations}/{ref['em_iterations']} ll rel max {llrel:.2e} "
      f"model err (w, mu, cov) {relerr_model(res.model, ref, 3)} cpu {tc:.2f}s gpu_em {res.ms_em:.2f}ms", flush=True)

# teacher-forced one step on cfg2 with a k-means init
p = gm.synthetic_frame_cloud()
t = time.time(); lab2, cen2 = oracle.kinit(p, 512, 0); tk = time.time() - t
glab, gcen = gm.kinit(p, 512, 0, ctx=ctx)
print(f"cfg2 kinit: centers equal {np.array_equal(gcen, cen2)} (first diff "
      f"{np.argmax(gcen != cen2) if not np.array_equal(gcen, cen2) else -1}), labels equal "
      f"{np.array_equal(glab, lab2)} mismatches {(glab != lab2).sum()} cpu {tk:.2f}s", flush=True)
w, mu, cov, rm = oracle.m_step_labels(p, lab2, 512, 1e-6)
m0 = gm.Gmm(w, mu, cov)
lg, llo = oracle.e_step(p, w, mu, cov)
w1, mu1, cov1, rm1 = oracle.m_step(p, lg, 1e-6)
ll_g, m1, rmg = gm.em_step(p, m0, 1e-6, ctx=ctx)
print(f"cfg2 teacher-forced step: ll rel {abs(ll_g - llo) / abs(llo):.2e} removed {rmg}/{rm1} "
      f"err {relerr_model(m1, dict(w=w1, mu=mu1, cov=cov1), 4)}", flush=True)

# full cfg2 fit on GPU, timing
em = gm.EmParams(100, 1e-3, 1e-6, 0)
ctx.upload(p)
for i in range(3):
    r = ctx.fit_k_resident(512, em)
    print(f"cfg2 gpu fit: iters {r.em_iterations} ll {r.final_log_likelihood:.6f} K {r.model.components()} "
          f"layout {r.ms_layout:.3f} kinit {r.ms_kinit:.3f} m0 {r.ms_mstep0:.3f} em {r.ms_em:.3f} ms "
          f"units {r.units:.3e} -> {r.units / (r.ms_em * 1e-3):.3e} u/s (EM)", flush=True)
t = time.time(); ref2 = oracle.fit_k(p, 512, 100, 1e-3, 1e-6, 0); tc2 = time.time() - t
llrel = np.max(np.abs(r.ll_trace - ref2["ll_trace"][:len(r.ll_trace)]) / np.abs(ref2["ll_trace"][:len(r.ll_trace)])) if len(r.ll_trace) == len(ref2["ll_trace"]) else -1
print(f"cfg2 oracle: iters {ref2['em_iterations']} ll {ref2['final_ll']:.6f} cpu {tc2:.1f}s; "
      f"ll rel {llrel:.2e} err {relerr_model(r.model, ref2, 4) if r.model.components() == len(ref2['w']) else 'K differs'}", flush=True)
