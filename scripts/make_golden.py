"""Generate the golden fixtures in tests/golden/ from the FP64 oracle.

The reference (gmmscape) cannot be built here (no Eigen / libpng / vendored
CLI11 + json) and ships no golden vectors, so the goldens are
the oracle restatement's outputs on the BASELINE configurations: they pin
the oracle against regressions (tests/test_golden.py, CPU) and give the GPU
parity tests fixed expected values that need no CPU oracle run on the box.

Contents (npz, FP64 values stored exactly):
  cfg1_3d_fixed50.npz : N=20,000 structured scene (3D), kinit K=32 seed 0
                        centres + labels sha256, fixed init (w, mu, cov),
                        50 fixed iterations: ll trace, final model
  cfg2_frame_k512.npz : 640x480 frame, K=512 seed 0 tol 1e-3: centres,
                        labels sha256, em_iterations, ll trace, final model
  cfg5_frame_k64.npz / cfg5_frame_k128.npz : K sweep subset (same frame)
  cfg3_f3_k256.npz    : frame 3 of the cfg3 batch (2 mm jitter, seed 3), K=256

usage: python scripts/make_golden.py   (~1 min on 8 threads)
"""
import hashlib, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import oracle
import paper_2307_00071_b200 as gm

OUT = os.path.join(ROOT, "tests", "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


def fit_case(name, pts, k, seed, tol=1e-3, max_iters=100):
    r = oracle.fit_k(pts, k, max_iters, tol, 1e-6, seed)
    lab, cen = r["labels"], r["centers"]
    np.savez_compressed(os.path.join(OUT, name), centers=cen, labels_sha256=sha(lab),
                        label_counts=np.bincount(lab, minlength=k), k=k, seed=seed, tol=tol,
                        em_iterations=r["em_iterations"], ll_trace=np.asarray(r["ll_trace"]),
                        final_ll=r["final_ll"], w=r["w"], mu=r["mu"], cov=r["cov"],
                        removed=r.get("removed", 0))
    print(name, "iters", r["em_iterations"], "K_out", len(r["w"]))


def main():
    os.makedirs(OUT, exist_ok=True)
    s1 = gm.structured_scene(20000, 1, 0.005)[:, :3]
    lab, cen = oracle.kinit(s1, 32, 0)
    w, mu, cov, _ = oracle.m_step_labels(s1, lab, 32, 1e-6)
    w0, mu0, cov0 = w, mu[:, :3].copy(), cov[:, :6].copy()
    r = oracle.fit_from(s1, w0, mu0, cov0, 50, 0.0, 1e-6)
    np.savez_compressed(os.path.join(OUT, "cfg1_3d_fixed50.npz"), centers=cen,
                        labels_sha256=sha(lab), w0=w0, mu0=mu0, cov0=cov0,
                        em_iterations=r["em_iterations"], ll_trace=np.asarray(r["ll_trace"]),
                        final_ll=r["final_ll"], w=r["w"], mu=r["mu"], cov=r["cov"])
    print("cfg1 iters", r["em_iterations"])
    frame = gm.synthetic_frame_cloud()
    fit_case("cfg2_frame_k512.npz", frame, 512, 0)
    fit_case("cfg5_frame_k64.npz", frame, 64, 0)
    fit_case("cfg5_frame_k128.npz", frame, 128, 0)
    fit_case("cfg3_f3_k256.npz", gm.jitter_cloud(frame, 0.002, 3), 256, 3)


if __name__ == "__main__":
    main()
