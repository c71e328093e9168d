"""Golden fixtures (tests/golden/, made by scripts/make_golden.py from the
FP64 oracle on the BASELINE configurations).

CPU: the oracle reproduces the committed goldens (regression pin of the
restatement: centres, label hashes and iteration counts exact, ll traces and
parameters to 1e-12). GPU: the CUDA path through the C ABI against the same
goldens with the BASELINE bars — no oracle run needed on the GPU box.
"""
import hashlib
import os

import numpy as np
import pytest

from parity import LL_TOL, assert_model_close, ll_err

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIT_CASES = ["cfg5_frame_k64", "cfg5_frame_k128", "cfg3_f3_k256", "cfg2_frame_k512"]


def gold(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz"), allow_pickle=False))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


def case_points(gm, name):
    f = gm.synthetic_frame_cloud()
    return gm.jitter_cloud(f, 0.002, 3) if name.startswith("cfg3") else f


def close12(a, b):
    return np.allclose(a, b, rtol=1e-12, atol=0)


# ---- CPU: the oracle is pinned to the goldens -------------------------------
@pytest.mark.parametrize("name", ["cfg5_frame_k64", "cfg3_f3_k256"])
def test_oracle_matches_golden_fit(gm, orc, name):
    g = gold(name)
    r = orc.fit_k(case_points(gm, name), int(g["k"]), 100, float(g["tol"]), 1e-6, int(g["seed"]))
    assert np.array_equal(r["centers"], g["centers"])
    assert sha(r["labels"]) == str(g["labels_sha256"])
    assert r["em_iterations"] == int(g["em_iterations"])
    assert close12(r["ll_trace"], g["ll_trace"])
    assert close12(r["w"], g["w"]) and close12(r["mu"], g["mu"]) and close12(r["cov"], g["cov"])


def test_oracle_matches_golden_cfg1(gm, orc):
    g = gold("cfg1_3d_fixed50")
    s1 = gm.structured_scene(20000, 1, 0.005)[:, :3]
    lab, cen = orc.kinit(s1, 32, 0)
    assert np.array_equal(cen, g["centers"]) and sha(lab) == str(g["labels_sha256"])
    w, mu, cov, _ = orc.m_step_labels(s1, lab, 32, 1e-6)
    assert close12(w, g["w0"]) and close12(mu[:, :3], g["mu0"]) and close12(cov[:, :6], g["cov0"])
    r = orc.fit_from(s1, g["w0"], g["mu0"], g["cov0"], 50, 0.0, 1e-6)
    assert r["em_iterations"] == 50 and close12(r["ll_trace"], g["ll_trace"])


def test_golden_files_consistent():
    for name in FIT_CASES:
        g = gold(name)
        k = int(g["k"])
        assert len(g["centers"]) == k and int(g["label_counts"].sum()) > 0
        assert np.all(g["label_counts"] >= 1)          # fix-up leaves no empty cluster
        assert len(g["ll_trace"]) == int(g["em_iterations"])
        assert np.all(np.diff(g["ll_trace"]) > 0)      # EM monotone on these fits
        assert abs(g["w"].sum() - 1.0) < 1e-12


# ---- GPU: the CUDA path against the goldens ---------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("name", FIT_CASES)
def test_gpu_fit_matches_golden(gm, ctx, name):
    g = gold(name)
    r = gm.fit_k(case_points(gm, name), int(g["k"]),
                 gm.EmParams(100, float(g["tol"]), 1e-6, int(g["seed"])), ctx=ctx, want_labels=True)
    assert np.array_equal(r.centers, g["centers"])
    assert sha(r.labels) == str(g["labels_sha256"])
    assert r.em_iterations == int(g["em_iterations"])
    assert ll_err(r.ll_trace, g["ll_trace"]) <= LL_TOL
    assert_model_close(r.model.weights, r.model.means, r.model.covariances, g["w"], g["mu"], g["cov"])


@pytest.mark.gpu
def test_gpu_cfg1_matches_golden(gm, ctx):
    g = gold("cfg1_3d_fixed50")
    s1 = gm.structured_scene(20000, 1, 0.005)[:, :3]
    lab, cen = gm.kinit(s1, 32, 0, ctx=ctx)
    assert np.array_equal(cen, g["centers"]) and sha(lab) == str(g["labels_sha256"])
    r = gm.fit_from(s1, gm.Gmm(g["w0"], g["mu0"], g["cov0"]), gm.EmParams(50, 0.0, 1e-6), ctx=ctx)
    assert r.em_iterations == 50
    assert ll_err(r.ll_trace, g["ll_trace"]) <= LL_TOL
    assert_model_close(r.model.weights, r.model.means, r.model.covariances, g["w"], g["mu"], g["cov"])
