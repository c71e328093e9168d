"""CUDA path (through the C ABI) vs the FP64 oracle on identical inputs.

Bars (BASELINE.json north_star): kinit centres/labels, iteration counts and
K bit-exact; per-iteration ll within 1e-5 relative; weights / means /
covariances within 1e-4 (normalised metrics, tests/parity.py).
"""
import numpy as np
import pytest

from parity import LL_TOL, assert_model_close, ll_err

pytestmark = pytest.mark.gpu


def frame(gm):
    return gm.synthetic_frame_cloud()


def fixed_init(orc, pts, k, cov_reg=1e-6, seed=0):
    lab, cen = orc.kinit(pts, k, seed)
    w, mu, cov, _ = orc.m_step_labels(pts, lab, k, cov_reg)
    d = pts.shape[1]
    return w, mu[:, :d].copy(), cov[:, :d * (d + 1) // 2].copy()


# ---- kinit: bit-exact -------------------------------------------------------
@pytest.mark.parametrize("k,seed", [(1, 0), (7, 3), (64, 0), (512, 0), (512, 5)])
def test_kinit_frame_exact(gm, orc, ctx, k, seed):
    p = frame(gm)
    lab, cen = gm.kinit(p, k, seed, ctx=ctx)
    rl, rc = orc.kinit(p, k, seed)
    assert np.array_equal(cen, rc)
    assert np.array_equal(lab, rl)


def test_kinit_3d_scene_exact(gm, orc, ctx):
    p = gm.structured_scene(60000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
    lab, cen = gm.kinit(p, 256, 0, ctx=ctx)
    rl, rc = orc.kinit(p, 256, 0)
    assert np.array_equal(cen, rc) and np.array_equal(lab, rl)


def test_kinit_duplicates_fallback_and_fixup(gm, orc, ctx):
    base = np.array([[0, 0, 0, 0.1], [1, 0, 0, 0.2], [0, 1, 0, 0.3], [0, 0, 1, 0.4],
                     [1, 1, 1, 0.5]], float)
    p = np.repeat(base, 40, axis=0)
    lab, cen = gm.kinit(p, 8, 0, ctx=ctx)
    rl, rc = orc.kinit(p, 8, 0)
    assert np.array_equal(cen, rc) and np.array_equal(lab, rl)
    assert np.all(np.bincount(lab, minlength=8) >= 1)


def test_kinit_k_equals_n(gm, orc, ctx):
    rng = np.random.default_rng(4)
    p = np.column_stack([rng.normal(size=(300, 3)), rng.random(300)])
    lab, cen = gm.kinit(p, 300, 1, ctx=ctx)
    rl, rc = orc.kinit(p, 300, 1)
    assert np.array_equal(cen, rc) and np.array_equal(lab, rl)


def test_kinit_large_cloud_memory_variant(gm, orc, ctx):
    """N beyond the register-resident seeding kernel (148*384*8 = 454,656)."""
    p = gm.structured_scene(600000, 7, 0.005)
    lab, cen = gm.kinit(p, 32, 0, ctx=ctx)
    rl, rc = orc.kinit(p, 32, 0)
    assert np.array_equal(cen, rc) and np.array_equal(lab, rl)


# ---- one production EM step, teacher forced ----------------------------------
@pytest.mark.parametrize("k", [32, 256, 512, 1024, 2048])
def test_em_step_teacher_forced_frame(gm, orc, ctx, k):
    p = frame(gm)
    if k > 512:  # cluster path (K > 512); keep the oracle quick
        p = p[::2].copy()
    w, mu, cov = fixed_init(orc, p, k)
    ll, m1, rm = gm.em_step(p, gm.Gmm(w, mu, cov), 1e-6, ctx=ctx)
    lg, rll = orc.e_step(p, w, mu, cov)
    rw, rmu, rcov, rrm = orc.m_step(p, lg, 1e-6)
    assert abs(ll - rll) / abs(rll) < LL_TOL
    assert rm == rrm
    assert_model_close(m1.weights, m1.means, m1.covariances, rw, rmu, rcov, tol=1e-5)


def test_em_step_3d_offset_scene(gm, orc, ctx):
    """cfg4-like coordinates (x25, offset (100,-40,0) m) stress the FP32
    recentring; D = 3 native kernels."""
    p = gm.structured_scene(100000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
    w, mu, cov = fixed_init(orc, p, 128)
    ll, m1, rm = gm.em_step(p, gm.Gmm(w, mu, cov), 1e-6, ctx=ctx)
    r = orc.fit_from(p, w, mu, cov, max_iters=1, ll_rel_tol=0.0, cov_reg=1e-6)
    assert abs(ll - r["final_ll"]) / abs(r["final_ll"]) < LL_TOL
    assert_model_close(m1.weights, m1.means, m1.covariances, r["w"], r["mu"], r["cov"], tol=1e-5)


def test_em_step_removes_degenerate_component(gm, orc, ctx):
    rng = np.random.default_rng(12)
    p = np.column_stack([rng.normal(size=(20000, 3)) * 0.1, rng.random(20000)])
    w = np.array([0.5, 0.4999, 0.0001])
    mu = np.array([[0.05, 0, 0, 0.5], [-0.05, 0, 0, 0.5], [50.0, 50.0, 50.0, 0.5]])
    cov = np.array([[0.01, 0, 0.01, 0, 0, 0.01, 0, 0, 0, 0.1]] * 3)
    ll, m1, rm = gm.em_step(p, gm.Gmm(w, mu, cov), 1e-6, ctx=ctx)
    lg, rll = orc.e_step(p, w, mu, cov)
    rw, rmu, rcov, rrm = orc.m_step(p, lg, 1e-6)
    assert rm == rrm == 1
    assert_model_close(m1.weights, m1.means, m1.covariances, rw, rmu, rcov, tol=1e-5)


# ---- end-to-end fits -----------------------------------------------------------
def test_cfg1_fixed_init_50_iterations(gm, orc, ctx):
    """BASELINE cfg1: 3D, N=20,000, K=32, fixed init, 50 EM iterations."""
    p = gm.structured_scene(20000, 1, 0.005)[:, :3]
    w, mu, cov = fixed_init(orc, p, 32)
    res = gm.fit_from(p, gm.Gmm(w, mu, cov), gm.EmParams(50, 0.0, 1e-6), ctx=ctx)
    ref = orc.fit_from(p, w, mu, cov, max_iters=50, ll_rel_tol=0.0, cov_reg=1e-6)
    assert res.em_iterations == ref["em_iterations"] == 50
    assert ll_err(res.ll_trace, ref["ll_trace"]) < LL_TOL
    assert_model_close(res.model.weights, res.model.means, res.model.covariances,
                       ref["w"], ref["mu"], ref["cov"])


def test_cfg2_fit_k512_end_to_end(gm, orc, ctx):
    """BASELINE cfg2: one 640x480 frame, K=512, k-means++ + EM to tol 1e-3."""
    p = frame(gm)
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    res = gm.fit_k(p, 512, em, ctx=ctx, want_labels=True)
    ref = orc.fit_k(p, 512, max_iters=100, ll_rel_tol=1e-3, cov_reg=1e-6, seed=0)
    assert np.array_equal(res.centers, ref["centers"])
    assert np.array_equal(res.labels, ref["labels"])
    assert res.em_iterations == ref["em_iterations"]
    assert res.removed_components == ref["removed"]
    assert ll_err(res.ll_trace, ref["ll_trace"]) < LL_TOL
    assert_model_close(res.model.weights, res.model.means, res.model.covariances,
                       ref["w"], ref["mu"], ref["cov"])
    assert res.units == pytest.approx(len(p) * 512 * res.em_iterations)


def test_cfg3_jittered_frame_k256(gm, orc, ctx):
    """BASELINE cfg3 frame f: xyz jittered by 2 mm (seed f), K=256, seed f."""
    f = 3
    p = gm.jitter_cloud(frame(gm), 0.002, f)
    em = gm.EmParams(100, 1e-3, 1e-6, f)
    res = gm.fit_k(p, 256, em, ctx=ctx)
    ref = orc.fit_k(p, 256, max_iters=100, ll_rel_tol=1e-3, cov_reg=1e-6, seed=f)
    assert res.em_iterations == ref["em_iterations"]
    assert ll_err(res.ll_trace, ref["ll_trace"]) < LL_TOL
    assert_model_close(res.model.weights, res.model.means, res.model.covariances,
                       ref["w"], ref["mu"], ref["cov"])


def test_blobs_3d_fit_converged_model(gm, orc, ctx):
    c = np.array([[0.1, 0.1, 0.1, 0.0], [0.5, 0.5, 0.5, 0.0], [0.9, 0.9, 0.9, 0.0]])
    p = gm.blob_cloud(c, 0.02, 2000, 7)[:, :3]
    em = gm.EmParams(200, 1e-7, 1e-6, 0)
    res = gm.fit_k(p, 5, em, ctx=ctx)
    ref = orc.fit_k(p, 5, max_iters=200, ll_rel_tol=1e-7, cov_reg=1e-6, seed=0)
    assert res.em_iterations == ref["em_iterations"]
    assert ll_err(res.ll_trace, ref["ll_trace"]) < LL_TOL
    assert_model_close(res.model.weights, res.model.means, res.model.covariances,
                       ref["w"], ref["mu"], ref["cov"])


def test_deterministic_bits(gm, ctx):
    p = frame(gm)[::3].copy()
    em = gm.EmParams(10, 0.0, 1e-6, 0)
    a = gm.fit_k(p, 128, em, ctx=ctx)
    b = gm.fit_k(p, 128, em, ctx=ctx)
    assert np.array_equal(a.ll_trace, b.ll_trace)
    assert np.array_equal(a.model.means, b.model.means)
    assert np.array_equal(a.model.covariances, b.model.covariances)


def test_resident_matches_host_api(gm, ctx):
    p = frame(gm)[::4].copy()
    em = gm.EmParams(20, 1e-4, 1e-6, 0)
    a = gm.fit_k(p, 64, em, ctx=ctx)
    ctx.upload(p)
    b = ctx.fit_k_resident(64, em)
    assert np.array_equal(a.ll_trace, b.ll_trace)
    assert np.array_equal(a.model.weights, b.model.weights)


# ---- single-step APIs ------------------------------------------------------------
def test_e_step_api(gm, orc, ctx):
    p = frame(gm)[::50].copy()
    w, mu, cov = fixed_init(orc, p, 16)
    lg, ll = gm.e_step(p, gm.Gmm(w, mu, cov), ctx=ctx)
    rlg, rll = orc.e_step(p, w, mu, cov)
    assert abs(ll - rll) / abs(rll) < 1e-12
    big = rlg > -30
    assert np.max(np.abs(lg[big] - rlg[big])) < 1e-8


def test_m_step_api(gm, orc, ctx):
    rng = np.random.default_rng(5)
    p = frame(gm)[::40].copy()
    lg = rng.normal(size=(len(p), 12)) * 3
    lg -= np.log(np.exp(lg).sum(1, keepdims=True))
    m, rm = gm.m_step(p, lg, 1e-6, ctx=ctx)
    rw, rmu, rcov, rrm = orc.m_step(p, lg, 1e-6)
    assert rm == rrm
    assert_model_close(m.weights, m.means, m.covariances, rw, rmu, rcov, tol=1e-10)


def test_cholesky_cache_api(gm, orc, ctx):
    rng = np.random.default_rng(6)
    a = rng.normal(size=(50, 4, 4))
    s = np.einsum("mij,mkj->mik", a, a) + 1e-3 * np.eye(4)
    r, c = np.array([0, 1, 1, 2, 2, 2, 3, 3, 3, 3]), np.array([0, 0, 1, 0, 1, 2, 0, 1, 2, 3])
    cov = s[:, r, c]
    cc = gm.cholesky_cache(gm.Gmm(np.full(50, 0.02), np.zeros((50, 4)), cov), ctx=ctx)
    lo, pr, ld = orc.cholesky_cache(cov)
    assert np.max(np.abs(cc.lower - lo)) < 1e-12
    assert np.max(np.abs(cc.precision - pr)) < 1e-9
    assert np.max(np.abs(cc.log_det_terms - ld)) < 1e-12


# ---- error behaviour (gmmscape_cli.cpp:508-528 classes) --------------------------
def test_errors(gm, ctx):
    p = frame(gm)[::100].copy()
    bad = p.copy()
    bad[5, 2] = np.nan
    with pytest.raises(gm.NumericalError):
        gm.fit_k(bad, 4, gm.EmParams(5, 1e-3), ctx=ctx)
    bad = p.copy()
    bad[5, 3] = 1.5
    with pytest.raises(gm.NumericalError, match="intensity"):
        gm.fit_k(bad, 4, gm.EmParams(5, 1e-3), ctx=ctx)
    with pytest.raises(ValueError):
        gm.fit_k(p, 0, gm.EmParams(5, 1e-3), ctx=ctx)
    with pytest.raises(ValueError):
        gm.fit_k(p, 4, gm.EmParams(0, 1e-3), ctx=ctx)
    with pytest.raises(ValueError):
        gm.kinit(p, len(p) + 1, 0, ctx=ctx)
    w = np.array([0.5, 0.5])
    mu = np.zeros((2, 4))
    cov = np.array([[1, 0, 1, 0, 0, 1, 0, 0, 0, 1.0], [-1, 0, 1, 0, 0, 1, 0, 0, 0, 1.0]])
    with pytest.raises(gm.NumericalError, match="block 1"):
        gm.fit_from(p, gm.Gmm(w, mu, cov), gm.EmParams(5, 1e-3), ctx=ctx)
    # K > N is clamped to N (sogmm.cpp:477)
    r = gm.fit_k(p[:20], 50, gm.EmParams(3, 0.0, 1e-3), ctx=ctx)
    assert r.k_init == 20


def test_cpp_example_fits_blobs(gm, tmp_path):
    import subprocess
    from test_abi import build_cpp_example
    exe = build_cpp_example(gm, tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "K=3" in r.stdout


# ---- edge shapes of the fused kernels (partial tiles / sub-tiles, tiny N) ---
@pytest.mark.parametrize("n,k,d", [(7, 1, 4), (50, 3, 4), (129, 4, 4), (1000, 17, 3),
                                   (4097, 64, 4), (20011, 300, 4)])
def test_small_and_ragged_fits(gm, orc, ctx, n, k, d):
    # k separated blobs (EM well conditioned, so parameter errors measure the
    # kernels, not EM's amplification on unstructured data), N not a multiple
    # of the 128-point tile or the 16-point sub-tile
    rng = np.random.default_rng(n)
    centers = np.column_stack([rng.random((k, 3)) * 10.0, 0.2 + 0.6 * rng.random(k)])
    lab = rng.integers(0, k, n)
    base = centers[lab] + np.column_stack([0.05 * rng.normal(size=(n, 3)),
                                          0.01 * rng.normal(size=n)])
    base[:, 3] = np.clip(base[:, 3], 0.0, 1.0)
    base = base[:, :d].copy()
    em = gm.EmParams(40, 1e-6, 1e-6, 1)
    r = gm.fit_k(base, k, em, ctx=ctx, want_labels=True)
    ref = orc.fit_k(base, k, 40, 1e-6, 1e-6, 1)
    assert np.array_equal(r.centers, ref["centers"]) and np.array_equal(r.labels, ref["labels"])
    assert r.em_iterations == ref["em_iterations"] and r.removed_components == ref["removed"]
    assert ll_err(r.ll_trace, ref["ll_trace"]) <= LL_TOL
    assert_model_close(r.model.weights, r.model.means, r.model.covariances,
                       ref["w"], ref["mu"][:, :d], ref["cov"][:, :d * (d + 1) // 2])


@pytest.mark.gpu
@pytest.mark.parametrize("k,seed", [(512, 0), (97, 5)])
def test_kinit_depth3_exact(gm, orc, ctx, k, seed, monkeypatch):
    """The three-rounds-per-exchange seeding variant (not the default) is bit-exact too."""
    monkeypatch.setenv("GMMB_KPP_DEPTH", "3")
    p = frame(gm)
    lab, cen = gm.kinit(p, k, seed, ctx=ctx)
    rl, rc = orc.kinit(p, k, seed)
    assert np.array_equal(cen, rc)
    assert np.array_equal(lab, rl)


@pytest.mark.gpu
def test_kinit_memory_variant_3d_duplicates_fallback(gm, orc, ctx):
    """Memory-resident seeding (N > the shared-memory budget) on a 3D cloud of
    20 distinct points repeated: after 20 rounds every d2 is 0 and the rounds
    take the lowest unchosen index (sogmm.cpp:276-284)."""
    base = gm.structured_scene(20, 3, 0.005)[:, :3]
    p = np.repeat(base, 20000, axis=0)  # 400,000 points
    lab, cen = gm.kinit(p, 32, 0, ctx=ctx)
    rl, rc = orc.kinit(p, 32, 0)
    assert np.array_equal(cen, rc) and np.array_equal(lab, rl)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [64, 1024])
def test_em_step_far_outliers_exact_path(gm, orc, ctx, k):
    """Points far from every component: their unshifted density sums leave
    [2^-64, 2^64], so the fused E kernel redoes those sub-tiles with the
    exact max shift (both the single-CTA and the cluster kernel). (Offsets of
    metres, not kilometres: log-densities of 1e10 are beyond FP32's
    resolution of which component a point belongs to, a documented limit.)"""
    base = gm.structured_scene(30000, 9, 0.005)
    w, mu, cov = fixed_init(orc, base, k)
    far = base[:40].copy()
    far[:, :3] += 3.0
    p = np.vstack([base, far])
    ll, m1, rm = gm.em_step(p, gm.Gmm(w, mu, cov), 1e-6, ctx=ctx)
    lg, rll = orc.e_step(p, w, mu, cov)
    rw, rmu, rcov, rrm = orc.m_step(p, lg, 1e-6)
    assert rm == rrm
    assert abs(ll - rll) / abs(rll) < LL_TOL
    # 3e-5 (a single step; the fit-level bar is 1e-4): the 40 far points
    # dominate the scatter of the components that absorb them (|d| ~ 3 m
    # against ~5 cm), which magnifies FP32 rounding of their r d d^T terms
    # ~300x; the dense and the pruned kernels both sit at that floor
    # (scripts/outlier_err.py: 5e-6 and 1.1e-5 for K = 64, 6e-6 for both at
    # K = 1024; the pruned kernel with every pair kept gives the same 1.1e-5)
    assert_model_close(m1.weights, m1.means, m1.covariances, rw, rmu, rcov, tol=3e-5)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1024, 2048])
def test_em_step_3d_cluster_kernels(gm, orc, ctx, k):
    """D = 3 with K > 512 (the cfg4 path: clusters of K / 512 CTAs), on
    cfg4-like map coordinates."""
    p = gm.structured_scene(120000, 5, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
    w, mu, cov = fixed_init(orc, p, k)
    ll, m1, rm = gm.em_step(p, gm.Gmm(w, mu, cov), 1e-6, ctx=ctx)
    r = orc.fit_from(p, w, mu, cov, max_iters=1, ll_rel_tol=0.0, cov_reg=1e-6)
    assert abs(ll - r["final_ll"]) / abs(r["final_ll"]) < LL_TOL
    assert_model_close(m1.weights, m1.means, m1.covariances, r["w"], r["mu"], r["cov"], tol=1e-5)


@pytest.mark.gpu
@pytest.mark.parametrize("k,d", [(700, 4), (1500, 3)])
def test_em_step_ragged_k_cluster_padding(gm, orc, ctx, k, d):
    """K between the 512-component CTA sizes: the last CTA of each cluster
    holds padding components (zero weight, excluded from the statistics)."""
    p = gm.structured_scene(80000, 6, 0.005)[:, :d]
    w, mu, cov = fixed_init(orc, p, k)
    ll, m1, rm = gm.em_step(p, gm.Gmm(w, mu, cov), 1e-6, ctx=ctx)
    r = orc.fit_from(p, w, mu, cov, max_iters=1, ll_rel_tol=0.0, cov_reg=1e-6)
    assert abs(ll - r["final_ll"]) / abs(r["final_ll"]) < LL_TOL
    assert_model_close(m1.weights, m1.means, m1.covariances, r["w"], r["mu"], r["cov"], tol=1e-5)


@pytest.mark.gpu
def test_em_step_k4096_stats_kernel(gm, orc, ctx):
    """K = 4096 (kMaxK) goes through estep_stats_kernel (barrier per sub-tile,
    clusters) and a four-chunk commit."""
    p = gm.structured_scene(60000, 8, 0.005)
    w, mu, cov = fixed_init(orc, p, 4096)
    ll, m1, rm = gm.em_step(p, gm.Gmm(w, mu, cov), 1e-6, ctx=ctx)
    lg, rll = orc.e_step(p, w, mu, cov)
    rw, rmu, rcov, rrm = orc.m_step(p, lg, 1e-6)
    assert rm == rrm
    assert abs(ll - rll) / abs(rll) < LL_TOL
    assert_model_close(m1.weights, m1.means, m1.covariances, rw, rmu, rcov, tol=1e-5)


@pytest.mark.gpu
@pytest.mark.parametrize("k,stride", [(1024, 4), (2048, 2)])
def test_fit_large_k_end_to_end(gm, orc, ctx, k, stride):
    """cfg5's large-K end: k-means++ + EM to tol 1e-3 through the cluster
    kernels, on a subsampled cfg2 frame (the oracle's run time) with ~75
    points per component. (Below ~40 points per component EM amplifies FP32
    rounding past 1e-4 on any K: scripts/studies/large_k_precision.py.)"""
    p = frame(gm)[::stride].copy()
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    res = gm.fit_k(p, k, em, ctx=ctx, want_labels=True)
    ref = orc.fit_k(p, k, max_iters=100, ll_rel_tol=1e-3, cov_reg=1e-6, seed=0)
    assert np.array_equal(res.centers, ref["centers"])
    assert res.em_iterations == ref["em_iterations"]
    assert res.removed_components == ref["removed"]
    assert ll_err(res.ll_trace, ref["ll_trace"]) < LL_TOL
    assert_model_close(res.model.weights, res.model.means, res.model.covariances,
                       ref["w"], ref["mu"], ref["cov"])


@pytest.mark.gpu
@pytest.mark.parametrize("k", [4608, 5000])
def test_em_step_above_4096_chunked(gm, orc, ctx, k):
    """K > 4096 (the reference accepts any 1 <= k <= N, sogmm.cpp:200-202):
    the chunked two-pass E step (9-10 chunks of 512) and the run-time-chunked
    commit (compaction map in global memory)."""
    p = gm.structured_scene(60000, 8, 0.005)
    w, mu, cov = fixed_init(orc, p, k)
    ll, m1, rm = gm.em_step(p, gm.Gmm(w, mu, cov), 1e-6, ctx=ctx)
    lg, rll = orc.e_step(p, w, mu, cov)
    rw, rmu, rcov, rrm = orc.m_step(p, lg, 1e-6)
    assert rm == rrm
    assert abs(ll - rll) / abs(rll) < LL_TOL
    assert_model_close(m1.weights, m1.means, m1.covariances, rw, rmu, rcov, tol=1e-5)


@pytest.mark.gpu
def test_single_step_calls_invalidate_resident_cloud(gm, orc, ctx):
    """e_step / kinit / ... stage their own input: a later *_resident fit
    must not silently fit that input (or the old cloud with another D)."""
    p = frame(gm)[::8].copy()
    ctx.upload(p)
    ctx.fit_k_resident(16, gm.EmParams(3, 0.0, 1e-6, 0))
    w, mu, cov = fixed_init(orc, p[:, :3].copy(), 4)
    gm.e_step(p[:, :3].copy(), gm.Gmm(w, mu, cov), ctx=ctx)
    with pytest.raises(ValueError, match="no point cloud"):
        ctx.fit_k_resident(16, gm.EmParams(3, 0.0, 1e-6, 0))
    ctx.upload(p)
    assert ctx.fit_k_resident(16, gm.EmParams(3, 0.0, 1e-6, 0)).em_iterations == 3


@pytest.mark.gpu
def test_cfg3_frame_batch_matches_single_fits_and_oracle(gm, orc, ctx):
    """BASELINE cfg3 batch: frames f (2 mm jitter, seed f), K=256, seed f,
    through gmmb_fit_k_batch (the next frame's copy overlaps this frame's
    fit): every frame bit-identical to its own fit_k, and frame 2 against
    the oracle."""
    base = frame(gm)[::2].copy()
    frames = [gm.jitter_cloud(base, 0.002, f) for f in range(4)]
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    batch = gm.fit_k_batch(frames, 256, em, seeds=list(range(4)), ctx=ctx)
    for f, (p, r) in enumerate(zip(frames, batch)):
        one = gm.fit_k(p, 256, gm.EmParams(100, 1e-3, 1e-6, f), ctx=ctx)
        assert r.em_iterations == one.em_iterations
        assert r.final_log_likelihood == one.final_log_likelihood
        assert np.array_equal(r.model.covariances, one.model.covariances)
    ref = orc.fit_k(frames[2], 256, max_iters=100, ll_rel_tol=1e-3, cov_reg=1e-6, seed=2)
    r = batch[2]
    assert r.em_iterations == ref["em_iterations"]
    assert abs(r.final_log_likelihood - ref["final_ll"]) / abs(ref["final_ll"]) < LL_TOL
    assert_model_close(r.model.weights, r.model.means, r.model.covariances,
                       ref["w"], ref["mu"], ref["cov"])
