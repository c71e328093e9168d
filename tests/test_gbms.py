"""§8(f) row 1: GBMS component estimation (sogmm.cpp:22-195) on the device
vs the oracle (which restates the reference's kd-tree, kdtree.hpp, so its
radius queries visit seeds in the reference's order). The device sums
neighbours in grid order, so seeds differ at the rounding level only:
component and iteration counts must match exactly, modes within 1e-9."""
import numpy as np
import pytest

from parity import LL_TOL, assert_model_close


def test_oracle_gbms_invariants(gm, orc):
    # two well separated blobs -> two modes near the blob centres
    centers = np.array([[0.1, 0.1, 0.1, 0.2], [0.9, 0.9, 0.9, 0.8]])
    p = gm.blob_cloud(centers, 0.01, 2000, seed=1)
    comp, it, s0, modes = orc.gbms(p, 0.1)
    assert comp == 2 and s0 >= comp and it >= 1
    assert np.allclose(np.sort(modes[:, 0]), [0.1, 0.9], atol=0.02)
    with pytest.raises(orc.OracleError):
        orc.gbms(p, 1.5)


@pytest.mark.gpu
@pytest.mark.parametrize("case,bw", [("frame", 0.03), ("frame", 0.015), ("scene", 0.03),
                                     ("blobs", 0.1)])
def test_gbms_matches_oracle(gm, orc, ctx, case, bw):
    if case == "frame":
        p = gm.synthetic_frame_cloud()
    elif case == "scene":
        p = gm.structured_scene(20000, 1, 0.005)[:, :3]
    else:
        p = gm.blob_cloud(np.array([[0.1, 0.1, 0.1, 0.2], [0.5, 0.4, 0.6, 0.5],
                                    [0.9, 0.9, 0.9, 0.8]]), 0.02, 5000, seed=4)
    comp, it, modes = gm.gbms(p, gm.GbmsParams(bandwidth=bw), ctx=ctx)
    rc, rit, _, rmodes = orc.gbms(p, bw)
    assert (comp, it) == (rc, rit)
    scale = np.maximum(np.abs(rmodes), 1.0)
    assert np.max(np.abs(modes[:, :p.shape[1]] - rmodes[:, :p.shape[1]]) / scale[:, :p.shape[1]]) < 1e-9


@pytest.mark.gpu
def test_fit_with_gbms(gm, orc, ctx):
    p = gm.synthetic_frame_cloud(160, 120)
    r = gm.fit(p, gm.GbmsParams(bandwidth=0.05), gm.EmParams(50, 1e-3, 1e-6, 0), ctx=ctx)
    rc, _, _, _ = orc.gbms(p, 0.05)
    assert r.gbms_components == rc and r.k_init == min(rc, len(p))
    ref = orc.fit_k(p, rc, 50, 1e-3, 1e-6, 0)
    assert r.em_iterations == ref["em_iterations"]
    assert abs(r.final_log_likelihood - ref["final_ll"]) <= 1e-5 * abs(ref["final_ll"])
    with pytest.raises(ValueError, match="bandwidth"):
        gm.fit(p, gm.GbmsParams(bandwidth=0.0), ctx=ctx)


@pytest.mark.gpu
def test_gbms_merge_radius_above_bandwidth(gm, orc, ctx):
    """merge_radius > bandwidth: the merge grid's cells are as wide as the
    merge radius (sogmm.cpp:148-168 links every pair within it)."""
    p = gm.synthetic_frame_cloud()
    comp, it, modes = gm.gbms(p, gm.GbmsParams(bandwidth=0.03, merge_radius=0.05), ctx=ctx)
    rc, rit, _, rmodes = orc.gbms(p, 0.03, merge_radius=0.05)
    assert (comp, it) == (rc, rit)
    assert np.max(np.abs(modes - rmodes) / np.maximum(np.abs(rmodes), 1.0)) < 1e-9


@pytest.mark.gpu
def test_gbms_tiny_bandwidth_cells_beyond_16_bits(gm, orc, ctx):
    """bandwidth < 1/65535: cell coordinates beyond 16 bits (hashed keys)."""
    rng = np.random.default_rng(3)
    p = np.column_stack([rng.random((3000, 3)) * 1e-3, rng.random(3000)])
    p[:1500, :3] += 1.0   # two far clusters: normalised bandwidth 1e-5 of the range
    comp, it, modes = gm.gbms(p, gm.GbmsParams(bandwidth=1e-5), ctx=ctx)
    rc, rit, _, rmodes = orc.gbms(p, 1e-5)
    assert (comp, it) == (rc, rit)
    assert np.all(np.isfinite(modes))


@pytest.mark.gpu
@pytest.mark.slow
def test_fit_default_bandwidth_above_4096_components(gm, orc, ctx):
    """fit(cloud, 0.015) on the cfg2 frame: GBMS finds 5,844 components, so
    K > 4096 (sogmm.cpp:475-477 accepts any K <= N). GBMS count vs the
    oracle, k-means++ centres bit-exact, one EM step (E + M) from the
    oracle's initial model within the BASELINE bars, and fit() == fit_k(K)
    bitwise."""
    p = gm.synthetic_frame_cloud()
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    r = gm.fit(p, gm.GbmsParams(bandwidth=0.015), em, ctx=ctx)
    rc, _, _, _ = orc.gbms(p, 0.015)
    assert r.gbms_components == rc == r.k_init and rc > 4096
    rk = gm.fit_k(p, rc, em, ctx=ctx)
    assert np.array_equal(rk.ll_trace, r.ll_trace)
    assert np.array_equal(rk.model.covariances, r.model.covariances)
    lab, cen = gm.kinit(p, rc, 0, ctx=ctx)
    rl, rcen = orc.kinit(p, rc, 0)
    assert np.array_equal(cen, rcen) and np.array_equal(lab, rl)
    w, mu, cov, _ = orc.m_step_labels(p, rl, rc, 1e-6)
    one = gm.fit_from(p, gm.Gmm(w, mu, cov), gm.EmParams(1, 0.0, 1e-6), ctx=ctx)
    ref = orc.fit_from(p, w, mu, cov, max_iters=1, ll_rel_tol=0.0, cov_reg=1e-6, streaming=True)
    assert abs(one.final_log_likelihood - ref["final_ll"]) / abs(ref["final_ll"]) < LL_TOL
    # the first step from the hard-assignment model (~53 points per
    # component): the BASELINE bar (1.8e-5 measured)
    assert_model_close(one.model.weights, one.model.means, one.model.covariances,
                       ref["w"], ref["mu"], ref["cov"])
