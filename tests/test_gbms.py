"""§8(f) row 1: GBMS component estimation (sogmm.cpp:22-195) on the device
vs the oracle (which restates the reference's kd-tree, kdtree.hpp, so its
radius queries visit seeds in the reference's order). The device sums
neighbours in grid order, so seeds differ at the rounding level only:
component and iteration counts must match exactly, modes within 1e-9."""
import numpy as np
import pytest


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
