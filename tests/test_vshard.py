"""The point-sharded fit executed for real: G virtual
ranks on one device run the sharded driver path of libgmmb (per-rank shard
upload with the (size, error) exchange, sharded k-means++ keys and rounds
with the candidate all-gather, owned-count sum + lowest-index fix-up, the
per-iteration statistics all-reduce, agreed cloud validation), the
collectives being fixed-order device reductions (comm.cu VirtualComm)
instead of NCCL. Checked against the unsharded fit and the FP64 oracle
(sogmm.cpp:197-337, 477-509).
"""
import numpy as np
import pytest

from parity import LL_TOL, assert_model_close, ll_err

pytestmark = pytest.mark.gpu


def _same_model(rs):
    for r in rs[1:]:
        assert np.array_equal(r.model.weights, rs[0].model.weights)
        assert np.array_equal(r.model.means, rs[0].model.means)
        assert np.array_equal(r.model.covariances, rs[0].model.covariances)
        assert np.array_equal(r.ll_trace, rs[0].ll_trace)
        assert r.em_iterations == rs[0].em_iterations


@pytest.mark.parametrize("world", [2, 4, 8])
def test_vshard_frame_matches_unsharded_and_oracle(gm, orc, ctx, world):
    p = gm.synthetic_frame_cloud()[::2].copy()      # 153,600 4D points
    k = 128
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    rs = gm.fit_k_vsharded(p, k, em, world=world, want_labels=True)
    _same_model(rs)
    one = gm.fit_k(p, k, em, ctx=ctx, want_labels=True)
    ref = orc.fit_k(p, k, max_iters=100, ll_rel_tol=1e-3, cov_reg=1e-6, seed=0)
    # k-means++ centres (global indices) and labels: bit-exact
    assert np.array_equal(rs[0].centers, ref["centers"])
    assert np.array_equal(np.concatenate([r.labels for r in rs]), ref["labels"])
    assert np.array_equal(one.centers, ref["centers"])
    assert rs[0].em_iterations == one.em_iterations == ref["em_iterations"]
    assert rs[0].removed_components == ref["removed"]
    assert ll_err(rs[0].ll_trace, ref["ll_trace"]) < LL_TOL
    assert ll_err(rs[0].ll_trace, one.ll_trace) < 1e-7
    m = rs[0].model
    # 2e-4: shards re-tile the cloud, so the FP32 rounding pattern differs
    # from the unsharded fit's; EM on this frame amplifies a 1e-7 relative
    # perturbation to ~1e-4 in the covariances even in FP64
    # (profiles/r2_em_sensitivity.txt), and the measured sharded/unsharded,
    # dense/pruned errors scatter over 1.4e-5 .. 1.3e-4 (scripts/vshard_err.py,
    # profiles/r2g_vshard.txt)
    assert_model_close(m.weights, m.means, m.covariances, ref["w"], ref["mu"], ref["cov"], tol=2e-4)
    # both within 2 PARAM_TOL of the oracle: within 4 PARAM_TOL of each other
    assert_model_close(m.weights, m.means, m.covariances, one.model.weights, one.model.means,
                       one.model.covariances, tol=4e-4)
    # units count every rank's points once (the global N)
    assert rs[0].units == pytest.approx(len(p) * k * rs[0].em_iterations)


def test_vshard_cfg1_fixed_init_3d(gm, orc):
    """cfg1 through the sharded fit_from: 3D, N=20,000, K=32, 50 iterations."""
    p = gm.structured_scene(20000, 1, 0.005)[:, :3]
    lab, _ = orc.kinit(p, 32, 0)
    w, mu, cov, _ = orc.m_step_labels(p, lab, 32, 1e-6)
    w, mu, cov = w, mu[:, :3].copy(), cov[:, :6].copy()
    em = gm.EmParams(50, 0.0, 1e-6)
    rs = gm.fit_k_vsharded(p, 32, em, world=4, fit_from=gm.Gmm(w, mu, cov))
    _same_model(rs)
    ref = orc.fit_from(p, w, mu, cov, max_iters=50, ll_rel_tol=0.0, cov_reg=1e-6)
    assert rs[0].em_iterations == 50
    assert ll_err(rs[0].ll_trace, ref["ll_trace"]) < LL_TOL
    m = rs[0].model
    assert_model_close(m.weights, m.means, m.covariances, ref["w"], ref["mu"], ref["cov"])


def test_vshard_duplicates_fallback_and_fixup(gm, orc):
    """Few distinct points: the fallback centres and the owned fix-up run
    across shards (donor's lowest GLOBAL index, min over ranks)."""
    base = np.array([[0, 0, 0, 0.1], [1, 0, 0, 0.2], [0, 1, 0, 0.3], [0, 0, 1, 0.4],
                     [1, 1, 1, 0.5]], float)
    p = np.repeat(base, 40, axis=0)
    em = gm.EmParams(3, 0.0, 1e-6, 0)
    rl, rc = orc.kinit(p, 8, 0)
    for world in (2, 3, 8):
        rs = gm.fit_k_vsharded(p, 8, em, world=world, want_labels=True)
        assert np.array_equal(rs[0].centers, rc), world
        assert np.array_equal(np.concatenate([r.labels for r in rs]), rl), world


def test_vshard_ragged_shards_and_key_tails(gm, orc):
    """Uneven shard sizes (N = 20,011 over 7 ranks): the column-major key
    quirk needs the 3 doubles that follow each shard's x column
    (sogmm.cpp:210-213); centres and labels stay bit-exact."""
    rng = np.random.default_rng(11)
    p = np.column_stack([rng.normal(size=(20011, 3)), rng.random(20011)])
    em = gm.EmParams(4, 0.0, 1e-6, 2)
    rs = gm.fit_k_vsharded(p, 40, em, world=7, want_labels=True)
    rl, rc = orc.kinit(p, 40, 2)
    assert np.array_equal(rs[0].centers, rc)
    assert np.array_equal(np.concatenate([r.labels for r in rs]), rl)


def test_vshard_validation_is_agreed(gm):
    """A rank whose shard is invalid makes every rank fail (no rank left
    waiting in a collective): non-finite point on one rank -> all raise
    NumericalError; an empty shard -> all raise."""
    p = gm.synthetic_frame_cloud()[::8].copy()
    p[len(p) - 5, 1] = np.nan                        # lands on the last rank
    with pytest.raises(gm.NumericalError):
        gm.fit_k_vsharded(p, 16, gm.EmParams(5, 0.0, 1e-6, 0), world=3)
    ctxs = gm.vshard_contexts(2)
    import threading
    errs = [None, None]

    def run(r, pts):
        try:
            gm.fit_k(pts, 8, gm.EmParams(3, 0.0, 1e-6, 0), ctx=ctxs[r])
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    q = gm.synthetic_frame_cloud()[::16].copy()
    th = [threading.Thread(target=run, args=(0, q)),
          threading.Thread(target=run, args=(1, q[:0]))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in th)
    assert errs[0] is not None and errs[1] is not None
    for c in ctxs:
        c.close()


def test_vshard_repeated_fits_reuse_contexts(gm):
    p = gm.synthetic_frame_cloud()[::4].copy()
    ctxs = gm.vshard_contexts(4)
    em = gm.EmParams(8, 0.0, 1e-6, 0)
    a = gm.fit_k_vsharded(p, 32, em, contexts=ctxs)
    b = gm.fit_k_vsharded(p, 32, em, contexts=ctxs)
    _same_model(a + b)                                # deterministic bits
    for c in ctxs:
        c.close()


def test_vshard_gathered_seeding_equals_per_round_exchange(gm, monkeypatch):
    """Sharded k-means++ two ways: the default gathers the cloud once and
    seeds it whole on every rank; GMMB_KINIT_SHARDED=rounds keeps the shards
    and exchanges one candidate per round. Same centres and labels."""
    p = gm.structured_scene(60000, 5, 0.005)
    em = gm.EmParams(2, 0.0, 1e-6, 3)
    a = gm.fit_k_vsharded(p, 96, em, world=3, want_labels=True)
    monkeypatch.setenv("GMMB_KINIT_SHARDED", "rounds")
    b = gm.fit_k_vsharded(p, 96, em, world=3, want_labels=True)
    assert np.array_equal(a[0].centers, b[0].centers)
    for x, y in zip(a, b):
        assert np.array_equal(x.labels, y.labels)
