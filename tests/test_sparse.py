"""The exact-zero-pruned E step (estep_sparse.cu) and the tile-pruned
k-means++ (kinit_tile.cu) against the dense kernels / the memory-resident
seeding and the FP64 oracle (sogmm.cpp:197-337, 341-383, 399-509).

Pruning skips only pairs whose FP32 density is exactly 0, so the pruned and
dense E steps differ by FP32 summation order alone; the seeding is
decision-for-decision identical."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from parity import LL_TOL, assert_model_close, ll_err
from test_gpu_parity import fixed_init

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ctx(gm, dense):
    c = gm.Context(0)
    c.set_estep_mode(dense)
    return c


@pytest.mark.parametrize("k", [96, 512, 1536])
def test_pruned_step_matches_dense_and_oracle(gm, orc, k):
    p = gm.synthetic_frame_cloud()[::2].copy()          # 153,600 4D points
    w, mu, cov = fixed_init(orc, p, k)
    lg, rll = orc.e_step(p, w, mu, cov)
    rw, rmu, rcov, rrm = orc.m_step(p, lg, 1e-6)
    out = {}
    for dense in (True, False):
        c = _ctx(gm, dense)
        ll, m1, rm = gm.em_step(p, gm.Gmm(w, mu, cov), 1e-6, ctx=c)
        c.close()
        assert rm == rrm
        assert abs(ll - rll) / abs(rll) < LL_TOL
        # 2e-5: one step at ~100 points per component (K = 1536) sits near the
        # FP32 statistics' floor for both kernels
        assert_model_close(m1.weights, m1.means, m1.covariances, rw, rmu, rcov, tol=2e-5)
        out[dense] = (ll, m1)
    (lld, md), (llp, mp) = out[True], out[False]
    assert abs(lld - llp) / abs(lld) < 1e-7
    assert_model_close(mp.weights, mp.means, mp.covariances, md.weights, md.means, md.covariances,
                       tol=2e-5)


def test_pruned_fit_matches_dense_fit(gm, orc):
    p = gm.synthetic_frame_cloud()[::2].copy()
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    rd = gm.fit_k(p, 256, em, ctx=_ctx(gm, True), want_labels=True)
    rp = gm.fit_k(p, 256, em, ctx=_ctx(gm, False), want_labels=True)
    assert np.array_equal(rd.centers, rp.centers) and np.array_equal(rd.labels, rp.labels)
    assert rd.em_iterations == rp.em_iterations
    assert ll_err(rp.ll_trace, rd.ll_trace) < 1e-7
    # both within the bars of the oracle; EM amplifies the summation-order
    # difference
    ref = orc.fit_k(p, 256, max_iters=100, ll_rel_tol=1e-3, cov_reg=1e-6, seed=0)
    assert rp.em_iterations == ref["em_iterations"]
    assert ll_err(rp.ll_trace, ref["ll_trace"]) < LL_TOL
    assert_model_close(rp.model.weights, rp.model.means, rp.model.covariances,
                       ref["w"], ref["mu"], ref["cov"], tol=2e-4)
    # the pruned step evaluated a small fraction of the pairs; dense all of them
    assert rd.units_evaluated == rd.units
    assert 0 < rp.units_evaluated < 0.25 * rp.units


def _child(code, env):
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


_FIT = """
import json, numpy as np, paper_2307_00071_b200 as gm
p = gm.synthetic_frame_cloud()[::2].copy()
r = gm.fit_k(p, 512, gm.EmParams(100, 1e-3, 1e-6, 0))
print(json.dumps({"w": r.model.weights.tolist(), "mu": r.model.means.ravel().tolist(),
                  "cov": r.model.covariances.ravel().tolist(), "it": r.em_iterations}))
"""


def test_pool_overflow_rerun_is_bit_identical():
    """One reserved pool entry per item: every item with candidates spills
    into the overflow region, which overflows, so the EM run repeats from its
    start with larger pools until it fits. Results are bit-identical to the
    normal run (a unit's statistics do not depend on where they are stored)."""
    a = _child(_FIT, {})
    b = _child(_FIT, {"GMMB_SPARSE_ITEM_CAP": "1"})
    assert a == b


def test_split_units_with_exact_path_rerun_unsplit():
    """Heavy units are split over warps by 16-point slices. A split unit that
    needs the max-shift (exact) path could re-select different candidates in
    its sub-units, so the EM run is repeated without splits: with the exact
    path forced everywhere (GMMB_SPARSE_EXACT), the result is bit-identical
    to a run with splits disabled; and splitting moves results only at the
    rounding level."""
    forced = _child(_FIT, {"GMMB_SPARSE_EXACT": "1"})
    forced_nosplit = _child(_FIT, {"GMMB_SPARSE_EXACT": "1", "GMMB_SPARSE_NOSPLIT": "1"})
    assert forced == forced_nosplit
    a = _child(_FIT, {})
    b = _child(_FIT, {"GMMB_SPARSE_NOSPLIT": "1"})
    assert a["it"] == b["it"]
    for key in ("w", "mu", "cov"):
        x, y = np.array(a[key]), np.array(b[key])
        assert np.max(np.abs(x - y) / np.maximum(np.abs(y), 1e-3)) < 1e-6, key


_KINIT = """
import json, numpy as np, paper_2307_00071_b200 as gm
rng = np.random.default_rng(7)
s = gm.structured_scene(420000, 3, 0.005)
lab, cen = gm.kinit(s, 200, 3)
f = gm.synthetic_frame_cloud()
lab2, cen2 = gm.kinit(f, 96, 1)
print(json.dumps({"lab": int(np.sum(lab.astype(np.int64) * np.arange(len(lab)) % 1000003)),
                  "cen": cen.tolist(), "lab2": int(np.sum(lab2.astype(np.int64) * np.arange(len(lab2)) % 1000003)),
                  "cen2": cen2.tolist()}))
"""


def test_tile_kinit_equals_resident_and_memory_kernels():
    """420k points (past the shared-memory kernel): the tile kernel and the
    memory-resident rounds; the cfg2 frame: the resident kernel and the tile
    kernel forced (GMMB_KINIT=tile); the tile kernel with one round per grid
    exchange (GMMB_KPP_TILE=ws1) and with two (default). Same centres and
    labels."""
    tile = _child(_KINIT, {})
    mem = _child(_KINIT, {"GMMB_KINIT": "mem"})
    forced = _child(_KINIT, {"GMMB_KINIT": "tile"})
    one_round = _child(_KINIT, {"GMMB_KPP_TILE": "ws1", "GMMB_KINIT": "tile"})
    assert tile["cen"] == mem["cen"] and tile["lab"] == mem["lab"]
    assert tile["cen2"] == forced["cen2"] and tile["lab2"] == forced["lab2"]
    # two rounds per exchange (default) = one round per exchange
    assert one_round == forced


def test_tile_kinit_matches_oracle(gm, orc):
    s = gm.structured_scene(400000, 8, 0.005)[:, :3] * 5 + np.array([30.0, 0.0, -2.0])
    lab, cen = gm.kinit(s, 48, 2)
    rl, rc = orc.kinit(s, 48, 2)
    assert np.array_equal(cen, rc) and np.array_equal(lab, rl)
