"""Small fits that reach every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck). scripts/sanitize.sh runs this file under
each tool; the logs go to profiles/.

usage: python scripts/sanitize_cases.py [case ...]   (default: all)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2307_00071_b200 as gm


def blobs(d, k, per, seed):
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.0, 1.0, size=(k, d))
    return gm.blob_cloud(np.pad(c, ((0, 0), (0, 4 - d))), 0.02, per, seed=seed)[:, :d].copy()


def case_ws():
    """single-CTA warp-specialised E kernel, register kinit, graph + timing."""
    pts = blobs(4, 12, 300, 1)
    for timing in (False, True):
        ctx = gm.Context(0)
        ctx.set_timing(timing)
        r = gm.fit_k(pts, 24, gm.EmParams(6, 1e-4, 1e-6, 0), ctx=ctx)
        print("ws", timing, r.k_init, r.em_iterations, r.final_log_likelihood)
        ctx.close()


def case_ws_t():
    """as ws, plain launches only (no CUDA graph)."""
    pts = blobs(4, 12, 300, 1)
    ctx = gm.Context(0)
    ctx.set_timing(True)
    r = gm.fit_k(pts, 24, gm.EmParams(6, 1e-4, 1e-6, 0), ctx=ctx)
    print("ws_t", r.k_init, r.em_iterations, r.final_log_likelihood)
    ctx.close()


def case_ws_g():
    """as ws, the EM loop as one CUDA graph only."""
    pts = blobs(4, 12, 300, 1)
    ctx = gm.Context(0)
    r = gm.fit_k(pts, 24, gm.EmParams(6, 1e-4, 1e-6, 0), ctx=ctx)
    print("ws_g", r.k_init, r.em_iterations, r.final_log_likelihood)
    ctx.close()


def case_sparse_split():
    """the pruned E step with heavy units split over warps (the frame at
    K = 512 has units with up to ~400 candidates), plain launches then graph."""
    pts = gm.synthetic_frame_cloud()[::4].copy()
    for timing in (True, False):
        ctx = gm.Context(0)
        ctx.set_timing(timing)
        r = gm.fit_k(pts, 512, gm.EmParams(4, 0.0, 1e-6, 0), ctx=ctx)
        print("sparse_split", timing, r.em_iterations, r.final_log_likelihood, r.units_evaluated)
        ctx.close()


def case_sparse_split_g():
    """as sparse_split, the EM graph only (fresh process)."""
    pts = gm.synthetic_frame_cloud()[::4].copy()
    ctx = gm.Context(0)
    r = gm.fit_k(pts, 512, gm.EmParams(4, 0.0, 1e-6, 0), ctx=ctx)
    print("sparse_split_g", r.em_iterations, r.final_log_likelihood, r.units_evaluated)
    ctx.close()


def case_sparse_exact():
    """as sparse_split with the exact path forced on every slice: the split
    conflict is flagged and the EM run repeated without splits."""
    os.environ["GMMB_SPARSE_EXACT"] = "1"
    pts = gm.synthetic_frame_cloud()[::4].copy()
    ctx = gm.Context(0)
    ctx.set_timing(True)
    r = gm.fit_k(pts, 512, gm.EmParams(3, 0.0, 1e-6, 0), ctx=ctx)
    print("sparse_exact", r.em_iterations, r.final_log_likelihood)
    ctx.close()


def case_dense():
    """the dense E kernels (warp-specialised K <= 512, chunked K > 512)."""
    pts = blobs(4, 12, 300, 1)
    ctx = gm.Context(0)
    ctx.set_estep_mode(True)
    r = gm.fit_k(pts, 24, gm.EmParams(4, 1e-4, 1e-6, 0), ctx=ctx)
    r2 = gm.fit_k(pts, 600 if len(pts) >= 600 else 100, gm.EmParams(2, 0.0, 1e-6, 0), ctx=ctx)
    print("dense", r.em_iterations, r2.em_iterations)
    ctx.close()


def case_cluster():
    """K > 512 through the pruned E step (block candidate lists, items)."""
    pts = blobs(4, 40, 200, 2)
    r = gm.fit_k(pts, 600, gm.EmParams(3, 0.0, 1e-6, 0))
    print("k600", r.k_init, r.em_iterations, r.final_log_likelihood)
    pts3 = blobs(3, 40, 150, 3)
    r = gm.fit_k(pts3, 1100, gm.EmParams(2, 0.0, 1e-6, 0))
    print("k1100 d3", r.k_init, r.em_iterations, r.final_log_likelihood)


def case_kinit_mem():
    """k-means++ past the shared-memory budget (tile-pruned warp-specialised
    kernel; GMMB_KINIT=mem selects the memory-resident rounds)."""
    rng = np.random.default_rng(4)
    pts = rng.uniform(0.0, 1.0, size=(400_000, 3))
    lab, cen = gm.kinit(pts, 5, seed=1)
    print("kinit mem", cen, int(lab.max()))


def case_vshard():
    """sharded driver (virtual ranks: comm layer, sharded kinit rounds, fix-up)."""
    pts = blobs(4, 8, 250, 5)
    r = gm.fit_k_vsharded(pts, 16, gm.EmParams(4, 0.0, 1e-6, 0), world=2)[0]
    print("vshard", r.k_init, r.em_iterations, r.final_log_likelihood)


def case_batch():
    """cfg3-style frame batch (two streams)."""
    frames = [blobs(4, 6, 200, 10 + i) for i in range(3)]
    rs = gm.fit_k_batch(frames, 12, gm.EmParams(4, 1e-4, 1e-6, 0))
    print("batch", [r.em_iterations for r in rs])


def case_aux():
    """GBMS, fit via GBMS, single-step APIs, inference, ingest."""
    pts = blobs(4, 5, 150, 6)
    gp = gm.GbmsParams()
    comp, it, _ = gm.gbms(pts, gp)
    print("gbms", comp, it)
    r = gm.fit(pts, gp, gm.EmParams(4, 1e-4, 1e-6, 0))
    m = r.model
    lg, _ = gm.e_step(pts, m)
    gm.m_step(pts, lg)
    gm.em_step(pts, m)
    gm.score(pts, m, per_point=True)
    gm.joint_dist_sample(m, 500, seed=1)
    gm.color_conditional(m, pts[:200, :3])
    gm.cholesky_cache(m)
    depth, inten, intr = gm.synthetic_frame_images(64, 48)
    ctx = gm.Context(0)
    ctx.ingest_images(depth, inten, intr)
    ctx.close()
    print("aux ok")


CASES = {"ws": case_ws, "sparse_split": case_sparse_split, "sparse_split_g": case_sparse_split_g, "sparse_exact": case_sparse_exact, "ws_t": case_ws_t, "ws_g": case_ws_g, "dense": case_dense, "cluster": case_cluster, "kinit_mem": case_kinit_mem,
         "vshard": case_vshard, "batch": case_batch, "aux": case_aux}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
