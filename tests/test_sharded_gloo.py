"""Multi-rank host logic on CPU (world_size 2, gloo, 127.0.0.1).

The product's sharded path (gmmb_ctx_create_sharded) splits the cloud into
contiguous shards and exchanges (a) the K x (1 + D + D(D+1)/2) sufficient
statistics, centred at the previous means, with one sum all-reduce per EM
iteration, and (b) one (clock, global index) candidate per rank per
k-means++ round with an all-gather. This test runs exactly that protocol
over torch.distributed/gloo with FP64 numpy stand-ins for the per-rank
kernels and checks it against the unsharded oracle: statistics to 1e-10,
k-means++ centres bit-exact (keys use gmmb_shard_key_tail)."""
import math
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cloud():
    sys.path.insert(0, ROOT)
    import paper_2307_00071_b200 as gm
    c = np.array([[0.1, 0.2, 0.3, 0.2], [0.6, 0.5, 0.4, 0.5], [0.9, 0.1, 0.8, 0.7],
                  [0.3, 0.8, 0.6, 0.9]])
    return gm.blob_cloud(c, 0.05, 150, seed=21)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import oracle
    import paper_2307_00071_b200 as gm
    from test_rng_keys import bits, hash_coords

    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = _cloud()
    n = len(x)
    bounds = np.linspace(0, n, world + 1).astype(int)
    lo, hi = bounds[rank], bounds[rank + 1]
    xs = x[lo:hi]
    res = {}

    # (a) one EM iteration: local E step + centred statistics, all-reduce
    lab, _ = oracle.kinit(x, 4, 0)
    w, mu, cov, _ = oracle.m_step_labels(x, lab, 4, 1e-6)
    lg, ll_local = oracle.e_step(xs, w, mu, cov)
    r = np.exp(lg)
    d = xs[:, None, :] - mu[None, :, :]                      # (n, K, 4)
    s0 = r.sum(0)
    s1 = np.einsum("nk,nkd->kd", r, d)
    s2 = np.einsum("nk,nki,nkj->kij", r, d, d)
    buf = torch.from_numpy(np.concatenate([s0, s1.ravel(), s2.ravel(), [ll_local]]))
    dist.all_reduce(buf)
    b = buf.numpy()
    k = 4
    s0, s1 = b[:k], b[k:k + 4 * k].reshape(k, 4)
    s2 = b[5 * k:5 * k + 16 * k].reshape(k, 4, 4)
    delta = s1 / s0[:, None]
    mean = mu + delta
    scat = s2 / s0[:, None, None] - delta[:, :, None] * delta[:, None, :]
    lg_full, ll_full = oracle.e_step(x, w, mu, cov)
    w2, mu2, cov2, _ = oracle.m_step(x, lg_full, 1e-6)
    res["ll_err"] = abs(b[-1] - ll_full) / abs(ll_full)
    res["w_err"] = float(np.max(np.abs(s0 / s0.sum() - w2)))
    res["mu_err"] = float(np.max(np.abs(mean - mu2)))
    r_, c_ = np.array([0, 1, 1, 2, 2, 2, 3, 3, 3, 3]), np.array([0, 0, 1, 0, 1, 2, 0, 1, 2, 3])
    res["cov_err"] = float(np.max(np.abs(scat[:, r_, c_] + 1e-6 * (r_ == c_) - cov2)))

    # (b) sharded k-means++: local (clock, global index) -> all-gather -> min
    heads = np.zeros(8)
    m = min(3, len(xs))
    heads[:m], heads[3:3 + m], heads[6] = xs[:m, 0], xs[:m, 1], len(xs)
    allh = [None] * world
    dist.all_gather_object(allh, heads.tolist())
    tail = gm.shard_key_tail(np.array(allh), rank)
    flat_x = np.concatenate([xs[:, 0], tail])
    keys = [hash_coords([flat_x[i], flat_x[i + 1], flat_x[i + 2], flat_x[i + 3]])
            for i in range(len(xs))]
    d2 = np.full(len(xs), np.inf)
    centers = []
    c = None
    for rnd in range(6):
        if c is not None:
            e = xs - c
            d2 = np.minimum(d2, ((e[:, 0] * e[:, 0] + e[:, 1] * e[:, 1]) + e[:, 2] * e[:, 2])
                            + e[:, 3] * e[:, 3])
        best = (math.inf, -1)
        for i in range(len(xs)):
            u = ((bits(0, rnd, keys[i]) >> 11) + 1) * 2.0**-53
            nl = -math.log(u)
            if rnd == 0:
                cand = (nl, lo + i)
            elif d2[i] > 0:
                cand = (nl / d2[i], lo + i)
            else:
                continue
            if cand < best:
                best = cand
        got = [None] * world
        dist.all_gather_object(got, best)
        win = min(got)[1]
        centers.append(win)
        c = x[win]
    full_lab, full_cen = oracle.kinit(x, 6, 0)
    res["centers_equal"] = centers == full_cen.tolist()
    out[rank] = res
    dist.destroy_process_group()


def test_two_rank_protocol_matches_unsharded():
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for rank in range(2):
        r = out[rank]
        assert r["ll_err"] < 1e-12
        assert r["w_err"] < 1e-12 and r["mu_err"] < 1e-10 and r["cov_err"] < 1e-10
        assert r["centers_equal"], "sharded k-means++ diverged from the oracle"
