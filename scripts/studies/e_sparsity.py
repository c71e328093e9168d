"""How many (point, component) pairs of the E step are non-zero in FP32
(log2 density > -126), and how many candidates an interval bound over a
tile's bounding box keeps (cfg2 frame, the oracle's fitted K = 512 model).
Output: profiles/r2_e_sparsity_study.txt. (Motivates estep_sparse.cu.)"""
import os
MODEL = os.environ.get('MODEL', '/tmp/model512.npz')
import sys, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle
oracle.set_num_threads(8)
p = oracle.synthetic_frame_cloud()
t = time.time()
r = oracle.fit_k(p, 512, max_iters=15, ll_rel_tol=1e-3, cov_reg=1e-6, seed=0)
print("fit", time.time() - t, r.keys() if hasattr(r, 'keys') else type(r))
np.savez(MODEL, w=r['w'], mu=r['mu'], cov=r['cov'])

p = oracle.synthetic_frame_cloud()
m = np.load(MODEL)
w, mu, cov = m['w'], m['mu'], m['cov']
K = len(w); D = 4
iu = [(i, j) for i in range(4) for j in range(i + 1)]
print(cov.shape)
C = np.zeros((K, 4, 4))
for q, (i, j) in enumerate(iu):
    C[:, i, j] = cov[:, q]; C[:, j, i] = cov[:, q]
L = np.linalg.cholesky(C)
Li = np.linalg.inv(L)
logdet = 2 * np.log(np.diagonal(L, axis1=1, axis2=2)).sum(1)
base = np.log(w) - 0.5 * logdet - 2 * np.log(2 * np.pi)   # natural log
# morton order of points (xyz)
xyz = p[:, :3]
lo, hi = xyz.min(0), xyz.max(0)
q = ((xyz - lo) / (hi - lo + 1e-12) * 1023).astype(np.int64)
def spread(v):
    out = np.zeros_like(v)
    for b in range(10):
        out |= ((v >> b) & 1) << (3 * b)
    return out
code = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
order = np.argsort(code, kind='stable')
ps = p[order]
# component Morton order
qm = ((np.clip(mu[:, :3], lo, hi) - lo) / (hi - lo + 1e-12) * 1023).astype(np.int64)
cm = spread(qm[:, 0]) | (spread(qm[:, 1]) << 1) | (spread(qm[:, 2]) << 2)
corder = np.argsort(cm, kind='stable')
N = len(ps); P = 16
nz = np.zeros((N // P, K), bool)
tot = 0
for s in range(0, N, 16384):
    x = ps[s:s + 16384]
    d = x[:, None, :] - mu[None, :, :]            # n, K, 4
    y = np.einsum('kij,nkj->nki', Li, d)
    lg = base[None, :] - 0.5 * (y ** 2).sum(2)     # ln density
    l2 = lg / np.log(2)
    z = l2 > -126
    tot += z.sum()
    nb = z.shape[0] // P
    nz[s // P: s // P + nb] = z[:nb * P].reshape(nb, P, K).any(1)
print("unit nonzero frac", tot / (N * K))
print("per sub-tile active comps mean", nz.sum(1).mean(), "max", nz.sum(1).max())
for name, perm in [("kinit order", np.arange(K)), ("morton-sorted", corder)]:
    for G in (64, 32):
        # warp = G consecutive components in this order
        blk = nz[:, perm].reshape(nz.shape[0], K // G, G).any(2)
        print(name, "group", G, "active (group, subtile) frac", blk.mean())

def bbox_cands(T):
    nt = N // T
    counts = []
    for t0 in range(0, nt, 256):
        t1 = min(nt, t0 + 256)
        x = ps[t0 * T:t1 * T].reshape(t1 - t0, T, 4)
        lo_, hi_ = x.min(1), x.max(1)
        c = 0.5 * (lo_ + hi_); h = 0.5 * (hi_ - lo_)
        yc = np.einsum('kij,tkj->tki', Li, c[:, None, :] - mu[None])
        r = np.einsum('kij,tj->tki', np.abs(Li), h)
        dist = np.maximum(0, np.abs(yc) - r)
        lb = (dist ** 2).sum(2)
        up = (base[None] - 0.5 * lb) / np.log(2)
        counts.append((up > -134).sum(1))
    counts = np.concatenate(counts)
    return counts
for T in (16, 32, 64, 128):
    c = bbox_cands(T)
    print(f"tile {T}: bbox-bound candidates mean {c.mean():.1f} p50 {np.median(c):.0f} p99 {np.percentile(c, 99):.0f} max {c.max()}  work frac {c.mean() / K:.4f}")
