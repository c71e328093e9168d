"""Accuracy study: quadratic-feature GEMM E step (tensor-core formulation)
against the FP64 oracle, on the cfg2 frame with the oracle's fitted K=512
model (north_star: 'A quadratic-feature GEMM formulation of the E-step on
tensor cores is evaluated and adopted only if ... accuracy holds').

log w_k N(x | mu_k, S_k) = c_k + phi(x) . theta_k with phi(x) = [1, x,
upper(x x^T)] (15 features at D = 4) is an N x 15 by 15 x K GEMM. Inputs
are tile-relative (x - c_t, mu - c_t) exactly as the CUDA-core kernel uses.
Compared: the shipped CUDA-core form |P'(x - mu')|^2 in FP32, and the
feature GEMM with FP32 operands / FP32 accumulation (best case for any
tensor-core path: 3xTF32 or BF16x9 emulation at best reaches this), TF32
operands (kind::tf32) and BF16 operands (kind::f16). Metric: max |error| of
the log2 density over (point, component) pairs whose responsibility is
> 1e-6 (the pairs that move the statistics), and the resulting max error
of the responsibilities.

usage: python scripts/studies/quadfeat_accuracy.py  (CPU only, ~1 min)
"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
import oracle
import paper_2307_00071_b200 as gm

pts = gm.synthetic_frame_cloud()
n = len(pts)
ref = oracle.fit_k(pts, 512, 100, 1e-3, 1e-6, 0)
w, mu, cov = ref["w"], ref["mu"], ref["cov"]
K = len(w)
LOG2E = 1.4426950408889634
# tiles of 128 points in Morton order are ~5 cm; emulate with 128-point
# chunks of a spatially sorted copy (row-major pixels, 16-pixel strips)
order = np.lexsort((np.arange(n) % 640 // 16, np.arange(n) // 640 // 8))
P = pts[order]
rng = np.random.default_rng(0)
sel = rng.choice(n // 128, 200, replace=False)  # 200 random tiles

def chol_prec(c10):
    S = np.zeros((4, 4))
    idx = [(0, 0), (1, 0), (1, 1), (2, 0), (2, 1), (2, 2), (3, 0), (3, 1), (3, 2), (3, 3)]
    for q, (i, j) in enumerate(idx):
        S[i, j] = S[j, i] = c10[q]
    L = np.linalg.cholesky(S)
    return np.linalg.inv(L), S

Pk, Lam, base = [], [], []
for k in range(K):
    Pm, S = chol_prec(cov[k])
    Pk.append(Pm)
    Lam.append(np.linalg.inv(S))
    base.append(np.log(w[k]) + np.sum(np.log(np.diag(Pm))) - 2 * np.log(2 * np.pi))
Pk, Lam, base = np.array(Pk), np.array(Lam), np.array(base)

def rnd(a, bits):  # round-to-nearest mantissa truncation (TF32: 10, BF16: 7)
    a = np.asarray(a, np.float32)
    i = a.view(np.uint32).astype(np.uint64)
    sh = 23 - bits
    i = ((i + (1 << (sh - 1))) >> sh) << sh
    return i.astype(np.uint32).view(np.float32)

err = {"cudacore_fp32": 0.0, "gemm_fp32": 0.0, "gemm_tf32": 0.0, "gemm_bf16": 0.0}
rerr = dict.fromkeys(err, 0.0)
for t in sel:
    X = P[t * 128:(t + 1) * 128]
    c = X.mean(axis=0)
    xr = X - c
    mr = mu - c
    # FP64 truth (natural log density)
    d = xr[:, None, :] - mr[None, :, :]
    y = np.einsum("kij,nkj->nki", Pk, d)
    l64 = base[None, :] - 0.5 * np.sum(y * y, axis=2)
    lse = np.log(np.sum(np.exp(l64 - l64.max(1, keepdims=True)), 1)) + l64.max(1)
    r64 = np.exp(l64 - lse[:, None])
    mask = r64 > 1e-6
    # shipped CUDA-core form in FP32 (P'x - P'mu' chains, then squares)
    xf, mf, Pf = xr.astype(np.float32), mr.astype(np.float32), Pk.astype(np.float32)
    nb = -np.einsum("kij,kj->ki", Pk, mf.astype(np.float64)).astype(np.float32)
    yf = np.einsum("kij,nj->nki", Pf, xf) + nb[None]
    lf = base.astype(np.float32)[None] - np.float32(0.5) * np.sum(yf * yf, axis=2)
    # quadratic features: theta_k from Lam_k, mu'_k (FP64 -> operand precision)
    iu = np.triu_indices(4)
    feat = np.concatenate([np.ones((128, 1)), xr, (xr[:, :, None] * xr[:, None, :])[:, iu[0], iu[1]]], 1)
    th = np.zeros((K, 15))
    for k in range(K):
        L_, m_ = Lam[k], mr[k]
        th[k, 0] = base[k] - 0.5 * m_ @ L_ @ m_
        th[k, 1:5] = L_ @ m_
        Q = -0.5 * L_ * (2 - np.eye(4))  # off-diagonal pairs counted once
        th[k, 5:] = Q[iu]
    for name, bits in [("gemm_fp32", 23), ("gemm_tf32", 10), ("gemm_bf16", 7)]:
        fa = rnd(feat, bits) if bits < 23 else feat.astype(np.float32)
        tb = rnd(th, bits) if bits < 23 else th.astype(np.float32)
        lg = (fa.astype(np.float32) @ tb.T.astype(np.float32)).astype(np.float64)
        e = np.abs(lg - l64)[mask].max() * LOG2E
        err[name] = max(err[name], e)
        lse_g = np.log(np.sum(np.exp(lg - lg.max(1, keepdims=True)), 1)) + lg.max(1)
        rerr[name] = max(rerr[name], np.abs(np.exp(lg - lse_g[:, None]) - r64).max())
    e = np.abs(lf.astype(np.float64) - l64)[mask].max() * LOG2E
    err["cudacore_fp32"] = max(err["cudacore_fp32"], e)
    lse_f = np.log(np.sum(np.exp(lf - lf.max(1, keepdims=True)), 1)) + lf.max(1)
    rerr["cudacore_fp32"] = max(rerr["cudacore_fp32"], np.abs(np.exp(lf - lse_f[:, None]) - r64).max())
print("max |log2 density error| over pairs with r > 1e-6, and max |responsibility error|,")
print("cfg2 frame, oracle-fitted K=512 model, 200 tiles of 128 points:")
for k in err:
    print(f"  {k:15s} log2-density {err[k]:.3e}   responsibility {rerr[k]:.3e}")
