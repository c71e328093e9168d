"""Tolerance metrics of BASELINE.json north_star, made well-posed as in
SURVEY.md §8(d): ll |dll|/|ll| <= 1e-5 per iteration; weights |dw|/w;
means |dmu_j| / max(|mu_j|, sigma_j); covariances |dS_ij| / sqrt(S_ii S_jj)
(regularised), each <= 1e-4. Integer results (labels, centres, iteration
counts, K) are compared exactly."""
import numpy as np

LL_TOL = 1e-5
PARAM_TOL = 1e-4


def unpack(p, d):
    m = np.zeros((d, d))
    k = 0
    for i in range(d):
        for j in range(i + 1):
            m[i, j] = m[j, i] = p[k]
            k += 1
    return m


def model_err(w, mu, cov, rw, rmu, rcov):
    """(weights, means, covariances) errors of (w, mu, cov) vs the oracle."""
    d = mu.shape[1]
    we = float(np.max(np.abs(w - rw) / rw))
    me, ce = 0.0, 0.0
    for k in range(len(rw)):
        A, B = unpack(cov[k], d), unpack(rcov[k], d)
        sig = np.sqrt(np.diag(B))
        me = max(me, float(np.max(np.abs(mu[k] - rmu[k]) / np.maximum(np.abs(rmu[k]), sig))))
        ce = max(ce, float(np.max(np.abs(A - B) / np.sqrt(np.outer(np.diag(B), np.diag(B))))))
    return we, me, ce


def ll_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.abs(b)))


def assert_model_close(w, mu, cov, rw, rmu, rcov, tol=PARAM_TOL):
    assert len(w) == len(rw), (len(w), len(rw))
    we, me, ce = model_err(w, mu, cov, rw, rmu, rcov)
    assert we <= tol and me <= tol and ce <= tol, (we, me, ce)
    return we, me, ce
