"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the FP64 CPU oracle.

The oracle (oracle/oracle.cpp) restates the reference gmmscape hot path
(kinit, e_step, m_step, cholesky_cache, the EM loop of fit) without Eigen.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
use it, as the checker / CPU baseline. The reference itself is unbuildable
here (Eigen3, libpng absent), so parity is pinned against SPEC.md's
known-answer tests (tests/test_oracle_kats.py) — see DESIGN.md §3.

3D clouds are evaluated through the exact 4D embedding [x, y, z, 0]
(SURVEY.md §8c): kinit is bit-identical, responsibilities identical up to a
per-component constant's rounding, and ll_4D = ll_3D + N(-1/2 ln 2pi -
1/2 ln cov_reg). `embed3` / `ll_offset_3d` implement that mapping.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


class _Em(ctypes.Structure):
    _fields_ = [("max_iters", ctypes.c_int), ("ll_rel_tol", ctypes.c_double),
                ("cov_reg", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("ll_offset", ctypes.c_double)]


class _Stats(ctypes.Structure):
    _fields_ = [("em_iterations", ctypes.c_int), ("final_log_likelihood", ctypes.c_double),
                ("removed_components", ctypes.c_int), ("k_out", ctypes.c_int),
                ("k_init", ctypes.c_int)]


def lib_path() -> str:
    return os.path.join(_HERE, "liboracle.so")


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return lib_path()


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(lib_path()):
            build()
        lib = ctypes.CDLL(lib_path())
        D = ctypes.POINTER(ctypes.c_double)
        I32 = ctypes.POINTER(ctypes.c_int32)
        I64 = ctypes.POINTER(ctypes.c_int64)
        I = ctypes.POINTER(ctypes.c_int)
        sig = {
            "orc_last_error": (ctypes.c_char_p, []),
            "orc_set_num_threads": (None, [ctypes.c_int]),
            "orc_num_threads": (ctypes.c_int, []),
            "orc_mix64": (ctypes.c_uint64, [ctypes.c_uint64]),
            "orc_bits": (ctypes.c_uint64, [ctypes.c_uint64] * 3),
            "orc_uniform": (ctypes.c_double, [ctypes.c_uint64] * 3),
            "orc_uniform_pos": (ctypes.c_double, [ctypes.c_uint64] * 3),
            "orc_hash_coords": (ctypes.c_uint64, [D, ctypes.c_int]),
            "orc_cholesky4": (ctypes.c_int, [D, D]),
            "orc_lower_inverse4": (None, [D, D]),
            "orc_batched_cholesky": (ctypes.c_int, [D, ctypes.c_int, D, I]),
            "orc_logsumexp_rows": (None, [D, ctypes.c_int64, ctypes.c_int64, D]),
            "orc_weighted_moments": (ctypes.c_int, [D, ctypes.c_int64, D, ctypes.c_int64,
                                                    D, D, D, I]),
            "orc_cholesky_cache": (ctypes.c_int, [D, ctypes.c_int, D, D, D]),
            "orc_validate_cloud": (ctypes.c_int, [D, ctypes.c_int64]),
            "orc_kinit": (ctypes.c_int, [D, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64,
                                         I64, I32]),
            "orc_e_step": (ctypes.c_int, [D, ctypes.c_int64, ctypes.c_int, D, D, D, D, D]),
            "orc_m_step": (ctypes.c_int, [D, ctypes.c_int64, D, ctypes.c_int, ctypes.c_double,
                                          D, D, D, I, I]),
            "orc_m_step_labels": (ctypes.c_int, [D, ctypes.c_int64, I32, ctypes.c_int,
                                                 ctypes.c_double, D, D, D, I, I]),
            "orc_fit_from": (ctypes.c_int, [D, ctypes.c_int64, ctypes.c_int, D, D, D,
                                            ctypes.POINTER(_Em), D, D, D, D,
                                            ctypes.POINTER(_Stats)]),
            "orc_fit_from_streaming": (ctypes.c_int, [D, ctypes.c_int64, ctypes.c_int, D, D, D,
                                                      ctypes.POINTER(_Em), D, D, D, D,
                                                      ctypes.POINTER(_Stats)]),
            "orc_fit_k": (ctypes.c_int, [D, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(_Em),
                                         D, D, D, D, ctypes.POINTER(_Stats), I64, I32]),
            "orc_gbms": (ctypes.c_int, [D, ctypes.c_int64, ctypes.c_double, ctypes.c_int,
                                        ctypes.c_double, ctypes.c_double, I, I, I, D,
                                        ctypes.c_int]),
            "orc_synthetic_frame_cloud": (ctypes.c_int, [ctypes.c_int, ctypes.c_int,
                                                         ctypes.c_double, D, I64]),
            "orc_structured_scene": (ctypes.c_int, [ctypes.c_int64, ctypes.c_uint64,
                                                    ctypes.c_double, D]),
            "orc_jitter_cloud": (ctypes.c_int, [D, ctypes.c_int64, ctypes.c_double,
                                                ctypes.c_uint64]),
            "orc_score": (ctypes.c_int, [D, ctypes.c_int64, ctypes.c_int, D, D, D, D]),
            "orc_sample": (ctypes.c_int, [ctypes.c_int, D, D, D, ctypes.c_int64,
                                          ctypes.c_uint64, D]),
            "orc_color_conditional": (ctypes.c_int, [ctypes.c_int, D, D, D, D, ctypes.c_int64,
                                                     ctypes.c_int, D, D]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _check(code):
    if code:
        raise OracleError(code, load().orc_last_error().decode())


def _p(a, t=ctypes.c_double):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(t))


def embed3(points) -> np.ndarray:
    """(N,3|4) -> (N,4) Fortran array; 3D gets intensity 0 (exact embedding)."""
    p = np.asarray(points, dtype=np.float64)
    if p.shape[1] == 3:
        p = np.concatenate([p, np.zeros((p.shape[0], 1))], axis=1)
    return np.asfortranarray(p)


def ll_offset_3d(n: int, cov_reg: float) -> float:
    """ll_4D - ll_3D for the [xyz, 0] embedding."""
    return n * (-0.5 * math.log(2 * math.pi) - 0.5 * math.log(cov_reg))


def embed_model3(w, mu, cov, cov_reg):
    """3D packed model -> 4D packed model with Sigma_ww = cov_reg."""
    m = len(w)
    mu4 = np.zeros((m, 4))
    mu4[:, :3] = mu
    cov4 = np.zeros((m, 10))
    cov4[:, :6] = cov
    cov4[:, 9] = cov_reg
    return np.ascontiguousarray(w, dtype=np.float64), mu4, cov4


def set_num_threads(n: int):
    load().orc_set_num_threads(n)


def num_threads() -> int:
    return load().orc_num_threads()


def kinit(points, k, seed=0):
    p = embed3(points)
    n = p.shape[0]
    lab = np.zeros(n, np.int32)
    cen = np.zeros(k, np.int64)
    _check(load().orc_kinit(_p(p), n, k, seed, _p(cen, ctypes.c_int64), _p(lab, ctypes.c_int32)))
    return lab, cen


def e_step(points, w, mu, cov):
    p = embed3(points)
    n, m = p.shape[0], len(w)
    lg = np.zeros((n, m), order="F")
    ll = ctypes.c_double()
    _check(load().orc_e_step(_p(p), n, m, _p(np.ascontiguousarray(w, dtype=np.float64)),
                             _p(np.ascontiguousarray(mu, dtype=np.float64)),
                             _p(np.ascontiguousarray(cov, dtype=np.float64)), _p(lg),
                             ctypes.byref(ll)))
    return lg, ll.value


def m_step(points, log_gamma, cov_reg):
    p = embed3(points)
    n = p.shape[0]
    lg = np.asfortranarray(log_gamma, dtype=np.float64)
    m = lg.shape[1]
    w, mu, cov = np.zeros(m), np.zeros((m, 4)), np.zeros((m, 10))
    mo, rm = ctypes.c_int(), ctypes.c_int()
    _check(load().orc_m_step(_p(p), n, _p(lg), m, cov_reg, _p(w), _p(mu), _p(cov),
                             ctypes.byref(mo), ctypes.byref(rm)))
    k = mo.value
    return w[:k], mu[:k], cov[:k], rm.value


def m_step_labels(points, labels, m, cov_reg):
    p = embed3(points)
    n = p.shape[0]
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    w, mu, cov = np.zeros(m), np.zeros((m, 4)), np.zeros((m, 10))
    mo, rm = ctypes.c_int(), ctypes.c_int()
    _check(load().orc_m_step_labels(_p(p), n, _p(lab, ctypes.c_int32), m, cov_reg, _p(w),
                                    _p(mu), _p(cov), ctypes.byref(mo), ctypes.byref(rm)))
    k = mo.value
    return w[:k], mu[:k], cov[:k], rm.value


def cholesky_cache(cov10):
    c = np.ascontiguousarray(cov10, dtype=np.float64)
    m = c.shape[0]
    lo, pr, ld = np.zeros((m, 16)), np.zeros((m, 16)), np.zeros(m)
    _check(load().orc_cholesky_cache(_p(c), m, _p(lo), _p(pr), _p(ld)))
    # column-major 4x4 -> (m, 4, 4) with [i, j] = (row i, col j)
    return (lo.reshape(m, 4, 4).transpose(0, 2, 1), pr.reshape(m, 4, 4).transpose(0, 2, 1), ld)


def logsumexp_rows(mat):
    a = np.asfortranarray(mat, dtype=np.float64)
    out = np.zeros(a.shape[0])
    load().orc_logsumexp_rows(_p(a), a.shape[0], a.shape[1], _p(out))
    return out


def weighted_moments(points, resp):
    p = embed3(points)
    r = np.asfortranarray(resp, dtype=np.float64)
    n, m = r.shape
    counts, means, sc = np.zeros(m), np.zeros((m, 4)), np.zeros((m, 16))
    deg = np.zeros(m, np.int32)
    _check(load().orc_weighted_moments(_p(p), n, _p(r), m, _p(counts), _p(means), _p(sc),
                                       _p(deg, ctypes.c_int)))
    return counts, means, sc.reshape(m, 4, 4), deg


def _fit_out(m, max_iters):
    return np.zeros(m), np.zeros((m, 4)), np.zeros((m, 10)), np.zeros(max(max_iters, 1))


def _dim(points) -> int:
    return int(np.asarray(points).shape[1])


def _slice(d, w, mu, cov):
    """4D embedded model -> D-dimensional packed model."""
    if d == 3:
        return w, mu[:, :3].copy(), cov[:, :6].copy()
    return w, mu, cov


def fit_from(points, w0, mu0, cov0, max_iters=100, ll_rel_tol=1e-5, cov_reg=1e-6,
             streaming=False):
    """EM from a given model. 3D inputs (points (N,3), model in 3D packed
    form) run through the exact embedding and report 3D quantities."""
    d = _dim(points)
    p = embed3(points)
    n, m = p.shape[0], len(w0)
    if d == 3:
        w0, mu0, cov0 = embed_model3(w0, mu0, cov0, cov_reg)
    w, mu, cov, ll = _fit_out(m, max_iters)
    st = _Stats()
    em = _Em(max_iters, ll_rel_tol, cov_reg, 0, ll_offset_3d(n, cov_reg) if d == 3 else 0.0)
    fn = load().orc_fit_from_streaming if streaming else load().orc_fit_from
    _check(fn(_p(p), n, m, _p(np.ascontiguousarray(w0, dtype=np.float64)),
              _p(np.ascontiguousarray(mu0, dtype=np.float64)),
              _p(np.ascontiguousarray(cov0, dtype=np.float64)), ctypes.byref(em), _p(w),
              _p(mu), _p(cov), _p(ll), ctypes.byref(st)))
    k = st.k_out
    w, mu, cov = _slice(d, w[:k], mu[:k], cov[:k])
    return dict(w=w, mu=mu, cov=cov, ll_trace=ll[:st.em_iterations],
                em_iterations=st.em_iterations, final_ll=st.final_log_likelihood,
                removed=st.removed_components, k_init=st.k_init)


def fit_k(points, K, max_iters=100, ll_rel_tol=1e-5, cov_reg=1e-6, seed=0):
    d = _dim(points)
    p = embed3(points)
    n = p.shape[0]
    k = min(K, n)
    w, mu, cov, ll = _fit_out(k, max_iters)
    st = _Stats()
    cen = np.zeros(k, np.int64)
    lab = np.zeros(n, np.int32)
    em = _Em(max_iters, ll_rel_tol, cov_reg, seed, ll_offset_3d(n, cov_reg) if d == 3 else 0.0)
    _check(load().orc_fit_k(_p(p), n, K, ctypes.byref(em), _p(w), _p(mu), _p(cov), _p(ll),
                            ctypes.byref(st), _p(cen, ctypes.c_int64), _p(lab, ctypes.c_int32)))
    kk = st.k_out
    w, mu, cov = _slice(d, w[:kk], mu[:kk], cov[:kk])
    return dict(w=w, mu=mu, cov=cov, ll_trace=ll[:st.em_iterations],
                em_iterations=st.em_iterations, final_ll=st.final_log_likelihood,
                removed=st.removed_components, k_init=st.k_init, centers=cen, labels=lab)


def _model4(w, mu, cov):
    return (np.ascontiguousarray(w, dtype=np.float64), np.ascontiguousarray(mu, dtype=np.float64),
            np.ascontiguousarray(cov, dtype=np.float64))


def score(points, w, mu, cov):
    """inference.cpp:141-172: average log-likelihood (4D model)."""
    p = embed3(points)
    w, mu, cov = _model4(w, mu, cov)
    out = ctypes.c_double()
    _check(load().orc_score(_p(p), p.shape[0], len(w), _p(w), _p(mu), _p(cov), ctypes.byref(out)))
    return out.value


def sample(w, mu, cov, n, seed=0):
    """inference.cpp:17-54: (n, 4) draws."""
    w, mu, cov = _model4(w, mu, cov)
    out = np.zeros((n, 4), order="F")
    _check(load().orc_sample(len(w), _p(w), _p(mu), _p(cov), n, seed, _p(out)))
    return out


def color_conditional(w, mu, cov, locs, clamp=True):
    """inference.cpp:56-139: (expected intensity, variance) at (n, 3) locations."""
    w, mu, cov = _model4(w, mu, cov)
    loc = np.asfortranarray(np.asarray(locs, dtype=np.float64)[:, :3])
    n = loc.shape[0]
    e, v = np.zeros(n), np.zeros(n)
    _check(load().orc_color_conditional(len(w), _p(w), _p(mu), _p(cov), _p(loc), n,
                                        1 if clamp else 0, _p(e), _p(v)))
    return e, v


def gbms(points, bandwidth=0.015, max_iters=100, tol=1e-5, merge_radius=-1.0):
    """sogmm.cpp:22-195: (components, iterations, initial seed count, modes (c, 4))."""
    p = embed3(points)
    comp, it, s0 = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    cap = 65536
    modes = np.zeros((cap, 4))
    _check(load().orc_gbms(_p(p), p.shape[0], bandwidth, max_iters, tol, merge_radius,
                           ctypes.byref(comp), ctypes.byref(it), ctypes.byref(s0), _p(modes), cap))
    return comp.value, it.value, s0.value, modes[:comp.value].copy()


# ---- benchmark inputs (synthetic.cpp:9-129, ingest.cpp:27-57 restated) ----
def synthetic_frame_cloud(width=640, height=480, depth_scale=1000.0):
    """make_synthetic_frame + image_pair_to_cloud: (N, 4) float64."""
    buf = np.zeros(4 * width * height)
    n = ctypes.c_int64()
    _check(load().orc_synthetic_frame_cloud(width, height, depth_scale, _p(buf),
                                            ctypes.byref(n)))
    return buf[:4 * n.value].reshape(4, n.value).T.copy()


def structured_scene(n, seed=0, noise_sigma=0.005):
    """make_structured_scene: (n, 4) float64."""
    buf = np.zeros(4 * n)
    _check(load().orc_structured_scene(n, seed, noise_sigma, _p(buf)))
    return buf.reshape(4, n).T.copy()


def jitter_cloud(points, sigma, seed):
    """cfg3 frame jitter: xyz += sigma * normal_pair(seed, 13, 4i ...)."""
    p = np.asfortranarray(np.array(points, dtype=np.float64))
    _check(load().orc_jitter_cloud(_p(p), len(p), sigma, seed))
    return np.ascontiguousarray(p)
