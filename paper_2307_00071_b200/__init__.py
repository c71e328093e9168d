"""B200-native Gaussian-mixture learner (k-means++ init + full-covariance EM).

Host-side mirror of the reference's fit API (gmmscape, /root/reference/proj/
include/gmmscape/sogmm.hpp + gmm.hpp) over the C ABI in include/gmmb.h
(libgmmb.so, built in-tree from paper_2307_00071_b200/csrc). Every compute
call runs the CUDA library; there is no CPU fallback — importing this module
without the built library raises.

Reference -> this module:
  EmParams            sogmm.hpp:36-41          EmParams
  Gmm4                gmm.hpp:15-34            Gmm (D = 3 or 4)
  FitResult           sogmm.hpp:65-71          FitResult
  kinit               sogmm.hpp:52             kinit
  e_step              sogmm.hpp:55-57          e_step
  m_step              sogmm.hpp:62-63          m_step
  fit(cloud, bw, em)  sogmm.hpp:74-75          fit_k(points, K, em)  (K given
                                               instead of GBMS-estimated) and
                                               fit_from(points, model, em)
  cholesky_cache      gmm.hpp:52               cholesky_cache
  NumericalError      common.hpp:27-30         NumericalError
  std::invalid_argument                        ValueError
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Optional

import numpy as np

__all__ = [
    "EmParams", "Gmm", "FitResult", "CholeskyCache", "Context",
    "NumericalError", "IoError", "fit_k", "fit_from", "kinit", "e_step",
    "m_step", "em_step", "cholesky_cache", "synthetic_frame_cloud",
    "structured_scene", "blob_cloud", "jitter_cloud", "lib_path", "load",
]

_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    # GMMB_LIB: alternative build of the same library (precision experiments)
    return os.environ.get("GMMB_LIB") or os.path.join(_HERE, "libgmmb.so")


class NumericalError(RuntimeError):
    """common.hpp:27-30 — non-SPD matrices, degenerate models, bad clouds."""


class IoError(RuntimeError):
    """common.hpp:23-25 — here: CUDA / NCCL / device failures (code 1)."""


class _EmParams(ctypes.Structure):
    _fields_ = [("max_iters", ctypes.c_int), ("ll_rel_tol", ctypes.c_double),
                ("cov_reg", ctypes.c_double), ("seed", ctypes.c_uint64)]


class _GbmsParams(ctypes.Structure):  # gmmb_gbms_params (sogmm.hpp:12-22)
    _fields_ = [("bandwidth", ctypes.c_double), ("max_iters", ctypes.c_int),
                ("convergence_tol", ctypes.c_double), ("merge_radius", ctypes.c_double)]


class _FitStats(ctypes.Structure):
    _fields_ = [("em_iterations", ctypes.c_int),
                ("final_log_likelihood", ctypes.c_double),
                ("removed_components", ctypes.c_int), ("k_out", ctypes.c_int),
                ("k_init", ctypes.c_int), ("converged", ctypes.c_int),
                ("ms_layout", ctypes.c_double), ("ms_kinit", ctypes.c_double),
                ("ms_mstep0", ctypes.c_double), ("ms_em", ctypes.c_double),
                ("units", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("ms_estep", ctypes.c_double), ("launches", ctypes.c_longlong),
                ("units_evaluated", ctypes.c_double)]


_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I32 = ctypes.POINTER(ctypes.c_int32)
_I64 = ctypes.POINTER(ctypes.c_int64)
_I = ctypes.POINTER(ctypes.c_int)
_V = ctypes.c_void_p
_SIGS = {
    "gmmb_last_error": (ctypes.c_char_p, []),
    "gmmb_em_params_default": (None, [ctypes.POINTER(_EmParams)]),
    "gmmb_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_V)]),
    "gmmb_nccl_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "gmmb_ctx_create_sharded": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_char_p, ctypes.POINTER(_V)]),
    "gmmb_ctx_destroy": (None, [_V]),
    "gmmb_vgroup_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(_V)]),
    "gmmb_vgroup_release": (None, [_V]),
    "gmmb_ctx_create_virtual": (ctypes.c_int, [_V, ctypes.c_int, ctypes.POINTER(_V)]),
    "gmmb_device_info": (ctypes.c_int, [_V, _I, _I, _I]),
    "gmmb_fit_k": (ctypes.c_int, [_V, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                  ctypes.POINTER(_EmParams), _D, _D, _D, _D,
                                  ctypes.POINTER(_FitStats), _I32, _I64]),
    "gmmb_fit_k_batch": (ctypes.c_int, [_V, ctypes.c_int, ctypes.POINTER(_D), _I64, ctypes.c_int,
                                        ctypes.c_int, ctypes.POINTER(_EmParams),
                                        ctypes.POINTER(ctypes.c_uint64), _D, _D, _D,
                                        ctypes.POINTER(_FitStats)]),
    "gmmb_fit_from": (ctypes.c_int, [_V, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                     _D, _D, _D, ctypes.POINTER(_EmParams), _D, _D, _D, _D,
                                     ctypes.POINTER(_FitStats)]),
    "gmmb_upload": (ctypes.c_int, [_V, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
                                   ctypes.c_int64]),
    "gmmb_fit_k_resident": (ctypes.c_int, [_V, ctypes.c_int, ctypes.POINTER(_EmParams),
                                           _D, _D, _D, _D, ctypes.POINTER(_FitStats),
                                           _I32, _I64]),
    "gmmb_fit_from_resident": (ctypes.c_int, [_V, ctypes.c_int, _D, _D, _D,
                                              ctypes.POINTER(_EmParams), _D, _D, _D, _D,
                                              ctypes.POINTER(_FitStats)]),
    "gmmb_kinit": (ctypes.c_int, [_V, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_uint64, _I32, _I64]),
    "gmmb_e_step": (ctypes.c_int, [_V, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                   _D, _D, _D, _D, _D]),
    "gmmb_m_step": (ctypes.c_int, [_V, _D, ctypes.c_int64, ctypes.c_int, _D, ctypes.c_int,
                                   ctypes.c_double, _D, _D, _D, _I, _I]),
    "gmmb_em_step": (ctypes.c_int, [_V, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                    _D, _D, _D, ctypes.c_double, _D, _D, _D, _D, _I, _I]),
    "gmmb_cholesky_cache": (ctypes.c_int, [_V, ctypes.c_int, ctypes.c_int, _D, _D, _D, _D]),
    "gmmb_synthetic_frame_cloud": (ctypes.c_int, [ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_double, _D, _I64]),
    "gmmb_structured_scene": (ctypes.c_int, [ctypes.c_int64, ctypes.c_uint64,
                                             ctypes.c_double, _D]),
    "gmmb_blob_cloud": (ctypes.c_int, [_D, ctypes.c_int, ctypes.c_double, ctypes.c_int64,
                                       ctypes.c_uint64, _D]),
    "gmmb_jitter_cloud": (ctypes.c_int, [_D, ctypes.c_int64, ctypes.c_double,
                                         ctypes.c_uint64]),
    "gmmb_shard_key_tail": (ctypes.c_int, [_D, ctypes.c_int, ctypes.c_int, _D]),
    "gmmb_ffma_peak": (ctypes.c_int, [_V, ctypes.c_double, _D, _D]),
    "gmmb_ctx_set_timing": (ctypes.c_int, [_V, ctypes.c_int]),
    "gmmb_ctx_set_estep_mode": (ctypes.c_int, [_V, ctypes.c_int]),
    "gmmb_ingest_images": (ctypes.c_int, [_V, ctypes.POINTER(ctypes.c_uint16),
                                          ctypes.POINTER(ctypes.c_uint16), ctypes.c_int,
                                          ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_int, _D,
                                          ctypes.POINTER(ctypes.c_int64)]),
    "gmmb_synthetic_frame_images": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                                   ctypes.POINTER(ctypes.c_uint16),
                                                   ctypes.POINTER(ctypes.c_uint16), _D]),
    "gmmb_io_last_error": (ctypes.c_char_p, []),
    "gmmb_save_model": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _D, _D, _D]),
    "gmmb_load_model": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _D, _D, _D,
                                       ctypes.POINTER(ctypes.c_int)]),
    "gmmb_save_model_json": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _D, _D, _D]),
    "gmmb_load_model_json": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _D, _D, _D,
                                            ctypes.POINTER(ctypes.c_int)]),
    "gmmb_gbms": (ctypes.c_int, [_V, _D, ctypes.c_int64, ctypes.c_int,
                                 ctypes.POINTER(_GbmsParams), ctypes.POINTER(ctypes.c_int),
                                 ctypes.POINTER(ctypes.c_int), _D, ctypes.c_int]),
    "gmmb_fit": (ctypes.c_int, [_V, _D, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(_GbmsParams),
                                ctypes.POINTER(_EmParams), ctypes.c_int, _D, _D, _D, _D,
                                ctypes.POINTER(_FitStats), ctypes.POINTER(ctypes.c_int)]),
    "gmmb_score": (ctypes.c_int, [_V, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _D, _D, _D,
                                  _D, _D]),
    "gmmb_sample": (ctypes.c_int, [_V, ctypes.c_int, ctypes.c_int, _D, _D, _D, ctypes.c_int64,
                                   ctypes.c_uint64, _D]),
    "gmmb_color_conditional": (ctypes.c_int, [_V, ctypes.c_int, _D, _D, _D, _D, ctypes.c_int64,
                                              ctypes.c_int, _D, _D]),
}


def load() -> ctypes.CDLL:
    """Loads libgmmb.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        p = lib_path()
        if not os.path.exists(p):
            raise ImportError(
                f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        lib = ctypes.CDLL(p)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(code: int) -> None:
    if code == 0:
        return
    msg = load().gmmb_last_error().decode(errors="replace")
    if code == 2:
        raise ValueError(msg)
    if code == 3:
        raise NumericalError(msg)
    raise IoError(msg)


def _ptr(a: Optional[np.ndarray], t=_D):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def _points(points) -> tuple[np.ndarray, int, int]:
    """(N, D) array-like -> Fortran-ordered float64 (Eigen MatX4 layout)."""
    p = np.asarray(points, dtype=np.float64)
    if p.ndim != 2 or p.shape[1] not in (3, 4):
        raise ValueError("points must be an (N, 3) or (N, 4) array")
    return np.asfortranarray(p), p.shape[0], p.shape[1]


@dataclasses.dataclass
class EmParams:
    """sogmm.hpp:36-41. ll_rel_tol = 0 runs exactly max_iters E steps."""
    max_iters: int = 100
    ll_rel_tol: float = 1e-5
    cov_reg: float = 1e-6
    seed: int = 0

    def _c(self) -> _EmParams:
        return _EmParams(self.max_iters, self.ll_rel_tol, self.cov_reg, self.seed)


@dataclasses.dataclass
class Gmm:
    """Gmm4 (gmm.hpp:15-34) generalised to D in {3, 4}: packed covariances in
    the packed10 order (0,0),(1,0),(1,1),(2,0),... (packed10.hpp:11-14)."""
    weights: np.ndarray      # (M,)
    means: np.ndarray        # (M, D)
    covariances: np.ndarray  # (M, D(D+1)/2)

    @property
    def dim(self) -> int:
        return int(self.means.shape[1])

    def components(self) -> int:
        return int(self.weights.shape[0])

    def covariance(self, b: int) -> np.ndarray:
        return unpack_symmetric(self.covariances[b], self.dim)

    def memory_footprint(self) -> int:
        """gmm.hpp:38-40: 4 bytes per float, 1 + D + D(D+1)/2 per component."""
        d = self.dim
        return 4 * self.components() * (1 + d + d * (d + 1) // 2)


def packed_index(d: int):
    rows, cols = [], []
    for i in range(d):
        for j in range(i + 1):
            rows.append(i)
            cols.append(j)
    return np.array(rows), np.array(cols)


def unpack_symmetric(p: np.ndarray, d: int) -> np.ndarray:
    r, c = packed_index(d)
    m = np.zeros((d, d))
    m[r, c] = p
    m[c, r] = p
    return m


def pack_symmetric(m: np.ndarray) -> np.ndarray:
    r, c = packed_index(m.shape[0])
    return m[r, c].copy()


@dataclasses.dataclass
class FitResult:
    """sogmm.hpp:65-71 (gbms_components -> k_init) plus the ll trace."""
    model: Gmm
    em_iterations: int
    final_log_likelihood: float
    removed_components: int
    k_init: int
    converged: bool
    ll_trace: np.ndarray
    units: float                  # sum over E steps of N * K_t
    ms_layout: float = 0.0
    ms_kinit: float = 0.0
    ms_mstep0: float = 0.0
    ms_em: float = 0.0
    ms_total: float = 0.0
    ms_estep: float = 0.0
    launches: int = 0
    labels: Optional[np.ndarray] = None
    centers: Optional[np.ndarray] = None
    gbms_components: int = 0      # fit(): GBMS's component estimate
    units_evaluated: float = 0.0  # pairs the E step evaluated (pruned E step: the
                                  # ones whose FP32 density can be non-zero)


@dataclasses.dataclass
class CholeskyCache:
    """gmm.hpp:44-48."""
    lower: np.ndarray       # (M, D, D)
    precision: np.ndarray   # (M, D, D) = L^-1
    log_det_terms: np.ndarray  # (M,) = sum ln diag P


class VGroup:
    """In-process group of `world` virtual ranks on one device
    (gmmb_vgroup): the sharded fit's validation mode, the collectives being
    fixed-order device reductions instead of NCCL (include/gmmb.h)."""

    def __init__(self, world: int, device: int = 0):
        h = ctypes.c_void_p()
        _check(load().gmmb_vgroup_create(device, world, ctypes.byref(h)))
        self._h, self.world, self.device = h, world, device

    def close(self) -> None:
        if getattr(self, "_h", None):
            load().gmmb_vgroup_release(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One CUDA device + stream + reusable device buffers (gmmb_ctx)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None, vgroup: Optional[VGroup] = None):
        lib = load()
        h = ctypes.c_void_p()
        if vgroup is not None:
            _check(lib.gmmb_ctx_create_virtual(vgroup._h, rank, ctypes.byref(h)))
            world, device = vgroup.world, vgroup.device
        elif world > 1:
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("sharded context needs the 128-byte NCCL id")
            _check(lib.gmmb_ctx_create_sharded(device, rank, world, nccl_id, ctypes.byref(h)))
        else:
            _check(lib.gmmb_ctx_create(device, ctypes.byref(h)))
        self._h = h
        self.rank, self.world, self.device = rank, world, device

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(load().gmmb_nccl_unique_id(buf))
        return buf.raw

    def close(self) -> None:
        if getattr(self, "_h", None):
            load().gmmb_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def device_info(self) -> tuple[int, int, int]:
        a, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(load().gmmb_device_info(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    @property
    def handle(self):
        return self._h

    def set_timing(self, per_kernel_events: bool) -> None:
        """EM loop mode: False (default) = one CUDA graph per fit (conditional
        WHILE node, no host round trip); True = chunked launches with CUDA
        events around every fused E kernel (FitResult.ms_estep)."""
        _check(load().gmmb_ctx_set_timing(self._h, 1 if per_kernel_events else 0))

    def set_estep_mode(self, dense: bool) -> None:
        """E-step kernels: False (default) = exact-zero-pruned (skips the
        (tile, component) pairs whose FP32 densities are provably exactly 0),
        True = dense (every pair). Same results up to FP32 summation order."""
        _check(load().gmmb_ctx_set_estep_mode(self._h, 1 if dense else 0))

    def ffma_peak(self, ms_target: float = 50.0) -> tuple[float, float]:
        """Measured FP32 FFMA TFLOP/s on this device (and the ms it took)."""
        tf, ms = ctypes.c_double(), ctypes.c_double()
        _check(load().gmmb_ffma_peak(self._h, ms_target, ctypes.byref(tf), ctypes.byref(ms)))
        return tf.value, ms.value

    # -- device-resident fits (bench "value": inputs already in HBM) ------
    def upload(self, points, offset: int = 0, n_global: int = 0) -> None:
        p, n, d = _points(points)
        self._n, self._d = n, d
        _check(load().gmmb_upload(self._h, _ptr(p), n, d, offset, n_global))

    def ingest_images(self, depth, intensity, intrinsics, intensity_max: float = 255.0,
                      depth_scale: float = 1000.0, factor: int = 1, want_points: bool = False):
        """Device ingest (ingest.cpp:27-75): decimate + image_pair_to_cloud on
        the GPU; the cloud becomes this context's resident cloud. intrinsics =
        (fx, fy, cx, cy) of the full-resolution image. Returns N, or (N,
        (N, 4) points) with want_points."""
        dep = np.ascontiguousarray(depth, dtype=np.uint16)
        inten = np.ascontiguousarray(intensity, dtype=np.uint16)
        if dep.shape != inten.shape or dep.ndim != 2:
            raise ValueError("depth and intensity dimensions differ")
        h, w = dep.shape
        fx, fy, cx, cy = (float(v) for v in intrinsics)
        cap = (w // max(factor, 1)) * (h // max(factor, 1))
        buf = np.zeros(4 * max(cap, 1)) if want_points else None
        n = ctypes.c_int64()
        U16 = ctypes.POINTER(ctypes.c_uint16)
        _check(load().gmmb_ingest_images(self._h, dep.ctypes.data_as(U16), inten.ctypes.data_as(U16),
                                         w, h, intensity_max, fx, fy, cx, cy, depth_scale, factor,
                                         _ptr(buf), ctypes.byref(n)))
        self._n, self._d = n.value, 4
        if not want_points:
            return n.value
        return n.value, buf[:4 * n.value].reshape(4, n.value).T.copy()

    def fit_k_resident(self, k: int, em: EmParams = EmParams(),
                       want_labels: bool = False) -> FitResult:
        n, d = self._n, self._d
        kk = max(1, min(k, 1 << 30))
        out = _alloc_model(kk, d)
        ll = np.zeros(max(em.max_iters, 1))
        st = _FitStats()
        lab = np.zeros(n, np.int32) if want_labels else None
        cen = np.zeros(kk, np.int64) if want_labels else None
        _check(load().gmmb_fit_k_resident(self._h, k, ctypes.byref(em._c()), _ptr(out[0]),
                                          _ptr(out[1]), _ptr(out[2]), _ptr(ll),
                                          ctypes.byref(st), _ptr(lab, _I32), _ptr(cen, _I64)))
        return _result(out, ll, st, lab, cen)


def _alloc_model(m: int, d: int):
    return (np.zeros(m), np.zeros((m, d)), np.zeros((m, d * (d + 1) // 2)))


def _result(out, ll, st: _FitStats, lab=None, cen=None) -> FitResult:
    k = st.k_out
    model = Gmm(out[0][:k].copy(), out[1][:k].copy(), out[2][:k].copy())
    if cen is not None:
        cen = cen[:st.k_init].copy()
    return FitResult(model, st.em_iterations, st.final_log_likelihood,
                     st.removed_components, st.k_init, bool(st.converged),
                     ll[:st.em_iterations].copy(), st.units, st.ms_layout,
                     st.ms_kinit, st.ms_mstep0, st.ms_em, st.ms_total, st.ms_estep,
                     st.launches, lab, cen, units_evaluated=st.units_evaluated)


_default_ctx: Optional[Context] = None


def _ctx(ctx: Optional[Context]) -> Context:
    global _default_ctx
    if ctx is not None:
        return ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def fit_k(points, k: int, em: EmParams = EmParams(), ctx: Optional[Context] = None,
          want_labels: bool = False) -> FitResult:
    """fit (sogmm.cpp:465-510) with K given: kinit -> m_step -> EM."""
    c = _ctx(ctx)
    p, n, d = _points(points)
    kk = max(1, min(int(k), n if c.world == 1 else int(k)))
    out = _alloc_model(kk, d)
    ll = np.zeros(max(em.max_iters, 1))
    st = _FitStats()
    lab = np.zeros(n, np.int32) if want_labels else None
    cen = np.zeros(kk, np.int64) if want_labels else None
    _check(load().gmmb_fit_k(c.handle, _ptr(p), n, d, int(k), ctypes.byref(em._c()),
                             _ptr(out[0]), _ptr(out[1]), _ptr(out[2]), _ptr(ll),
                             ctypes.byref(st), _ptr(lab, _I32), _ptr(cen, _I64)))
    return _result(out, ll, st, lab, cen)


def shard_bounds(n: int, world: int) -> list:
    """Contiguous shards [lo, hi) of n points over `world` ranks (the first
    n % world ranks take one more point)."""
    q, r = divmod(n, world)
    out, lo = [], 0
    for i in range(world):
        hi = lo + q + (1 if i < r else 0)
        out.append((lo, hi))
        lo = hi
    return out


def fit_k_vsharded(points, k: int, em: EmParams = EmParams(), world: int = 2,
                   device: int = 0, want_labels: bool = False, fit_from: Optional[Gmm] = None,
                   contexts: Optional[list] = None) -> list:
    """The point-sharded fit run as `world` virtual ranks
    on one device: contiguous shards, one host thread per rank calling
    gmmb_fit_k (or gmmb_fit_from with `fit_from`) on its own context; the
    statistics all-reduce and k-means++ exchange are fixed-order device
    reductions. Returns the per-rank FitResults (identical models; labels
    per shard). `contexts` (from vshard_contexts) reuses contexts."""
    import threading
    p, n, d = _points(points)
    own = contexts is None
    grp = None
    if own:
        grp = VGroup(world, device)
        contexts = [Context(vgroup=grp, rank=r) for r in range(world)]
    world = len(contexts)
    bounds = shard_bounds(n, world)
    res: list = [None] * world
    err: list = [None] * world

    def run(r):
        lo, hi = bounds[r]
        try:
            if fit_from is not None:
                res[r] = globals()["fit_from"](p[lo:hi], fit_from, em, ctx=contexts[r])
            else:
                res[r] = fit_k(p[lo:hi], k, em, ctx=contexts[r], want_labels=want_labels)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if own:
        for c in contexts:
            c.close()
        grp.close()
    for e in err:
        if e is not None:
            raise e
    return res


def vshard_contexts(world: int, device: int = 0) -> list:
    """`world` virtual-rank contexts sharing one group (for repeated
    fit_k_vsharded calls); close them with Context.close()."""
    grp = VGroup(world, device)
    ctxs = [Context(vgroup=grp, rank=r) for r in range(world)]
    grp.close()  # the contexts keep the group alive
    return ctxs


def fit_k_batch(frames, k: int, em: EmParams = EmParams(), seeds=None,
                ctx: Optional[Context] = None) -> list:
    """A batch of independent frames (BASELINE cfg3), each fitted exactly as
    fit_k(frame, k, em with seed seeds[f]); frame f+1 is copied to the device
    while frame f fits (pinned host frames overlap fully). Frames must share
    D; each needs k <= its N."""
    c = _ctx(ctx)
    ps = [_points(f) for f in frames]
    F = len(ps)
    if F == 0:
        raise ValueError("empty frame batch")
    d = ps[0][2]
    if any(q[2] != d for q in ps):
        raise ValueError("frames must share the dimension")
    kk = max(1, int(k))
    np_ = d * (d + 1) // 2
    w = np.zeros((F, kk))
    mu = np.zeros((F, kk, d))
    cov = np.zeros((F, kk, np_))
    stats = (_FitStats * F)()
    ptrs = (_D * F)(*[_ptr(q[0]) for q in ps])
    ns = np.array([q[1] for q in ps], dtype=np.int64)
    sd = None if seeds is None else np.ascontiguousarray(seeds, dtype=np.uint64)
    _check(load().gmmb_fit_k_batch(c.handle, F, ptrs, _ptr(ns, _I64), d, kk,
                                   ctypes.byref(em._c()),
                                   None if sd is None else sd.ctypes.data_as(
                                       ctypes.POINTER(ctypes.c_uint64)),
                                   _ptr(w), _ptr(mu), _ptr(cov), stats))
    out = []
    for f in range(F):
        st = stats[f]
        m = st.k_out
        model = Gmm(w[f, :m].copy(), mu[f, :m].copy(), cov[f, :m].copy())
        out.append(FitResult(model, st.em_iterations, st.final_log_likelihood,
                             st.removed_components, st.k_init, bool(st.converged),
                             np.zeros(0), st.units, st.ms_layout, st.ms_kinit, st.ms_mstep0,
                             st.ms_em, st.ms_total, st.ms_estep, st.launches,
                             units_evaluated=st.units_evaluated))
    return out


@dataclasses.dataclass
class GbmsParams:
    """GbmsParams (sogmm.hpp:12-22)."""
    bandwidth: float = 0.015
    max_iters: int = 100
    convergence_tol: float = 1e-5
    merge_radius: float = -1.0

    def _c(self):
        return _GbmsParams(self.bandwidth, self.max_iters, self.convergence_tol, self.merge_radius)


def gbms(points, params: GbmsParams = GbmsParams(), ctx: Optional[Context] = None):
    """gbms_estimate_components (sogmm.cpp:22-195): (components, iterations,
    modes (components, 4) in the original coordinates)."""
    c = _ctx(ctx)
    p, n, d = _points(points)
    comp, it = ctypes.c_int(), ctypes.c_int()
    cap = 8192
    while True:
        modes = np.zeros((cap, 4))
        _check(load().gmmb_gbms(c.handle, _ptr(p), n, d, ctypes.byref(params._c()),
                                ctypes.byref(comp), ctypes.byref(it), _ptr(modes), cap))
        if comp.value <= cap:
            return comp.value, it.value, modes[:comp.value].copy()
        cap = comp.value


def fit(points, params: GbmsParams = GbmsParams(), em: EmParams = EmParams(),
        ctx: Optional[Context] = None) -> FitResult:
    """fit (sogmm.cpp:465-510): GBMS decides K, then k-means++ -> m_step -> EM."""
    c = _ctx(ctx)
    p, n, d = _points(points)
    cap = max(n, 1)   # K <= N (sogmm.cpp:477)
    out = _alloc_model(cap, d)
    ll = np.zeros(max(em.max_iters, 1))
    st = _FitStats()
    comp = ctypes.c_int()
    _check(load().gmmb_fit(c.handle, _ptr(p), n, d, ctypes.byref(params._c()),
                           ctypes.byref(em._c()), cap, _ptr(out[0]), _ptr(out[1]), _ptr(out[2]),
                           _ptr(ll), ctypes.byref(st), ctypes.byref(comp)))
    r = _result(out, ll, st, None, None)
    r.gbms_components = comp.value
    return r


def _model_arrays(model: Gmm, d: int):
    w = np.ascontiguousarray(model.weights, dtype=np.float64)
    mu = np.ascontiguousarray(model.means, dtype=np.float64)
    cov = np.ascontiguousarray(model.covariances, dtype=np.float64)
    m = w.shape[0]
    if mu.shape != (m, d) or cov.shape != (m, d * (d + 1) // 2):
        raise ValueError("model field sizes disagree")
    return w, mu, cov, m


def fit_from(points, model: Gmm, em: EmParams = EmParams(),
             ctx: Optional[Context] = None) -> FitResult:
    """EM loop (sogmm.cpp:484-509) from a given initial model."""
    c = _ctx(ctx)
    p, n, d = _points(points)
    w, mu, cov, m = _model_arrays(model, d)
    out = _alloc_model(m, d)
    ll = np.zeros(max(em.max_iters, 1))
    st = _FitStats()
    _check(load().gmmb_fit_from(c.handle, _ptr(p), n, d, m, _ptr(w), _ptr(mu), _ptr(cov),
                                ctypes.byref(em._c()), _ptr(out[0]), _ptr(out[1]),
                                _ptr(out[2]), _ptr(ll), ctypes.byref(st)))
    return _result(out, ll, st)


def kinit(points, k: int, seed: int = 0, ctx: Optional[Context] = None):
    """sogmm.cpp:197-337. Returns (labels[N] int32, centers[k] int64); the
    reference's Responsibilities is the one-hot of labels (0 / -inf)."""
    c = _ctx(ctx)
    p, n, d = _points(points)
    lab = np.zeros(n, np.int32)
    cen = np.zeros(max(int(k), 1), np.int64)
    _check(load().gmmb_kinit(c.handle, _ptr(p), n, d, int(k), seed, _ptr(lab, _I32),
                             _ptr(cen, _I64)))
    return lab, cen


def e_step(points, model: Gmm, want_log_gamma: bool = True,
           ctx: Optional[Context] = None):
    """sogmm.cpp:387-395: (log_gamma (N, M) or None, log-likelihood)."""
    c = _ctx(ctx)
    p, n, d = _points(points)
    w, mu, cov, m = _model_arrays(model, d)
    ll = ctypes.c_double()
    lg = np.zeros((n, m), order="F") if want_log_gamma else None
    _check(load().gmmb_e_step(c.handle, _ptr(p), n, d, m, _ptr(w), _ptr(mu), _ptr(cov),
                              ctypes.byref(ll), _ptr(lg)))
    return lg, ll.value


def score(points, model: Gmm, ctx: Optional[Context] = None, per_point: bool = False):
    """inference.cpp:141-172: average log-likelihood of the cloud (and, with
    per_point, each point's log-sum-exp)."""
    c = _ctx(ctx)
    p, n, d = _points(points)
    w, mu, cov, m = _model_arrays(model, d)
    avg = ctypes.c_double()
    pp = np.zeros(n) if per_point else None
    _check(load().gmmb_score(c.handle, _ptr(p), n, d, m, _ptr(w), _ptr(mu), _ptr(cov),
                             ctypes.byref(avg), _ptr(pp)))
    return (avg.value, pp) if per_point else avg.value


def joint_dist_sample(model: Gmm, n: int, seed: int = 0, ctx: Optional[Context] = None):
    """inference.cpp:17-54: (n, D) draws; draw i depends only on (seed, i)."""
    c = _ctx(ctx)
    d = np.asarray(model.means).shape[1]
    w, mu, cov, m = _model_arrays(model, d)
    out = np.zeros((n, d), order="F")
    _check(load().gmmb_sample(c.handle, d, m, _ptr(w), _ptr(mu), _ptr(cov), n, seed, _ptr(out)))
    return out


def color_conditional(model: Gmm, locs, clamp: bool = True, ctx: Optional[Context] = None):
    """inference.cpp:56-139: (expected intensity, variance) at (n, 3) locations
    under a 4D model."""
    c = _ctx(ctx)
    w, mu, cov, m = _model_arrays(model, 4)
    loc = np.asfortranarray(np.asarray(locs, dtype=np.float64)[:, :3])
    n = loc.shape[0]
    e, v = np.zeros(n), np.zeros(n)
    _check(load().gmmb_color_conditional(c.handle, m, _ptr(w), _ptr(mu), _ptr(cov), _ptr(loc), n,
                                         1 if clamp else 0, _ptr(e), _ptr(v)))
    return e, v


def m_step(points, log_gamma, cov_reg: float = 1e-6, ctx: Optional[Context] = None):
    """sogmm.cpp:459-463: returns (Gmm, removed)."""
    c = _ctx(ctx)
    p, n, d = _points(points)
    lg = np.asfortranarray(np.asarray(log_gamma, dtype=np.float64))
    if lg.ndim != 2 or lg.shape[0] != n:
        raise ValueError("responsibility rows != point count")
    m = lg.shape[1]
    out = _alloc_model(m, d)
    mo, rm = ctypes.c_int(), ctypes.c_int()
    _check(load().gmmb_m_step(c.handle, _ptr(p), n, d, _ptr(lg), m, cov_reg, _ptr(out[0]),
                              _ptr(out[1]), _ptr(out[2]), ctypes.byref(mo), ctypes.byref(rm)))
    k = mo.value
    return Gmm(out[0][:k].copy(), out[1][:k].copy(), out[2][:k].copy()), rm.value


def em_step(points, model: Gmm, cov_reg: float = 1e-6, ctx: Optional[Context] = None):
    """One production EM iteration (fused E + statistics + M) from `model`:
    returns (ll of the E step, next model, removed)."""
    c = _ctx(ctx)
    p, n, d = _points(points)
    w, mu, cov, m = _model_arrays(model, d)
    out = _alloc_model(m, d)
    ll = ctypes.c_double()
    mo, rm = ctypes.c_int(), ctypes.c_int()
    _check(load().gmmb_em_step(c.handle, _ptr(p), n, d, m, _ptr(w), _ptr(mu), _ptr(cov),
                               cov_reg, ctypes.byref(ll), _ptr(out[0]), _ptr(out[1]),
                               _ptr(out[2]), ctypes.byref(mo), ctypes.byref(rm)))
    k = mo.value
    return ll.value, Gmm(out[0][:k].copy(), out[1][:k].copy(), out[2][:k].copy()), rm.value


def cholesky_cache(model: Gmm, ctx: Optional[Context] = None) -> CholeskyCache:
    """gmm.cpp:33-48 on the device (FP64)."""
    c = _ctx(ctx)
    d = model.dim
    cov = np.ascontiguousarray(model.covariances, dtype=np.float64)
    m = cov.shape[0]
    lo = np.zeros((m, d, d))
    pr = np.zeros((m, d, d))
    ld = np.zeros(m)
    _check(load().gmmb_cholesky_cache(c.handle, d, m, _ptr(cov), _ptr(lo), _ptr(pr), _ptr(ld)))
    return CholeskyCache(lo, pr, ld)


# ---- synthetic inputs (host C++ in libgmmb.so; no GPU needed) -----------
def synthetic_frame_cloud(width: int = 640, height: int = 480,
                          depth_scale: float = 1000.0) -> np.ndarray:
    """make_synthetic_frame + image_pair_to_cloud -> (N, 4)."""
    buf = np.zeros(width * height * 4)
    n = ctypes.c_int64()
    _check(load().gmmb_synthetic_frame_cloud(width, height, depth_scale, _ptr(buf),
                                             ctypes.byref(n)))
    nn = n.value
    return buf[:4 * nn].reshape(4, nn).T.copy()


class GmmFormatError(IoError):
    """gmm_io.hpp:10-13 — wrong magic or malformed structure."""


def _io_check(code: int) -> None:
    if code == 0:
        return
    msg = load().gmmb_io_last_error().decode(errors="replace")
    if code == 2:
        raise ValueError(msg)
    if code == 3:
        raise NumericalError(msg)
    if "magic" in msg or "malformed" in msg or "missing" in msg or "truncated" in msg \
            or "inconsistent" in msg or "bad row" in msg or "zero components" in msg:
        raise GmmFormatError(msg)
    raise IoError(msg)


def save_gmm(model: Gmm, path: str, json: bool = False) -> None:
    """gmm_io.cpp:71-85 (binary SGMM4D01, f32) / :120-141 (JSON mirror)."""
    w, mu, cov, m = _model_arrays(model, 4)
    fn = load().gmmb_save_model_json if json else load().gmmb_save_model
    _io_check(fn(path.encode(), m, _ptr(w), _ptr(mu), _ptr(cov)))


def load_gmm(path: str, json: bool = False) -> Gmm:
    """gmm_io.cpp:87-118 / :143-177 with finalize_loaded's checks."""
    fn = load().gmmb_load_model_json if json else load().gmmb_load_model
    m = ctypes.c_int()
    cap = 1
    while True:
        w, mu, cov = np.zeros(cap), np.zeros((cap, 4)), np.zeros((cap, 10))
        code = fn(path.encode(), cap, _ptr(w), _ptr(mu), _ptr(cov), ctypes.byref(m))
        if code == 2 and m.value > cap:
            cap = m.value
            continue
        _io_check(code)
        k = m.value
        return Gmm(w[:k].copy(), mu[:k].copy(), cov[:k].copy())


def synthetic_frame_images(width: int = 640, height: int = 480, depth_scale: float = 1000.0):
    """make_synthetic_frame (synthetic.cpp:9-72): (depth uint16 (H, W),
    intensity uint16 (H, W), (fx, fy, cx, cy))."""
    dep = np.zeros((height, width), np.uint16)
    inten = np.zeros((height, width), np.uint16)
    intr = np.zeros(4)
    U16 = ctypes.POINTER(ctypes.c_uint16)
    _check(load().gmmb_synthetic_frame_images(width, height, depth_scale, dep.ctypes.data_as(U16),
                                              inten.ctypes.data_as(U16), _ptr(intr)))
    return dep, inten, tuple(intr)


def structured_scene(n: int, seed: int = 0, noise_sigma: float = 0.005) -> np.ndarray:
    buf = np.zeros(4 * n)
    _check(load().gmmb_structured_scene(n, seed, noise_sigma, _ptr(buf)))
    return buf.reshape(4, n).T.copy()


def blob_cloud(centers, sigma: float, per_blob: int, seed: int = 0) -> np.ndarray:
    c = np.ascontiguousarray(centers, dtype=np.float64)
    k = c.shape[0]
    buf = np.zeros(4 * k * per_blob)
    _check(load().gmmb_blob_cloud(_ptr(c), k, sigma, per_blob, seed, _ptr(buf)))
    return buf.reshape(4, k * per_blob).T.copy()


def shard_key_tail(heads: np.ndarray, rank: int) -> np.ndarray:
    """The 3 doubles following shard `rank`'s last x in the global
    column-major buffer (sharded k-means++ keys, sogmm.cpp:210-213).
    heads: (world, 8) = first 3 x, first 3 y, point count, pad per shard."""
    h = np.ascontiguousarray(heads, dtype=np.float64)
    out = np.zeros(3)
    _check(load().gmmb_shard_key_tail(_ptr(h), h.shape[0], rank, _ptr(out)))
    return out


def jitter_cloud(points: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    p = np.asfortranarray(np.array(points, dtype=np.float64))
    _check(load().gmmb_jitter_cloud(_ptr(p), p.shape[0], sigma, seed))
    return np.ascontiguousarray(p)
