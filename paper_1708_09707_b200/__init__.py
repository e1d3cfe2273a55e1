"""paper_1708_09707_b200 -- B200-native H-matrix engine (setup + H-MVP on sm_100a).

Python mirror of the reference library's public API (proj/include/hmat/hmatrix.hpp,
solver.hpp, morton.hpp, aca.hpp) over the C ABI in include/hmat_b200.h, which is
implemented by ``libhmat_b200.so`` (hand-written CUDA for sm_100a, built in-tree by
``make -C paper_1708_09707_b200``).  There is no CPU fallback: importing this module
fails loudly when the shared library is missing, and every call fails with
``HmError`` when no CUDA device is present.

    import numpy as np
    import paper_1708_09707_b200 as hm
    pts = hm.inputs.uniform_points(1 << 14, 2)          # (d, n) SoA, like PointSet.coords
    h = hm.setup(pts, hm.KernelFunction("gaussian"), hm.HmatrixConfig(c_leaf=64))
    z = hm.mvp(h, x)                                      # original ordering in and out
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import inputs  # noqa: F401  (synthetic inputs, reference conventions)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhmat_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {_HERE}` (no CPU fallback exists)")
_lib = C.CDLL(LIB_PATH)

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_d = C.c_double

HM_OK, HM_EINVAL, HM_ERANGE, HM_ENOMEM, HM_ECUDA, HM_ENCCL, HM_ENONFINITE, HM_ELOGIC, HM_EIO = range(9)
_STATUS_NAMES = ["HM_OK", "HM_EINVAL", "HM_ERANGE", "HM_ENOMEM", "HM_ECUDA", "HM_ENCCL", "HM_ENONFINITE",
                 "HM_ELOGIC", "HM_EIO"]


class HmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS_NAMES[status] if 0 <= status < len(_STATUS_NAMES) else status}: {msg}")
        self.status = status


class InvalidArgument(HmError, ValueError):
    """std::invalid_argument in the reference."""


class OutOfRange(HmError, IndexError):
    """std::out_of_range in the reference."""


class NonFinite(HmError):
    """std::runtime_error from cg_solve on non-finite values (solver.cpp:51-54)."""


class _Config(C.Structure):
    _fields_ = [("eta", _d), ("c_leaf", _i64), ("k", _i64), ("bs_aca", _i64), ("bs_dense", _i64),
                ("precompute_aca", _i32), ("has_epsilon", _i32), ("epsilon", _d), ("adm_mode", _i32),
                ("near_stored", _i32), ("rank", _i32), ("world", _i32), ("device", _i32),
                ("aca_chunk_rows", _i64)]


class _Timings(C.Structure):
    _fields_ = [("setup_ms", _d), ("morton_ms", _d), ("tree_ms", _d), ("aca_ms", _d), ("near_ms", _d),
                ("mvp_ms", _d), ("mvp_dense_ms", _d), ("mvp_aca_ms", _d)]


class _Stats(C.Structure):
    _fields_ = [("n_dense", _i64), ("n_aca", _i64), ("S_d", _d), ("S_l", _d), ("sum_m_adm", _d),
                ("sum_n_adm", _d), ("S_lm", _d), ("S_ln", _d), ("S_d_own", _d), ("aca_rejections", _i64), ("dmax_leaf", _i32), ("row_begin", _i64),
                ("row_end", _i64), ("device_bytes", _d),
                ("S_d_stored", _d), ("near_sym", _i32), ("n_aca_batches", _i64), ("n_aca_chunks", _i64),
                ("aca_rejected_entries", _i64), ("S_chain", _d), ("near_pairs", _i64), ("near_sym_rc", _i32)]


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("hm_last_error", C.c_char_p, [])
_sig("hm_config_default", None, [C.POINTER(_Config)])
_sig("hm_device_count", C.c_int, [])
_sig("hm_setup", C.c_int, [_p, _i64, _i32, _i32, _d, C.POINTER(_Config), C.POINTER(_p)])
_sig("hm_setup_device", C.c_int, [_p, _i64, _i32, _i32, _d, C.POINTER(_Config), C.POINTER(_p)])
_sig("hm_destroy", None, [_p])
_sig("hm_mvp", C.c_int, [_p, _p, _p, C.POINTER(_Timings)])
_sig("hm_mvp_device", C.c_int, [_p, _p, _p, _p])
_sig("hm_mvp_local", C.c_int, [_p, _p, _p])
_sig("hm_nccl_unique_id", C.c_int, [_p])
_sig("hm_attach_nccl", C.c_int, [_p, _p])
_sig("hm_cg_solve", C.c_int, [_p, _p, _d, _d, _i64, _p, C.POINTER(_i64), C.POINTER(_d)])
_sig("hm_relative_error", C.c_int, [_p, _p, C.POINTER(_d)])
_sig("hm_dense_mvp", C.c_int, [_p, _p, _p])
_sig("hm_get_stats", C.c_int, [_p, C.POINTER(_Stats)])
_sig("hm_get_timings", C.c_int, [_p, C.POINTER(_Timings)])
_sig("hm_get_points", C.c_int, [_p, _p, _p])
_sig("hm_get_codes", C.c_int, [_p, _p])
_sig("hm_get_leaves", C.c_int, [_p, _i32, _p, _p])
_sig("hm_get_aca", C.c_int, [_p, _p, _p, _p, _p, _p])
_sig("hm_morton_codes", C.c_int, [_p, _i64, _i32, _p])
_sig("hm_morton_order", C.c_int, [_p, _i64, _i32, _p, _p, _p])
_sig("hm_aca_dense", C.c_int, [_i64, _p, _p, _i64, _i32, _d, _d, _p, _p, _p, _p, _p])
_sig("hm_eval_kernel", C.c_int, [_i32, _d, _i32, _i64, _p, _p, _p])
_sig("hm_exp_port_host", None, [_i64, _p, _p])
_sig("hm_exp_port_device", C.c_int, [_i64, _p, _p])
_sig("hm_profile_begin", C.c_int, [_p])
_sig("hm_profile_end", C.c_int, [_p, _p, _p])
_sig("hm_log_port_host", None, [_i64, _p, _p])
_sig("hm_log_port_device", C.c_int, [_i64, _p, _p])
_sig("hm_mvp_multi", C.c_int, [_p, _p, _p, _i64, _i32])
_sig("hm_dump_leaves_csv", C.c_int, [_p, C.c_char_p])
_sig("hm_mvp_multi_device", C.c_int, [_p, _p, _p, _i64, _i32, _p])
_sig("hm_cg_solve_multi", C.c_int, [_p, _p, _i64, _d, _d, _i64, _i32, _p, _p, _p])

HM_MULTI_EXACT = 0
HM_MULTI_DMMA = 1

EXPORTED_SYMBOLS = [
    "hm_last_error", "hm_config_default", "hm_device_count", "hm_setup", "hm_setup_device", "hm_destroy",
    "hm_mvp", "hm_mvp_device", "hm_mvp_local", "hm_nccl_unique_id", "hm_attach_nccl", "hm_cg_solve", "hm_relative_error",
    "hm_dense_mvp", "hm_get_stats", "hm_get_timings", "hm_get_points", "hm_get_codes", "hm_get_leaves",
    "hm_get_aca", "hm_morton_codes", "hm_morton_order", "hm_aca_dense", "hm_eval_kernel", "hm_exp_port_host",
    "hm_exp_port_device", "hm_log_port_host", "hm_log_port_device", "hm_profile_begin", "hm_profile_end",
    "hm_mvp_multi", "hm_mvp_multi_device", "hm_cg_solve_multi", "hm_dump_leaves_csv",
]

KERNEL_IDS = ["gather_x", "lowrank_t", "rows", "scatter_z", "aca", "rows_far", "allgather", "near_pairs"]


def _check(rc: int) -> None:
    if rc != HM_OK:
        msg = _lib.hm_last_error().decode()
        cls = {HM_EINVAL: InvalidArgument, HM_ERANGE: OutOfRange, HM_ENONFINITE: NonFinite}.get(rc, HmError)
        raise cls(rc, msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def device_count() -> int:
    return int(_lib.hm_device_count())


# ----------------------------------------------------------------------------- API types
@dataclass
class KernelFunction:
    """KernelFunction (core.hpp:35-40): 'gaussian' exp(-r^2) or 'matern' (order beta - d/2 = 1)."""
    kind: str = "gaussian"
    matern_beta: float = 0.0

    @property
    def code(self) -> int:
        k = self.kind.lower()
        if k in ("gaussian", "gauss"):
            return 0
        if k == "matern":
            return 1
        raise ValueError(f"unknown kernel kind {self.kind!r}")


@dataclass
class HmatrixConfig:
    """HmatrixConfig (hmatrix.hpp:15-34) plus B200 placement knobs."""
    eta: float = 1.5
    c_leaf: int = 256
    k: int = 16
    bs_aca: int = 1 << 20
    bs_dense: int = 1 << 22
    precompute_aca: bool = False
    epsilon: Optional[float] = None
    force_dense: bool = False
    force_admissible: bool = False  # test-only AdmissibilityMode::ForceAdmissible (tree.hpp:64-68)
    near_stored: bool = False       # keep the dense leaves in HBM (B200 extension)
    rank: int = 0
    world: int = 1
    device: int = 0
    aca_chunk_rows: int = 0

    @staticmethod
    def large_scale() -> "HmatrixConfig":
        return HmatrixConfig(c_leaf=2048, bs_aca=1 << 25, bs_dense=1 << 27)

    def _c(self) -> _Config:
        c = _Config()
        _lib.hm_config_default(C.byref(c))
        c.eta, c.c_leaf, c.k = float(self.eta), int(self.c_leaf), int(self.k)
        c.bs_aca, c.bs_dense = int(self.bs_aca), int(self.bs_dense)
        c.precompute_aca = int(bool(self.precompute_aca))
        c.has_epsilon = int(self.epsilon is not None)
        c.epsilon = float(self.epsilon or 0.0)
        c.adm_mode = 1 if self.force_dense else (2 if self.force_admissible else 0)
        c.near_stored = int(bool(self.near_stored))
        c.rank, c.world, c.device = int(self.rank), int(self.world), int(self.device)
        c.aca_chunk_rows = int(self.aca_chunk_rows)
        return c


@dataclass
class MvpTimings:
    """hmat::MvpTimings (hmatrix.hpp:50-54): dense = near-field phase, aca = far-field
    phase (incl. the recompute-mode factorisation), total = the whole call."""
    dense_ms: float = 0.0
    aca_ms: float = 0.0
    total_ms: float = 0.0


@dataclass
class Leaves:
    rows: np.ndarray   # (L, 4) int64 row.lower, row.upper, col.lower, col.upper
    boxes: Optional[np.ndarray] = None  # (L, 4, d): row a, row b, col a, col b


@dataclass
class SolveConfig:
    sigma2: float = 0.0
    tol: float = 1e-8
    max_iter: int = 500


@dataclass
class SolveResult:
    x: np.ndarray = field(default_factory=lambda: np.zeros(0))
    iterations: int = 0
    relative_residual: float = 0.0


class HMatrix:
    """Device-resident H-matrix (HMatrix, hmatrix.hpp:36-44)."""

    def __init__(self, handle, n: int, d: int, kernel: KernelFunction, config: HmatrixConfig):
        self._h = handle
        self.n, self.d = n, d
        self.kernel = kernel
        self.config = config

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.hm_destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    # --- products
    def mvp(self, x, timings: Optional[MvpTimings] = None, out: Optional[np.ndarray] = None) -> np.ndarray:
        """z = H x (original ordering).  out: optional preallocated float64 result buffer."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise InvalidArgument(HM_EINVAL, "mvp: vector length mismatch")
        if out is not None:
            if out.shape != (self.n,) or out.dtype != np.float64 or not out.flags["C_CONTIGUOUS"]:
                raise InvalidArgument(HM_EINVAL, "mvp: out must be a contiguous float64 vector of length n")
            z = out
        else:
            z = np.empty(self.n)
        t = _Timings()
        _check(_lib.hm_mvp(self._h, _ptr(x), _ptr(z), C.byref(t)))
        if timings is not None:
            timings.total_ms = t.mvp_ms
            timings.dense_ms = t.mvp_dense_ms
            timings.aca_ms = t.mvp_aca_ms
        return z

    def mvp_multi(self, X, dmma: bool = False) -> np.ndarray:
        """Z[:, r] = H X[:, r] for every column of X (n x nrhs), one operator pass per 16
        columns.  dmma=False: each column bitwise equal to mvp(X[:, r]); dmma=True: the
        recompute-mode near field on the FP64 tensor cores (nrhs 8 or 16 per pass)."""
        X = np.asarray(X, dtype=np.float64)
        if X.ndim != 2 or X.shape[0] != self.n:
            raise InvalidArgument(HM_EINVAL, "mvp_multi: X must be n x nrhs")
        Xc = np.ascontiguousarray(X.T)  # rhs-major = column-major n x nrhs
        Z = np.empty_like(Xc)
        _check(_lib.hm_mvp_multi(self._h, _ptr(Xc), _ptr(Z), Xc.shape[0], HM_MULTI_DMMA if dmma else HM_MULTI_EXACT))
        return Z.T

    def mvp_multi_device(self, x_ptr: int, z_ptr: int, nrhs: int, dmma: bool = False, stream: int = 0) -> None:
        """Device arrays, column-major n x nrhs (original ordering)."""
        _check(_lib.hm_mvp_multi_device(self._h, C.c_void_p(x_ptr), C.c_void_p(z_ptr), int(nrhs),
                                        HM_MULTI_DMMA if dmma else HM_MULTI_EXACT, C.c_void_p(stream or None)))

    def dump_leaves_csv(self, path: str) -> None:
        """dump_leaves_csv (tree.cpp:197-205): all leaves, canonical order, reference format."""
        _check(_lib.hm_dump_leaves_csv(self._h, os.fsencode(path)))

    def mvp_device(self, x_ptr: int, z_ptr: int, stream: int = 0) -> None:
        """Device pointers (original ordering) on a CUDA stream handle (0 = the handle's stream)."""
        _check(_lib.hm_mvp_device(self._h, C.c_void_p(x_ptr), C.c_void_p(z_ptr), C.c_void_p(stream or None)))

    def mvp_local(self, x) -> np.ndarray:
        """This rank's Morton-ordered row slice of H x, without the allgather."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        st = self.stats()
        z = np.empty(st["row_end"] - st["row_begin"])
        _check(_lib.hm_mvp_local(self._h, _ptr(x), _ptr(z)))
        return z

    def dense_mvp(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        z = np.empty(self.n)
        _check(_lib.hm_dense_mvp(self._h, _ptr(x), _ptr(z)))
        return z

    def attach_nccl(self, unique_id: bytes) -> None:
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        _check(_lib.hm_attach_nccl(self._h, buf))

    # --- per-kernel device timing (CUDA events on the launching stream)
    def profile_begin(self) -> None:
        _check(_lib.hm_profile_begin(self._h))

    def profile_end(self) -> dict:
        ms = np.zeros(8)
        cnt = np.zeros(8, dtype=np.int64)
        _check(_lib.hm_profile_end(self._h, _ptr(ms), _ptr(cnt)))
        return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(KERNEL_IDS) if cnt[i]}

    # --- introspection
    def stats(self) -> dict:
        s = _Stats()
        _check(_lib.hm_get_stats(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in _Stats._fields_}

    def timings(self) -> dict:
        t = _Timings()
        _check(_lib.hm_get_timings(self._h, C.byref(t)))
        return {f: getattr(t, f) for f, _ in _Timings._fields_}

    def points(self):
        coords = np.empty((self.d, self.n))
        perm = np.empty(self.n, dtype=np.int64)
        _check(_lib.hm_get_points(self._h, _ptr(coords), _ptr(perm)))
        return coords, perm

    def codes(self) -> np.ndarray:
        c = np.empty(self.n, dtype=np.uint64)
        _check(_lib.hm_get_codes(self._h, _ptr(c)))
        return c

    def leaves(self, which: int, boxes: bool = True) -> Leaves:
        st = self.stats()
        cnt = st["n_dense"] if which == 0 else st["n_aca"]
        rows = np.empty((cnt, 4), dtype=np.int64)
        bx = np.empty((cnt, 4, self.d)) if boxes else None
        _check(_lib.hm_get_leaves(self._h, which, _ptr(rows), _ptr(bx)))
        return Leaves(rows, bx)

    @property
    def dense_queue(self) -> np.ndarray:
        return self.leaves(0, boxes=False).rows

    @property
    def aca_queue(self) -> np.ndarray:
        return self.leaves(1, boxes=False).rows

    def aca_factors(self, factors: bool = True) -> dict:
        lv = self.aca_queue
        nb, k = lv.shape[0], self.config.k
        ms, ns = lv[:, 1] - lv[:, 0], lv[:, 3] - lv[:, 2]
        k_eff = np.empty(nb, dtype=np.int64)
        rp = np.empty(nb * k, dtype=np.int64)
        cp = np.empty(nb * k, dtype=np.int64)
        u = np.empty(k * int(ms.sum())) if factors else None
        v = np.empty(k * int(ns.sum())) if factors else None
        _check(_lib.hm_get_aca(self._h, _ptr(k_eff), _ptr(rp), _ptr(cp), _ptr(u), _ptr(v)))
        out = {"k_eff": k_eff, "row_piv": rp.reshape(nb, k), "col_piv": cp.reshape(nb, k)}
        if factors:
            us, vs, uo, vo = [], [], 0, 0
            for m, n in zip(ms, ns):
                us.append(u[uo:uo + k * m].reshape(k, m))
                vs.append(v[vo:vo + k * n].reshape(k, n))
                uo += k * m
                vo += k * n
            out["u"], out["v"] = us, vs
        return out


# ----------------------------------------------------------------------------- free functions
def setup(points, kernel: KernelFunction = KernelFunction(), config: HmatrixConfig = HmatrixConfig()) -> HMatrix:
    """hmat::setup (hmatrix.hpp:48).  points: (d, n) float64 SoA in [0,1]^d (host)."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.ndim != 2:
        raise InvalidArgument(HM_EINVAL, "points must be a (d, n) array")
    d, n = pts.shape
    out = C.c_void_p()
    cfg = config._c()
    _check(_lib.hm_setup(_ptr(pts), n, d, kernel.code, float(kernel.matern_beta), C.byref(cfg), C.byref(out)))
    return HMatrix(out.value, n, d, kernel, config)


def setup_device(coords_ptr: int, n: int, d: int, kernel: KernelFunction = KernelFunction(),
                 config: HmatrixConfig = HmatrixConfig()) -> HMatrix:
    out = C.c_void_p()
    cfg = config._c()
    _check(_lib.hm_setup_device(C.c_void_p(coords_ptr), n, d, kernel.code, float(kernel.matern_beta),
                                C.byref(cfg), C.byref(out)))
    return HMatrix(out.value, n, d, kernel, config)


def mvp(h: HMatrix, x, kernel: Optional[KernelFunction] = None, timings: Optional[MvpTimings] = None) -> np.ndarray:
    """hmat::mvp (hmatrix.hpp:58-59).  The kernel captured at setup is used (the
    reference requires the two to match without checking it)."""
    return h.mvp(x, timings)


def relative_error(h: HMatrix, kernel: Optional[KernelFunction] = None, x_rand=None) -> float:
    """hmat::relative_error (hmatrix.hpp:63); the exact product runs on the device (no N limit)."""
    x = np.ascontiguousarray(x_rand, dtype=np.float64)
    if x.shape != (h.n,):
        raise InvalidArgument(HM_EINVAL, "relative_error: vector length mismatch")
    out = C.c_double()
    _check(_lib.hm_relative_error(h._h, _ptr(x), C.byref(out)))
    return float(out.value)


def cg_solve(h: HMatrix, kernel: Optional[KernelFunction], b, config: SolveConfig = SolveConfig()) -> SolveResult:
    """hmat::cg_solve (solver.hpp:27-28)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.shape != (h.n,):
        raise InvalidArgument(HM_EINVAL, "cg_solve: rhs length mismatch")
    x = np.empty(h.n)
    it = C.c_int64()
    rr = C.c_double()
    _check(_lib.hm_cg_solve(h._h, _ptr(b), float(config.sigma2), float(config.tol), int(config.max_iter), _ptr(x),
                            C.byref(it), C.byref(rr)))
    return SolveResult(x, int(it.value), float(rr.value))


def cg_solve_multi(h: HMatrix, B, config: SolveConfig = SolveConfig(), dmma: bool = False):
    """nrhs independent cg_solve runs (solver.cpp:19-73) on multi-RHS products.
    B: n x nrhs.  Returns (X n x nrhs, iterations[nrhs], relative_residual[nrhs])."""
    B = np.asarray(B, dtype=np.float64)
    if B.ndim != 2 or B.shape[0] != h.n:
        raise InvalidArgument(HM_EINVAL, "cg_solve_multi: B must be n x nrhs")
    Bc = np.ascontiguousarray(B.T)
    R = Bc.shape[0]
    X = np.empty_like(Bc)
    it = np.zeros(R, dtype=np.int64)
    rr = np.zeros(R)
    _check(_lib.hm_cg_solve_multi(h._h, _ptr(Bc), R, float(config.sigma2), float(config.tol), int(config.max_iter),
                                  HM_MULTI_DMMA if dmma else HM_MULTI_EXACT, _ptr(X), _ptr(it), _ptr(rr)))
    return X.T, it, rr


def morton_codes(coords) -> np.ndarray:
    """compute_morton_codes (morton.hpp:23) on the device."""
    c = np.ascontiguousarray(coords, dtype=np.float64)
    d, n = c.shape
    out = np.empty(n, dtype=np.uint64)
    _check(_lib.hm_morton_codes(_ptr(c), n, d, _ptr(out)))
    return out


def morton_order(coords, perm=None):
    """morton_order (morton.hpp:26): returns (sorted coords, composed perm)."""
    c = np.ascontiguousarray(coords, dtype=np.float64)
    d, n = c.shape
    out = np.empty_like(c)
    pout = np.empty(n, dtype=np.int64)
    pin = None if perm is None else np.ascontiguousarray(perm, dtype=np.int64)
    _check(_lib.hm_morton_order(_ptr(c), n, d, _ptr(pin), _ptr(out), _ptr(pout)))
    return out, pout


def aca_batched_dense(blocks, kmax: int, epsilon: Optional[float] = None, eta: float = 0.0):
    """aca_batched on explicit blocks (aca.hpp:88-89) on the device.
    Returns (k_eff, row_piv (B,k), col_piv (B,k), [u (k,m)], [v (k,n)])."""
    shapes = np.array([b.shape for b in blocks], dtype=np.int64).reshape(-1)
    entries = np.concatenate([np.ascontiguousarray(b, dtype=np.float64).ravel() for b in blocks])
    nb = len(blocks)
    ms = [b.shape[0] for b in blocks]
    ns = [b.shape[1] for b in blocks]
    k_eff = np.empty(nb, dtype=np.int64)
    rp = np.empty(nb * kmax, dtype=np.int64)
    cp = np.empty(nb * kmax, dtype=np.int64)
    u = np.empty(kmax * sum(ms))
    v = np.empty(kmax * sum(ns))
    _check(_lib.hm_aca_dense(nb, _ptr(shapes), _ptr(entries), kmax, int(epsilon is not None), float(epsilon or 0.0),
                             float(eta), _ptr(k_eff), _ptr(rp), _ptr(cp), _ptr(u), _ptr(v)))
    us, vs, uo, vo = [], [], 0, 0
    for m, n in zip(ms, ns):
        us.append(u[uo:uo + kmax * m].reshape(kmax, m))
        vs.append(v[vo:vo + kmax * n].reshape(kmax, n))
        uo += kmax * m
        vo += kmax * n
    return k_eff, rp.reshape(nb, kmax), cp.reshape(nb, kmax), us, vs


def eval_kernel(kernel: KernelFunction, y, yp) -> np.ndarray:
    """phi(y_i, yp_i) for SoA point pairs (eval_kernel, core.hpp:63-64), on the device."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    yp = np.ascontiguousarray(yp, dtype=np.float64)
    d, n = y.shape
    out = np.empty(n)
    _check(_lib.hm_eval_kernel(kernel.code, float(kernel.matern_beta), d, n, _ptr(y), _ptr(yp), _ptr(out)))
    return out


def exp_port_host(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _lib.hm_exp_port_host(x.size, _ptr(x), _ptr(out))
    return out


def exp_port_device(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _check(_lib.hm_exp_port_device(x.size, _ptr(x), _ptr(out)))
    return out


def log_port_host(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _lib.hm_log_port_host(x.size, _ptr(x), _ptr(out))
    return out


def log_port_device(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _check(_lib.hm_log_port_device(x.size, _ptr(x), _ptr(out)))
    return out


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(_lib.hm_nccl_unique_id(buf))
    return bytes(buf)
