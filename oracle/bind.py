"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle()``    -- oracle/liboracle.so, the C restatement (hmat_oracle.c)
* ``Reference()`` -- oracle/_ref/libhmat_ref.so, the unmodified reference library
                     compiled from /root/reference by oracle/Makefile, run
                     single-threaded.

Both expose the same Python surface so tests can pin one against the other.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg
import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhmat_ref.so")

_p = C.c_void_p
_i64 = C.c_int64
_i = C.c_int
_d = C.c_double


def _ptr(a):
    return None if a is None else a.ctypes.data


@dataclass
class Leaves:
    rows: np.ndarray   # (L, 4) int64: row.lower, row.upper, col.lower, col.upper
    boxes: np.ndarray  # (L, 4, d): row a, row b, col a, col b


class _Checker:
    prefix = ""
    so = ""

    def __init__(self):
        if not os.path.exists(self.so):
            raise FileNotFoundError(f"{self.so} not built (run `make -C oracle`)")
        self.lib = C.CDLL(self.so)
        L, p = self.lib, self.prefix
        getattr(L, p + "last_error").restype = C.c_char_p
        getattr(L, p + "count").restype = _i64
        getattr(L, p + "count").argtypes = [_p, _i]
        getattr(L, p + "free").argtypes = [_p]
        for name in ("leaves", "points", "mvp", "mvp_rows", "aca_all", "relative_error", "cg"):
            getattr(L, p + name).restype = _i
        getattr(L, p + "leaves").argtypes = [_p, _i, _p, _p]
        getattr(L, p + "points").argtypes = [_p, _p, _p]
        getattr(L, p + "mvp_rows").argtypes = [_p, _p, _i64, _p, _p]
        getattr(L, p + "aca_all").argtypes = [_p, _p, _p, _p, _p, _p, _p]
        getattr(L, p + "relative_error").argtypes = [_p, _p, _p]
        getattr(L, p + "cg").argtypes = [_p, _p, _d, _d, _i64, _p, _p, _p]

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self._fn("last_error")().decode())

    # ---- core / morton --------------------------------------------------
    def bessel_k1(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._check(self._fn("bessel_k1")(_i64(x.size), _ptr(x), _ptr(out)))
        return out

    def eval_kernel(self, kind, beta, y, yp):
        y = np.ascontiguousarray(y, dtype=np.float64)
        yp = np.ascontiguousarray(yp, dtype=np.float64)
        d, n = y.shape
        out = np.empty(n)
        self._check(self._fn("eval_kernel")(_i(kind), _d(beta), _i(d), _i64(n), _ptr(y), _ptr(yp), _ptr(out)))
        return out

    def morton_codes(self, coords):
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        d, n = coords.shape
        codes = np.empty(n, dtype=np.uint64)
        self._check(self._fn("morton_codes")(_i64(n), _i(d), _ptr(coords), _ptr(codes)))
        return codes

    def morton_order(self, coords, perm=None):
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        d, n = coords.shape
        out = np.empty_like(coords)
        perm_out = np.empty(n, dtype=np.int64)
        pin = None if perm is None else np.ascontiguousarray(perm, dtype=np.int64)
        self._check(self._fn("morton_order")(_i64(n), _i(d), _ptr(coords), _ptr(pin), _ptr(out), _ptr(perm_out)))
        return out, perm_out

    # ---- H-matrix --------------------------------------------------------
    def setup(self, coords, kernel=0, beta=0.0, eta=1.5, c_leaf=256, k=16, precompute=False, epsilon=None,
              mode=0, bs_aca=1 << 20, bs_dense=1 << 22):
        return _Handle(self, np.ascontiguousarray(coords, dtype=np.float64), kernel, beta, eta, c_leaf, k,
                       precompute, epsilon, mode, bs_aca, bs_dense)

    def aca_dense(self, blocks, kmax, epsilon=None, eta=0.0, single=False):
        """Explicit-matrix seam: list of 2-D arrays -> (k_eff, row_piv, col_piv, [u], [v])."""
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
        args = [_i64(nb), _ptr(shapes), _ptr(entries), _i64(kmax), _i(epsilon is not None),
                _d(epsilon or 0.0), _d(eta)]
        if self.prefix == "ref_":
            args.append(_i(1 if single else 0))
        elif single:
            raise ValueError("the oracle restates the batched semantics only")
        self._check(self._fn("aca_dense")(*args, _ptr(k_eff), _ptr(rp), _ptr(cp), _ptr(u), _ptr(v)))
        us, vs, uo, vo = [], [], 0, 0
        for m, n in zip(ms, ns):
            us.append(u[uo:uo + kmax * m].reshape(kmax, m))
            vs.append(v[vo:vo + kmax * n].reshape(kmax, n))
            uo += kmax * m
            vo += kmax * n
        return k_eff, rp.reshape(nb, kmax), cp.reshape(nb, kmax), us, vs


class _Handle:
    def __init__(self, chk, coords, kernel, beta, eta, c_leaf, k, precompute, epsilon, mode, bs_aca, bs_dense):
        self.chk = chk
        d, n = coords.shape
        self.n, self.d, self.k = n, d, k
        has_eps = epsilon is not None
        f = chk._fn("setup")
        f.restype = _p
        if chk.prefix == "ref_":
            if mode == 2:
                raise ValueError("the reference setup() has no ForceAdmissible mode")
            f.argtypes = [_i64, _i, _p, _i, _d, _d, _i64, _i64, _i64, _i64, _i, _i, _d, _i]
            self.h = f(n, d, _ptr(coords), kernel, beta, eta, c_leaf, k, bs_aca, bs_dense, int(precompute),
                       int(has_eps), float(epsilon or 0.0), int(mode == 1))
        else:
            f.argtypes = [_i64, _i, _p, _i, _d, _d, _i64, _i64, _i, _i, _d, _i]
            self.h = f(n, d, _ptr(coords), kernel, beta, eta, c_leaf, k, int(precompute), int(has_eps),
                       float(epsilon or 0.0), mode)
        if not self.h:
            raise RuntimeError(chk._fn("last_error")().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.chk._fn("free")(self.h)
            self.h = None

    def count(self, which):
        return int(self.chk._fn("count")(self.h, which))

    def leaves(self, which, boxes=True):
        cnt = self.count(which)
        rows = np.empty((cnt, 4), dtype=np.int64)
        bx = np.empty((cnt, 4, self.d)) if boxes else None
        self.chk._check(self.chk._fn("leaves")(self.h, which, _ptr(rows), _ptr(bx)))
        return Leaves(rows, bx)

    def points(self):
        coords = np.empty((self.d, self.n))
        perm = np.empty(self.n, dtype=np.int64)
        self.chk._check(self.chk._fn("points")(self.h, _ptr(coords), _ptr(perm)))
        return coords, perm

    def mvp(self, x, timings=False):
        x = np.ascontiguousarray(x, dtype=np.float64)
        z = np.empty(self.n)
        f = self.chk._fn("mvp")
        if self.chk.prefix == "ref_":
            f.argtypes = [_p, _p, _p, _p]
            t = np.zeros(3)
            self.chk._check(f(self.h, _ptr(x), _ptr(z), _ptr(t)))
            return (z, t) if timings else z
        f.argtypes = [_p, _p, _p]
        self.chk._check(f(self.h, _ptr(x), _ptr(z)))
        return z

    def mvp_rows(self, x, ranges):
        x = np.ascontiguousarray(x, dtype=np.float64)
        r = np.ascontiguousarray(np.asarray(ranges, dtype=np.int64).reshape(-1))
        z = np.empty(self.n)
        self.chk._check(self.chk._fn("mvp_rows")(self.h, _ptr(x), _i64(r.size // 2), _ptr(r), _ptr(z)))
        return z

    def aca_all(self, factors=True):
        """Per admissible block: k_eff, pivots (B,k), and optionally u/v lists (k,m)/(k,n)."""
        lv = self.leaves(1, boxes=False).rows
        nb = lv.shape[0]
        k = self.k
        ms = lv[:, 1] - lv[:, 0]
        ns = lv[:, 3] - lv[:, 2]
        k_eff = np.empty(nb, dtype=np.int64)
        rp = np.empty(nb * k, dtype=np.int64)
        cp = np.empty(nb * k, dtype=np.int64)
        rej = np.zeros(nb, dtype=np.int64)
        u = np.empty(k * int(ms.sum())) if factors else None
        v = np.empty(k * int(ns.sum())) if factors else None
        if self.chk.prefix == "ref_" and not factors:
            u = np.empty(k * int(ms.sum()))
            v = np.empty(k * int(ns.sum()))
        self.chk._check(self.chk._fn("aca_all")(self.h, _ptr(k_eff), _ptr(rp), _ptr(cp), _ptr(u), _ptr(v),
                                                 _ptr(rej)))
        out = {"k_eff": k_eff, "row_piv": rp.reshape(nb, k), "col_piv": cp.reshape(nb, k), "rejections": rej}
        if factors:
            us, vs, uo, vo = [], [], 0, 0
            for m, n in zip(ms, ns):
                us.append(u[uo:uo + k * m].reshape(k, m))
                vs.append(v[vo:vo + k * n].reshape(k, n))
                uo += k * m
                vo += k * n
            out["u"], out["v"] = us, vs
        return out

    def relative_error(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(1)
        self.chk._check(self.chk._fn("relative_error")(self.h, _ptr(x), _ptr(out)))
        return float(out[0])

    def cg(self, b, sigma2, tol=1e-8, max_iter=500):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(self.n)
        it = np.zeros(1, dtype=np.int64)
        rr = np.zeros(1)
        self.chk._check(self.chk._fn("cg")(self.h, _ptr(b), _d(sigma2), _d(tol), _i64(max_iter), _ptr(x),
                                            _ptr(it), _ptr(rr)))
        return x, int(it[0]), float(rr[0])


class Oracle(_Checker):
    prefix = "orc_"
    so = ORACLE_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        L.orc_bessel_k1.argtypes = [_i64, _p, _p]
        L.orc_eval_kernel.argtypes = [_i, _d, _i, _i64, _p, _p, _p]
        L.orc_morton_codes.argtypes = [_i64, _i, _p, _p]
        L.orc_morton_order.argtypes = [_i64, _i, _p, _p, _p, _p]
        L.orc_aca_dense.argtypes = [_i64, _p, _p, _i64, _i, _d, _d, _p, _p, _p, _p, _p]
        L.orc_admissible.argtypes = [_i, _p, _p, _d, _p, _p, _p]
        L.orc_dense_mvp.argtypes = [_p, _p, _p]

    def admissible(self, box_t, box_s, eta):
        bt = np.ascontiguousarray(box_t, dtype=np.float64).ravel()
        bs = np.ascontiguousarray(box_s, dtype=np.float64).ravel()
        d = bt.size // 2
        out = np.zeros(3)
        adm = self.lib.orc_admissible(d, _ptr(bt), _ptr(bs), _d(eta), _ptr(out[0:]), _ptr(out[1:]), _ptr(out[2:]))
        return bool(adm), out


class Reference(_Checker):
    prefix = "ref_"
    so = REF_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        L.ref_bessel_k1.argtypes = [_i64, _p, _p]
        L.ref_eval_kernel.argtypes = [_i, _d, _i, _i64, _p, _p, _p]
        L.ref_morton_codes.argtypes = [_i64, _i, _p, _p]
        L.ref_morton_order.argtypes = [_i64, _i, _p, _p, _p, _p]
        L.ref_aca_dense.argtypes = [_i64, _p, _p, _i64, _i, _d, _d, _i, _p, _p, _p, _p, _p]
        L.ref_halton.argtypes = [_i64, _i, _p]
        L.ref_threads.restype = _i

    def halton(self, n, d):
        out = np.empty((d, n))
        self._check(self.lib.ref_halton(_i64(n), _i(d), _ptr(out)))
        return out


REF_DUMP_CSV = os.path.join(HERE, "_ref", "ref_dump_csv")


def reference_leaf_csv(coords, c_leaf, eta, path):
    """The reference's own dump_leaves_csv (tree.cpp:197-205) after its setup(), run in a
    separate process (oracle/ref_dump_csv.cpp)."""
    import subprocess
    import tempfile
    c = np.ascontiguousarray(coords, dtype=np.float64)
    d, n = c.shape
    with tempfile.NamedTemporaryFile(suffix=".bin") as f:
        c.tofile(f.name)
        subprocess.run([REF_DUMP_CSV, str(n), str(d), str(c_leaf), repr(float(eta)), f.name, str(path)], check=True)


def available(kind: str) -> bool:
    return os.path.exists(REF_SO if kind == "ref" else ORACLE_SO)
