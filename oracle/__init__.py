"""ctypes binding of the serial C++ IFGF oracle (oracle/ifgf_oracle.cpp).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this module.
The product package ``paper_2010_02857_b200`` never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ifgf_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

ST_NEAR, ST_COUSIN, ST_UPWARD = 1, 2, 4
ST_ALL = 7
MODE_NORMAL, MODE_BYPASS = 0, 1

CFLAGS = ["-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (the checker is built, not used, by build())."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *CFLAGS, _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            c_d, c_i, c_i64, c_p = ctypes.c_double, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
            L.oracle_plan_create.argtypes = [c_p, c_i64, c_d, c_i, c_i, c_i, c_i, c_i, c_i, c_p, c_d,
                                             ctypes.POINTER(c_p)]
            L.oracle_plan_create_part.argtypes = [c_p, c_i64, c_d, c_i, c_i, c_i, c_i, c_i, c_i, c_p, c_d,
                                                  ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(c_p)]
            L.oracle_plan_destroy.argtypes = [c_p]
            L.oracle_apply.argtypes = [c_p, c_p, c_p, ctypes.c_uint, c_i]
            L.oracle_recentering_check.argtypes = [c_p, c_p]
            L.oracle_recentering_check.restype = c_d
            L.oracle_level_info.argtypes = [c_p, c_i, c_p]
            L.oracle_level_boxes.argtypes = [c_p, c_i, c_p, c_i64]
            L.oracle_level_boxes.restype = c_i64
            L.oracle_level_segments.argtypes = [c_p, c_i, c_p, c_i64]
            L.oracle_level_segments.restype = c_i64
            L.oracle_box_list.argtypes = [c_p, c_i, c_i64, c_i, c_p, c_i64]
            L.oracle_box_list.restype = c_i64
            L.oracle_direct.argtypes = [c_p, c_i64, c_d, c_p, c_p, c_i64, c_p]
            L.oracle_green.argtypes = [c_p, c_p, c_d, c_p]
            L.oracle_analytic_factor.argtypes = [c_p, c_p, c_p, c_d, c_p]
            L.oracle_recenter.argtypes = [c_p, c_p, c_d, c_p]
            L.oracle_cheb_nodes.argtypes = [c_i, c_p]
            L.oracle_cheb_fit1d.argtypes = [c_i, c_p, c_p]
            L.oracle_cheb_eval1d.argtypes = [c_i, c_p, c_d, c_p]
            L.oracle_tensor_fit.argtypes = [c_i, c_i, c_p, c_p]
            L.oracle_tensor_eval.argtypes = [c_i, c_i, c_p, c_d, c_d, c_d, c_p]
            L.oracle_classify.argtypes = [c_d, c_i, c_i, c_p, c_p, c_p]
            L.oracle_node_offset.argtypes = [c_d, c_i, c_i, c_i, c_i, c_p, c_p, c_p]
            L.oracle_set_threads.argtypes = [c_i]
            L.oracle_get_threads.restype = c_i
            _lib = L
    return _lib


def set_threads(n: int) -> None:
    """Threads of the oracle's parallel loops (0 = all processors, 1 = serial).
    Results are bitwise independent of it (target- / parent-segment-major loops
    with one owner per output; oracle/ifgf_oracle.cpp header)."""
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


class OraclePlan:
    """Oracle plan: box tree, cone grids and relevant segments."""

    def __init__(self, points, k, levels, Ps, Pang, leaf_ns=1, leaf_nc=2, root=None, owned_morton=None):
        """owned_morton: optional half-open range (lo, hi) of leaf Morton keys whose
        sources this plan owns (source partition); apply() then
        returns the partial field over all targets."""
        L = lib()
        self.points = _f64(points).reshape(-1, 3)
        self.n = self.points.shape[0]
        self.D, self.Ps, self.Pang = int(levels), int(Ps), int(Pang)
        self.k = float(k)
        lo, hi = (0, 2 ** 64 - 1) if owned_morton is None else (int(owned_morton[0]), int(owned_morton[1]))
        h = ctypes.c_void_p()
        if root is not None:
            rc = _f64(root[0])
            st = L.oracle_plan_create_part(_ptr(self.points), self.n, self.k, self.D, self.Ps, self.Pang, leaf_ns,
                                           leaf_nc, 1, _ptr(rc), float(root[1]), lo, hi, ctypes.byref(h))
        else:
            st = L.oracle_plan_create_part(_ptr(self.points), self.n, self.k, self.D, self.Ps, self.Pang, leaf_ns,
                                           leaf_nc, 0, None, 0.0, lo, hi, ctypes.byref(h))
        if st != 0:
            raise OracleError(st, "oracle_plan_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().oracle_plan_destroy(h)
            self._h = None

    def apply(self, a, stage_mask: int = ST_ALL, mode: int = MODE_NORMAL) -> np.ndarray:
        a = _c128(a)
        assert a.shape == (self.n,)
        out = np.zeros(self.n, dtype=np.complex128)
        st = lib().oracle_apply(self._h, _ptr(a), _ptr(out), stage_mask, mode)
        if st != 0:
            raise OracleError(st, "oracle_apply")
        return out

    def recentering_check(self, a) -> float:
        a = _c128(a)
        return float(lib().oracle_recentering_check(self._h, _ptr(a)))

    def level_info(self, d: int) -> dict:
        info = np.zeros(10, dtype=np.float64)
        st = lib().oracle_level_info(self._h, d, _ptr(info))
        if st != 0:
            raise OracleError(st, "oracle_level_info")
        return dict(nbox=int(info[0]), nseg=int(info[1]), ns=int(info[2]), nC=int(info[3]), H=info[4], h=info[5],
                    x0=info[6:9].copy())

    def level_boxes(self, d: int) -> np.ndarray:
        nb = lib().oracle_level_boxes(self._h, d, None, 0)
        out = np.zeros((nb, 5), dtype=np.int64)
        lib().oracle_level_boxes(self._h, d, _ptr(out), nb)
        return out

    def level_segments(self, d: int) -> np.ndarray:
        ns = lib().oracle_level_segments(self._h, d, None, 0)
        out = np.zeros((ns, 4), dtype=np.int64)
        if ns:
            lib().oracle_level_segments(self._h, d, _ptr(out), ns)
        return out

    def box_list(self, d: int, b: int, which: str) -> np.ndarray:
        w = {"nbrs": 0, "cousins": 1, "children": 2}[which]
        cnt = lib().oracle_box_list(self._h, d, b, w, None, 0)
        out = np.zeros(max(cnt, 1), dtype=np.int64)
        lib().oracle_box_list(self._h, d, b, w, _ptr(out), cnt)
        return out[:cnt]


def direct(points, k, a, targets) -> np.ndarray:
    """Direct sum at the given target indices (eq. field1), Kahan-compensated."""
    pts = _f64(points).reshape(-1, 3)
    a = _c128(a)
    t = np.ascontiguousarray(np.asarray(targets, dtype=np.int64))
    out = np.zeros(t.shape[0], dtype=np.complex128)
    st = lib().oracle_direct(_ptr(pts), pts.shape[0], float(k), _ptr(a), _ptr(t), t.shape[0], _ptr(out))
    if st != 0:
        raise OracleError(st, "oracle_direct")
    return out


def green(x, y, k) -> complex:
    out = np.zeros(2)
    lib().oracle_green(_ptr(_f64(x)), _ptr(_f64(y)), float(k), _ptr(out))
    return complex(out[0], out[1])


def analytic_factor(x, xp, c, k) -> complex:
    out = np.zeros(2)
    lib().oracle_analytic_factor(_ptr(_f64(x)), _ptr(_f64(xp)), _ptr(_f64(c)), float(k), _ptr(out))
    return complex(out[0], out[1])


def recenter(off, delta, k) -> complex:
    out = np.zeros(2)
    lib().oracle_recenter(_ptr(_f64(off)), _ptr(_f64(delta)), float(k), _ptr(out))
    return complex(out[0], out[1])


def cheb_nodes(n: int) -> np.ndarray:
    t = np.zeros(n)
    lib().oracle_cheb_nodes(n, _ptr(t))
    return t


def cheb_fit1d(u) -> np.ndarray:
    u = _c128(u)
    a = np.zeros_like(u)
    lib().oracle_cheb_fit1d(u.shape[0], _ptr(u), _ptr(a))
    return a


def cheb_eval1d(a, x: float) -> complex:
    a = _c128(a)
    out = np.zeros(2)
    lib().oracle_cheb_eval1d(a.shape[0], _ptr(a), float(x), _ptr(out))
    return complex(out[0], out[1])


def tensor_fit(Ps, Pa, V) -> np.ndarray:
    V = _c128(V)
    C = np.zeros_like(V)
    lib().oracle_tensor_fit(Ps, Pa, _ptr(V), _ptr(C))
    return C


def tensor_eval(Ps, Pa, C, us, ut, up) -> complex:
    C = _c128(C)
    out = np.zeros(2)
    lib().oracle_tensor_eval(Ps, Pa, _ptr(C), float(us), float(ut), float(up), _ptr(out))
    return complex(out[0], out[1])


def classify(H, ns, nC, v):
    cell = np.zeros(3, dtype=np.int32)
    loc = np.zeros(6)
    lib().oracle_classify(float(H), int(ns), int(nC), _ptr(_f64(v)), _ptr(cell), _ptr(loc))
    return tuple(int(c) for c in cell), loc[:5].copy()


def node_offset(H, ns, nC, Ps, Pa, cell, node) -> np.ndarray:
    c = np.ascontiguousarray(np.asarray(cell, dtype=np.int32))
    nd = np.ascontiguousarray(np.asarray(node, dtype=np.int32))
    off = np.zeros(3)
    lib().oracle_node_offset(float(H), int(ns), int(nC), int(Ps), int(Pa), _ptr(c), _ptr(nd), _ptr(off))
    return off


def rel_l2(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.sqrt(np.sum(np.abs(a - b) ** 2) / np.sum(np.abs(b) ** 2)))
