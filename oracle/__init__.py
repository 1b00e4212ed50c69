"""ctypes view of oracle/build/liboracle.so — the CPU restatement of the reference path.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs, never by the product package (paper_1304_6514_b200/).
"""
from __future__ import annotations

import ctypes as C
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "liboracle.so"
REF_TOOL = HERE / "_ref" / "ref_tool"

_lib = None

_d = C.c_double
_i = C.c_int64
_pd = C.POINTER(C.c_double)
_pf = C.POINTER(C.c_float)
_pi = C.POINTER(C.c_int64)

_SIGS = {
    "or_steps_for": (_i, [_d, _d]),
    "or_decompose": (C.c_int, [_d, _d, _i, _d, _pd, _pd, _pi, _pd]),
    "or_riccati_step": (C.c_int, [_d, _d, _pd]),
    "or_riccati_integrate": (C.c_int, [_d, _i, _d, _pd]),
    "or_riccati_ensemble": (_i, [_i, _i, _pi, _pd, _pd, _pd, _pd]),
    "or_cheb_nodes1": (C.c_int, [_i, _d, _d, _pd]),
    "or_cheb_nodes2": (C.c_int, [_i, _d, _d, _pd]),
    "or_bary_weights": (C.c_int, [_pd, _i, _pd]),
    "or_bary_weights_closed2": (None, [_i, _pd]),
    "or_interp_eval": (_d, [_pd, _pd, _pd, _i, _d]),
    "or_scalar_sweep": (_d, [_pd, _pd, _pd, _i, _i, _d, _d, _d, _pd, _pi]),
    "or_matvec": (None, [_pd, _i, _i, _pd, _pd]),
    "or_matmul": (None, [_pd, _pd, _i, _i, _i, _pd]),
    "or_thomas": (C.c_int, [_pd, _pd, _pd, _i, _pd]),
    "or_heat_coefficient": (_d, [_d]),
    "or_heat_forcing": (_d, [_d, _d]),
    "or_heat_dim": (_i, [_d]),
    "or_heat_initial": (None, [_d, _i, _pd]),
    "or_heat_exact": (None, [_d, _i, _d, _pd]),
    "or_heat_integrate": (C.c_int, [_d, _i, _d, _d, _d, C.c_int, _pd]),
    "or_heat_build": (C.c_int, [_d, _i, _d, _d, _d, _pd, _pd]),
    "or_affine_chain": (None, [_pd, _pd, _i, _i, _pd, _pd]),
    "or_affine_tree": (None, [_pd, _pd, _i, _i, _pd, _pd, _pd, _pd]),
    "or_logistic_rk4_ensemble": (None, [_i, _i, _pi, _pd, _pd, _d, _d, _pd]),
    "or_logistic_rk4_ensemble_f32": (None, [_i, _i, _pi, _pd, _pf, C.c_float, C.c_float, _pf]),
    "or_lv_rk4_ensemble": (None, [_i, _i, _i, _pi, _pd, _pd, _pd, _pd, _pd]),
    "or_lv_rk4_subset": (None, [_i, _i, _i, _i, _pi, _pd, _pd, _pd, _pd, _pd]),
    "or_bracket": (_i, [_pd, _i, _d]),
    "or_lerp": (_d, [_d, _d, _d]),
    "or_bilinear_sweep": (_i, [_pd, _i, _pd, _i, _pd, _i, _d, _d, _pd, _pi]),
    "or_uniform_nodes": (None, [_i, _d, _d, _pd]),
}


def build() -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    if a.dtype == np.float64:
        return a.ctypes.data_as(_pd)
    if a.dtype == np.float32:
        return a.ctypes.data_as(_pf)
    if a.dtype == np.int64:
        return a.ctypes.data_as(_pi)
    raise TypeError(a.dtype)


def f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


# ---- thin numpy-facing wrappers -------------------------------------------------------------

def steps_for(width: float, dt: float) -> int:
    return int(lib().or_steps_for(width, dt))


def decompose(t0: float, T: float, N: int, dt: float):
    tb, te, h = (np.empty(N) for _ in range(3))
    st = np.empty(N, dtype=np.int64)
    if lib().or_decompose(t0, T, N, dt, _p(tb), _p(te), _p(st), _p(h)) != 0:
        raise ValueError("BadGrid")
    return tb, te, st, h


def riccati_step(y: float, dt: float):
    z = C.c_double()
    rc = lib().or_riccati_step(y, dt, C.byref(z))
    return rc, z.value


def riccati_ensemble(steps, h, nodes):
    steps, h, nodes = np.ascontiguousarray(steps, np.int64), f64(h), f64(nodes)
    N, M = len(steps), len(nodes)
    out = np.empty(N * M)
    fv = C.c_double(0.0)
    fail = lib().or_riccati_ensemble(N, M, _p(steps), _p(h), _p(nodes), _p(out), C.byref(fv))
    return out.reshape(N, M), int(fail), fv.value


def cheb_nodes(M: int, a: float, b: float, kind: int = 2) -> np.ndarray:
    x = np.empty(M)
    fn = lib().or_cheb_nodes2 if kind == 2 else lib().or_cheb_nodes1
    if fn(M, a, b, _p(x)) != 0:
        raise ValueError("BadGrid")
    return x


def bary_weights(x) -> np.ndarray:
    x = f64(x)
    w = np.empty(len(x))
    if lib().or_bary_weights(_p(x), len(x), _p(w)) != 0:
        raise ValueError("DuplicateNodes")
    return w


def bary_weights_closed2(M: int) -> np.ndarray:
    w = np.empty(M)
    lib().or_bary_weights_closed2(M, _p(w))
    return w


def interp_eval(x, w, v, xi: float) -> float:
    x, w, v = f64(x), f64(w), f64(v)
    return float(lib().or_interp_eval(_p(x), _p(w), _p(v), len(x), xi))


def scalar_sweep(x, w, values, a, b, y0):
    x, w, values = f64(x), f64(w), f64(values)
    N, M = values.shape
    lam = np.empty(N)
    ext = C.c_int64(0)
    y = lib().or_scalar_sweep(_p(x), _p(w), _p(values), N, M, a, b, y0, _p(lam), C.byref(ext))
    return float(y), lam, int(ext.value)


def thomas(sub, diag, sup, rhs) -> np.ndarray:
    sub, diag, sup, d = f64(sub), f64(diag), f64(sup), f64(rhs).copy()
    if lib().or_thomas(_p(sub), _p(diag), _p(sup), len(diag), _p(d)) != 0:
        raise ValueError("SingularSystem")
    return d


def matvec(A, x) -> np.ndarray:
    A, x = f64(A), f64(x)
    y = np.empty(A.shape[0])
    lib().or_matvec(_p(A), A.shape[0], A.shape[1], _p(x), _p(y))
    return y


def matmul(A, B) -> np.ndarray:
    A, B = f64(A), f64(B)
    C_ = np.empty((A.shape[0], B.shape[1]))
    lib().or_matmul(_p(A), _p(B), A.shape[0], A.shape[1], B.shape[1], _p(C_))
    return C_


def heat_dim(dx: float) -> int:
    n = int(lib().or_heat_dim(dx))
    if n < 0:
        raise ValueError("BadGrid")
    return n


def heat_initial(dx: float) -> np.ndarray:
    n = heat_dim(dx)
    u = np.empty(n)
    lib().or_heat_initial(dx, n, _p(u))
    return u


def heat_exact(dx: float, t: float) -> np.ndarray:
    n = heat_dim(dx)
    u = np.empty(n)
    lib().or_heat_exact(dx, n, t, _p(u))
    return u


def heat_integrate(dx, t_begin, t_end, dt_nominal, y, with_forcing=True) -> np.ndarray:
    y = f64(y).copy()
    if lib().or_heat_integrate(dx, len(y), t_begin, t_end, dt_nominal, int(with_forcing), _p(y)):
        raise ValueError("SingularSystem")
    return y


def heat_build(dx, t_begin, t_end, dt_nominal):
    n = heat_dim(dx)
    G = np.empty((n, n))
    c = np.empty(n)
    if lib().or_heat_build(dx, n, t_begin, t_end, dt_nominal, _p(G), _p(c)):
        raise ValueError("SingularSystem")
    return G, c


def affine_chain(G, c, y0) -> np.ndarray:
    G, c, y0 = f64(G), f64(c), f64(y0)
    N, n, _ = G.shape
    y = np.empty(n)
    lib().or_affine_chain(_p(G), _p(c), N, n, _p(y0), _p(y))
    return y


def affine_tree(G, c, y0):
    G, c, y0 = f64(G).copy(), f64(c).copy(), f64(y0)
    N, n, _ = G.shape
    Go, co, y = np.empty((n, n)), np.empty(n), np.empty(n)
    lib().or_affine_tree(_p(G), _p(c), N, n, _p(y0), _p(Go), _p(co), _p(y))
    return Go, co, y


def logistic_rk4_ensemble(steps, h, nodes, r, K) -> np.ndarray:
    steps, h, nodes = np.ascontiguousarray(steps, np.int64), f64(h), f64(nodes)
    out = np.empty(len(steps) * len(nodes))
    lib().or_logistic_rk4_ensemble(len(steps), len(nodes), _p(steps), _p(h), _p(nodes), r, K, _p(out))
    return out.reshape(len(steps), len(nodes))


def logistic_rk4_ensemble_f32(steps, h, nodes, r, K) -> np.ndarray:
    steps, h = np.ascontiguousarray(steps, np.int64), f64(h)
    nodes = np.ascontiguousarray(nodes, np.float32)
    out = np.empty(len(steps) * len(nodes), dtype=np.float32)
    lib().or_logistic_rk4_ensemble_f32(len(steps), len(nodes), _p(steps), _p(h), _p(nodes), r, K,
                                       _p(out))
    return out.reshape(len(steps), len(nodes))


def lv_rk4_ensemble(steps, h, un, vn, params) -> np.ndarray:
    steps, h, un, vn, params = (np.ascontiguousarray(steps, np.int64), f64(h), f64(un), f64(vn),
                                f64(params))
    N, Mu, Mv = len(steps), len(un), len(vn)
    out = np.empty(N * 2 * Mu * Mv)
    lib().or_lv_rk4_ensemble(N, Mu, Mv, _p(steps), _p(h), _p(un), _p(vn), _p(params), _p(out))
    return out.reshape(N, 2, Mu, Mv)


def lv_rk4_subset(lo, hi, steps, h, un, vn, params) -> np.ndarray:
    steps, h, un, vn, params = (np.ascontiguousarray(steps, np.int64), f64(h), f64(un), f64(vn),
                                f64(params))
    out = np.empty((hi - lo) * 2)
    lib().or_lv_rk4_subset(lo, hi, len(un), len(vn), _p(steps), _p(h), _p(un), _p(vn), _p(params),
                           _p(out))
    return out.reshape(hi - lo, 2)


def bracket(x, xi: float) -> int:
    x = f64(x)
    return int(lib().or_bracket(_p(x), len(x), xi))


def bilinear_sweep(un, vn, tables, u0, v0):
    un, vn, tables = f64(un), f64(vn), f64(tables)
    N = tables.shape[0]
    lam = np.empty(2 * N)
    br = np.empty(2 * N, dtype=np.int64)
    ext = lib().or_bilinear_sweep(_p(un), len(un), _p(vn), len(vn), _p(tables), N, u0, v0, _p(lam),
                                  _p(br))
    return lam.reshape(N, 2), br.reshape(N, 2), int(ext)


def uniform_nodes(M: int, a: float, b: float) -> np.ndarray:
    x = np.empty(M)
    lib().or_uniform_nodes(M, a, b, _p(x))
    return x
