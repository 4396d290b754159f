"""ctypes binding of the C oracle (oracle/bsde_oracle.c).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  Argument marshalling only;
all arithmetic is in bsde_oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bsde_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

DRIVERS = {"zero": 0, "affine": 1, "ex1": 2, "ex2": 3, "diff_rates": 4}
TERMINALS = {"const": 0, "poly": 1, "logistic": 2, "ex2": 3, "call_w": 4, "sin_sum": 5,
             "exchange_w": 6, "geo_basket_w": 7, "call_x": 8}
SDES = {"brownian": 0, "gbm": 1, "ou": 2}
INTERPS = {"spline": 0, "fd_bicubic": 1}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with -O2 -ffp-contract=off (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "bsde_oracle.h"))):
        cmd = ["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", "-Wall", "-Wno-unused-function", "-o", _LIB_PATH + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


class _Cfg(C.Structure):
    _fields_ = [("d", C.c_int32), ("t0", C.c_double), ("T", C.c_double), ("N", C.c_int32),
                ("Ky", C.c_int32), ("Kz", C.c_int32), ("L", C.c_int32),
                ("npts", C.c_int64 * 3), ("xlo", C.c_double * 3), ("xhi", C.c_double * 3),
                ("r", C.c_int32), ("driver_id", C.c_int32), ("dp", C.c_double * 12),
                ("terminal_id", C.c_int32), ("tp", C.c_double * 12),
                ("picard_max", C.c_int32), ("picard_tol", C.c_double),
                ("bootstrap", C.c_int32), ("bootstrap_substeps", C.c_int32),
                ("smoothing", C.c_int32), ("nthreads", C.c_int32),
                ("sde_id", C.c_int32), ("sp", C.c_double * 12), ("interp", C.c_int32)]


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = C.CDLL(build_oracle())
            D, I, I64 = C.POINTER(C.c_double), C.c_int, C.c_int64
            lib.orc_gauss_hermite.argtypes = [I, D, D]
            lib.orc_gamma.argtypes = [I, I, D]
            lib.orc_balance_npts.argtypes = [C.c_double, C.c_double, I, I, I]
            lib.orc_balance_npts.restype = I64
            lib.orc_spline_moments.argtypes = [D, I64, C.c_double, D]
            lib.orc_spline_eval.argtypes = [D, D, I64, C.c_double, C.c_double, C.c_double]
            lib.orc_spline_eval.restype = C.c_double
            lib.orc_thomas.argtypes = [I64, D, D, D, D, D]
            lib.orc_terminal.argtypes = [C.POINTER(_Cfg), D, D, D]
            lib.orc_exact.argtypes = [C.POINTER(_Cfg), C.c_double, D, D, D]
            lib.orc_driver.argtypes = [C.POINTER(_Cfg), C.c_double, C.c_double, D]
            lib.orc_driver.restype = C.c_double
            lib.orc_fd_weights.argtypes = [C.POINTER(C.c_int), D]
            lib.orc_fd_deriv.argtypes = [D, I64, C.c_double, D]
            lib.orc_create.argtypes = [C.POINTER(_Cfg), C.POINTER(C.c_void_p)]
            lib.orc_step.argtypes = [C.c_void_p]
            lib.orc_solve.argtypes = [C.c_void_p, D, D]
            lib.orc_level.argtypes = [C.c_void_p]
            lib.orc_get_layer.argtypes = [C.c_void_p, I, D, I64]
            lib.orc_get_picard_counts.argtypes = [C.c_void_p, C.POINTER(C.c_int32), I64]
            lib.orc_query_grid.argtypes = [C.c_void_p, C.POINTER(C.c_int64), D]
            lib.orc_step_points.argtypes = [C.c_void_p, I64, C.POINTER(C.c_int64), D, C.POINTER(C.c_int32)]
            lib.orc_eval_newest.argtypes = [C.c_void_p, D, D]
            lib.orc_destroy.argtypes = [C.c_void_p]
            lib.orc_destroy.restype = None
            lib.orc_last_error.restype = C.c_char_p
            _lib = lib
    return _lib


def _check(code):
    if code != 0:
        raise OracleError(code, _load().orc_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def make_cfg(spec: dict, nthreads: int = 0) -> _Cfg:
    c = _Cfg()
    d = int(spec["d"])
    c.d = d
    c.t0 = float(spec.get("t0", 0.0))
    c.T = float(spec["T"])
    c.N = int(spec["N"])
    c.Ky = int(spec["Ky"])
    c.Kz = int(spec["Kz"])
    c.L = int(spec["L"])
    npts = list(spec.get("npts", [0, 0, 0])) + [0, 0, 0]
    xlo = list(spec["xlo"]) + [0.0, 0.0, 0.0]
    xhi = list(spec["xhi"]) + [0.0, 0.0, 0.0]
    for a in range(3):
        c.npts[a] = int(npts[a]) if a < d else 1
        c.xlo[a] = float(xlo[a])
        c.xhi[a] = float(xhi[a])
    c.r = int(spec.get("r", 4))
    c.driver_id = DRIVERS[spec["driver"]]
    c.terminal_id = TERMINALS[spec["terminal"]]
    dp = list(spec.get("driver_params", [])) + [0.0] * 12
    tp = list(spec.get("terminal_params", [])) + [0.0] * 12
    for k in range(12):
        c.dp[k] = float(dp[k])
        c.tp[k] = float(tp[k])
    c.picard_max = int(spec.get("picard_max", 30))
    c.picard_tol = float(spec.get("picard_tol", 0.0))
    c.bootstrap = int(spec.get("bootstrap", 0))
    c.bootstrap_substeps = int(spec.get("bootstrap_substeps", 1))
    c.smoothing = int(spec.get("smoothing", 0))
    c.nthreads = int(nthreads)
    c.sde_id = SDES[spec.get("sde", "brownian")]
    sp = list(spec.get("sde_params", [])) + [0.0] * 12
    for k in range(12):
        c.sp[k] = float(sp[k])
    c.interp = INTERPS[spec.get("interp", "spline")]
    return c


# ---------------------------------------------------------------- building blocks
def gauss_hermite(L: int):
    a = np.zeros(L)
    w = np.zeros(L)
    _check(_load().orc_gauss_hermite(L, _dp(a), _dp(w)))
    return a, w


def gamma_row(K: int, which: str):
    g = np.zeros(K + 1)
    _check(_load().orc_gamma(K, 0 if which == "y" else 1, _dp(g)))
    return g


def balance_npts(width, dt, Ky, Kz, r=4) -> int:
    return int(_load().orc_balance_npts(float(width), float(dt), Ky, Kz, r))


def spline_moments(F, dx):
    F = np.ascontiguousarray(F, dtype=np.float64)
    M = np.zeros_like(F)
    _check(_load().orc_spline_moments(_dp(F), len(F), float(dx), _dp(M)))
    return M


def spline_eval(F, M, xlo, dx, X):
    F = np.ascontiguousarray(F, dtype=np.float64)
    M = np.ascontiguousarray(M, dtype=np.float64)
    lib = _load()
    return np.array([lib.orc_spline_eval(_dp(F), _dp(M), len(F), float(xlo), float(dx), float(x))
                     for x in np.atleast_1d(X)])


def thomas(a, b, c, r):
    a, b, c, r = (np.ascontiguousarray(v, dtype=np.float64) for v in (a, b, c, r))
    x = np.zeros_like(r)
    _check(_load().orc_thomas(len(r), _dp(a), _dp(b), _dp(c), _dp(r), _dp(x)))
    return x


def fd_weights(offsets):
    off = (C.c_int * 5)(*[int(o) for o in offsets])
    w = np.zeros(5)
    _check(_load().orc_fd_weights(off, _dp(w)))
    return w


def fd_deriv(f, h):
    f = np.ascontiguousarray(f, dtype=np.float64)
    df = np.zeros_like(f)
    _check(_load().orc_fd_deriv(_dp(f), len(f), float(h), _dp(df)))
    return df


def terminal(spec, w):
    cfg = make_cfg(spec)
    w = np.ascontiguousarray(np.atleast_1d(w), dtype=np.float64)
    y = np.zeros(1)
    z = np.zeros(3)
    _check(_load().orc_terminal(C.byref(cfg), _dp(w), _dp(y), _dp(z)))
    return y[0], z[:cfg.d].copy()


def exact(spec, t, w):
    cfg = make_cfg(spec)
    w = np.ascontiguousarray(np.atleast_1d(w), dtype=np.float64)
    y = np.zeros(1)
    z = np.zeros(3)
    _check(_load().orc_exact(C.byref(cfg), float(t), _dp(w), _dp(y), _dp(z)))
    return y[0], z[:cfg.d].copy()


def driver(spec, t, y, z):
    cfg = make_cfg(spec)
    z = np.ascontiguousarray(list(np.atleast_1d(z)) + [0.0] * 3, dtype=np.float64)
    return _load().orc_driver(C.byref(cfg), float(t), float(y), _dp(z))


# ---------------------------------------------------------------- the solver
class Oracle:
    """Full backward solve on the CPU (Eq. 20 with Eq. 21 expectations)."""

    def __init__(self, spec: dict, nthreads: int = 0):
        self.spec = dict(spec)
        self.cfg = make_cfg(spec, nthreads)
        self._lib = _load()
        h = C.c_void_p()
        _check(self._lib.orc_create(C.byref(self.cfg), C.byref(h)))
        self._h = h
        n = (C.c_int64 * 3)()
        dx = (C.c_double * 3)()
        self._lib.orc_query_grid(h, n, dx)
        self.d = self.cfg.d
        self.shape = tuple(int(n[a]) for a in range(self.d))
        self.dx = tuple(float(dx[a]) for a in range(self.d))
        self.npts = int(np.prod(self.shape))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.orc_destroy(self._h)
            self._h = None

    __del__ = close

    @property
    def level(self) -> int:
        return int(self._lib.orc_level(self._h))

    def step(self):
        _check(self._lib.orc_step(self._h))

    def solve(self):
        y0 = np.zeros(1)
        z0 = np.zeros(3)
        _check(self._lib.orc_solve(self._h, _dp(y0), _dp(z0)))
        return float(y0[0]), z0[:self.d].copy()

    def layer(self, field: int = 0) -> np.ndarray:
        out = np.zeros(self.npts)
        _check(self._lib.orc_get_layer(self._h, field, _dp(out), self.npts))
        return out.reshape(self.shape)

    def layers(self) -> np.ndarray:
        return np.stack([self.layer(f) for f in range(1 + self.d)])

    def picard_counts(self) -> np.ndarray:
        out = np.zeros(self.npts, dtype=np.int32)
        _check(self._lib.orc_get_picard_counts(self._h, out.ctypes.data_as(C.POINTER(C.c_int32)), self.npts))
        return out.reshape(self.shape)

    def step_points(self, idx):
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.zeros((1 + self.d) * len(idx))
        pic = np.zeros(len(idx), dtype=np.int32)
        _check(self._lib.orc_step_points(self._h, len(idx), idx.ctypes.data_as(C.POINTER(C.c_int64)),
                                         _dp(out), pic.ctypes.data_as(C.POINTER(C.c_int32))))
        return out.reshape(1 + self.d, len(idx)), pic

    def eval_newest(self, x):
        x = np.ascontiguousarray(list(np.atleast_1d(x)) + [0.0] * 3, dtype=np.float64)
        out = np.zeros(4)
        _check(self._lib.orc_eval_newest(self._h, _dp(x), _dp(out)))
        return out[:1 + self.d]
