"""Thin Python binding of the C ABI in include/bsde.h (argument marshalling only).

Every step of the method runs in the CUDA kernels of libbsde_b200.so; this module
never computes anything of the scheme and has no CPU fallback: it raises if the
library is missing or no CUDA device is present.  PyTorch is used only for the
optional caller-owned device workspace and the CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbsde_b200.so")

BSDE_OK = 0
STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "RESOURCE_LIMIT", 3: "SINGULAR", 4: "NUMERICAL_DOMAIN",
          5: "CUDA", 6: "COMM", 7: "STATE"}
DRIVERS = {"zero": 0, "affine": 1, "ex1": 2, "ex2": 3, "diff_rates": 4}
TERMINALS = {"const": 0, "poly": 1, "logistic": 2, "ex2": 3, "call_w": 4, "sin_sum": 5,
             "exchange_w": 6, "geo_basket_w": 7, "call_x": 8}
SDES = {"brownian": 0, "gbm": 1, "ou": 2}
INTERPS = {"spline": 0, "fd_bicubic": 1}

# every symbol include/bsde.h declares
EXPORTS = ["bsde_query_workspace", "bsde_setup", "bsde_step", "bsde_solve", "bsde_level", "bsde_get_layer",
           "bsde_get_picard_counts", "bsde_query_grid", "bsde_query_taps", "bsde_eval", "bsde_layer_device_ptr",
           "bsde_query_partition", "bsde_query_partition_cfg", "bsde_nccl_unique_id", "bsde_group_step",
           "bsde_group_solve", "bsde_solve_batch", "bsde_solve_batch_mode", "bsde_kernel_launches",
           "bsde_measure_fp64_peak",
           "bsde_last_error", "bsde_destroy"]


class BsdeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"bsde {STATUS.get(code, code)}: {msg}")
        self.code = code


class bsde_config(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("d", C.c_int32), ("m", C.c_int32),
                ("t0", C.c_double), ("T", C.c_double), ("N", C.c_int32),
                ("Ky", C.c_int32), ("Kz", C.c_int32), ("L", C.c_int32),
                ("npts", C.c_int64 * 3), ("xlo", C.c_double * 3), ("xhi", C.c_double * 3),
                ("r", C.c_int32), ("driver_id", C.c_int32), ("driver_params", C.c_double * 12),
                ("terminal_id", C.c_int32), ("terminal_params", C.c_double * 12),
                ("picard_max", C.c_int32), ("picard_tol", C.c_double),
                ("bootstrap", C.c_int32), ("bootstrap_substeps", C.c_int32), ("smoothing", C.c_int32),
                ("nranks", C.c_int32), ("rank", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("stream", C.c_void_p), ("device", C.c_int32), ("kernel_variant", C.c_int32),
                ("interp", C.c_int32), ("sde_id", C.c_int32), ("sde_params", C.c_double * 12),
                ("timing", C.c_int32), ("slab_spline", C.c_int32)]


class bsde_result(C.Structure):
    _fields_ = [("y0", C.c_double), ("z0", C.c_double * 3), ("t_setup_s", C.c_double),
                ("t_sweep_s", C.c_double), ("t_total_s", C.c_double), ("updates", C.c_int64),
                ("picard_max_used", C.c_int32), ("t_bootstrap_s", C.c_double), ("t_spline_s", C.c_double),
                ("t_quad_s", C.c_double), ("t_comm_s", C.c_double), ("picard_iters", C.c_int64),
                ("batch_ctas", C.c_int32), ("batch_tiles", C.c_int32)]


_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH):
    """Load libbsde_b200.so (fails loudly if it has not been built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise BsdeError(-1, f"{path} not built: run `python -m paper_1909_13560_b200.build`")
            lib = C.CDLL(path)
            P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)
            lib.bsde_query_workspace.argtypes = [C.POINTER(bsde_config), C.POINTER(C.c_size_t)]
            lib.bsde_setup.argtypes = [C.POINTER(bsde_config), P, C.c_size_t, C.POINTER(P)]
            lib.bsde_step.argtypes = [P]
            lib.bsde_solve.argtypes = [P, C.POINTER(bsde_result)]
            lib.bsde_level.argtypes = [P, C.POINTER(I32)]
            lib.bsde_get_layer.argtypes = [P, I32, D, I64]
            lib.bsde_get_picard_counts.argtypes = [P, C.POINTER(I32), I64]
            lib.bsde_query_grid.argtypes = [P, C.POINTER(I64), D]
            lib.bsde_query_taps.argtypes = [P, I32, I32, C.POINTER(I32), D, D, D]
            lib.bsde_eval.argtypes = [P, D, D]
            lib.bsde_layer_device_ptr.argtypes = [P, I32, C.POINTER(C.c_void_p)]
            lib.bsde_kernel_launches.argtypes = [P, C.POINTER(I64)]
            lib.bsde_query_partition.argtypes = [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)]
            lib.bsde_query_partition_cfg.argtypes = [C.POINTER(bsde_config), C.POINTER(I64)]
            lib.bsde_nccl_unique_id.argtypes = [C.c_void_p, C.c_size_t]
            lib.bsde_group_step.argtypes = [C.POINTER(C.c_void_p), I32]
            lib.bsde_group_solve.argtypes = [C.POINTER(C.c_void_p), I32, C.POINTER(bsde_result)]
            lib.bsde_solve_batch.argtypes = [C.POINTER(C.c_void_p), I32, C.POINTER(bsde_result)]
            lib.bsde_solve_batch_mode.argtypes = [C.POINTER(C.c_void_p), I32, I32, C.POINTER(bsde_result)]
            lib.bsde_measure_fp64_peak.argtypes = [I32, I32, D, D]
            lib.bsde_last_error.argtypes = [P]
            lib.bsde_last_error.restype = C.c_char_p
            lib.bsde_destroy.argtypes = [P]
            lib.bsde_destroy.restype = None
            for name in EXPORTS:
                if name not in ("bsde_last_error", "bsde_destroy"):
                    getattr(lib, name).restype = C.c_int
            _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def make_config(spec: dict, device: int = 0, stream: int | None = None, kernel_variant: int = 0,
                nranks: int = 1, rank: int = 0, nccl_id=None, timing: int = 0) -> bsde_config:
    c = bsde_config()
    c.struct_size = C.sizeof(bsde_config)
    d = int(spec["d"])
    c.d, c.m = d, 1
    c.t0, c.T, c.N = float(spec.get("t0", 0.0)), float(spec["T"]), int(spec["N"])
    c.Ky, c.Kz, c.L = int(spec["Ky"]), int(spec["Kz"]), int(spec["L"])
    npts = list(spec.get("npts", [0] * d)) + [0, 0, 0]
    xlo = list(spec["xlo"]) + [0.0] * 3
    xhi = list(spec["xhi"]) + [0.0] * 3
    for a in range(3):
        c.npts[a] = int(npts[a]) if a < d else 1
        c.xlo[a], c.xhi[a] = float(xlo[a]), float(xhi[a])
    c.r = int(spec.get("r", 4))
    c.driver_id = DRIVERS[spec["driver"]]
    c.terminal_id = TERMINALS[spec["terminal"]]
    dp = list(spec.get("driver_params", [])) + [0.0] * 12
    tp = list(spec.get("terminal_params", [])) + [0.0] * 12
    for k in range(12):
        c.driver_params[k] = float(dp[k])
        c.terminal_params[k] = float(tp[k])
    c.picard_max = int(spec.get("picard_max", 30))
    c.picard_tol = float(spec.get("picard_tol", 0.0))
    c.bootstrap = int(spec.get("bootstrap", 0))
    c.bootstrap_substeps = int(spec.get("bootstrap_substeps", 1))
    c.smoothing = int(spec.get("smoothing", 0))
    c.nranks, c.rank = int(nranks), int(rank)
    c.nccl_unique_id = C.cast(nccl_id, C.c_void_p) if nccl_id is not None else None
    c.stream = stream
    c.device = int(device)
    c.kernel_variant = int(kernel_variant)
    c.interp = INTERPS[spec.get("interp", "spline")]
    c.sde_id = SDES[spec.get("sde", "brownian")]
    sp = list(spec.get("sde_params", [])) + [0.0] * 12
    for k in range(12):
        c.sde_params[k] = float(sp[k])
    c.timing = int(timing)
    c.slab_spline = int(spec.get("slab_spline", 0))
    return c


def measure_fp64_peak(device: int = 0, iters: int = 200000) -> dict:
    """Measured FP64 DFMA throughput of `device` (bsde_measure_fp64_peak)."""
    lib = load_library()
    tf, ms = C.c_double(), C.c_double()
    st = lib.bsde_measure_fp64_peak(int(device), int(iters), C.byref(tf), C.byref(ms))
    if st:
        raise BsdeError(st, lib.bsde_last_error(None).decode())
    return {"tflops": tf.value, "ms": ms.value}


def query_workspace(spec: dict, kernel_variant: int = 0) -> int:
    lib = load_library()
    cfg = make_config(spec, kernel_variant=kernel_variant)
    n = C.c_size_t()
    st = lib.bsde_query_workspace(C.byref(cfg), C.byref(n))
    if st != BSDE_OK:
        raise BsdeError(st, lib.bsde_last_error(None).decode())
    return int(n.value)


def query_partition(spec: dict, nranks: int, rank: int) -> dict:
    """Host-only: the slab (global axis-0 rows) a rank would own (bsde_query_partition_cfg)."""
    lib = load_library()
    cfg = make_config(spec, nranks=nranks, rank=rank)
    out = (C.c_int64 * 5)()
    st = lib.bsde_query_partition_cfg(C.byref(cfg), out)
    if st != BSDE_OK:
        raise BsdeError(st, lib.bsde_last_error(None).decode())
    return dict(own_lo=out[0], own_hi=out[1], halo=out[2], slab_lo=out[3], slab_hi=out[4])


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = C.create_string_buffer(128)
    st = lib.bsde_nccl_unique_id(buf, 128)
    if st != BSDE_OK:
        raise BsdeError(st, lib.bsde_last_error(None).decode())
    return buf.raw


class Solver:
    """One bsde_ctx: ``bsde_setup`` on construction, ``bsde_destroy`` on close.  With
    ``nranks > 1`` the context holds the slab of ``rank`` (d >= 2); ``nccl_id`` (128 bytes)
    selects the multi-process NCCL mode, None an in-process group (see ``GroupSolver``)."""

    def __init__(self, spec: dict, device: int = 0, stream: int | None = None, workspace=None,
                 kernel_variant: int = 0, nranks: int = 1, rank: int = 0, nccl_id: bytes | None = None,
                 timing: int = 0):
        self._lib = load_library()
        self.spec = dict(spec)
        self._id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        self.cfg = make_config(spec, device, stream, kernel_variant, nranks, rank, self._id, timing)
        h = C.c_void_p()
        ptr, nbytes = None, 0
        if workspace is not None:          # caller-owned device memory (e.g. a torch uint8 tensor)
            ptr, nbytes = C.c_void_p(workspace.data_ptr()), workspace.numel() * workspace.element_size()
            self._ws = workspace
        st = self._lib.bsde_setup(C.byref(self.cfg), ptr, nbytes, C.byref(h))
        if st != BSDE_OK:
            raise BsdeError(st, self._lib.bsde_last_error(None).decode())
        self._h = h
        n = (C.c_int64 * 3)()
        dx = (C.c_double * 3)()
        self._call(self._lib.bsde_query_grid(h, n, dx))
        self.d = int(spec["d"])
        self.global_shape = tuple(int(n[a]) for a in range(self.d))
        self.dx = tuple(float(dx[a]) for a in range(self.d))
        lo, hi, halo = C.c_int64(), C.c_int64(), C.c_int64()
        self._call(self._lib.bsde_query_partition(h, C.byref(lo), C.byref(hi), C.byref(halo)))
        self.own = (int(lo.value), int(hi.value))
        self.halo = int(halo.value)
        self.shape = (self.own[1] - self.own[0],) + self.global_shape[1:]     # owned part
        self.npts = int(np.prod(self.shape))

    def _call(self, st):
        if st != BSDE_OK:
            raise BsdeError(st, self._lib.bsde_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.bsde_destroy(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def level(self) -> int:
        n = C.c_int32()
        self._call(self._lib.bsde_level(self._h, C.byref(n)))
        return n.value

    def step(self):
        self._call(self._lib.bsde_step(self._h))

    def solve(self) -> bsde_result:
        r = bsde_result()
        self._call(self._lib.bsde_solve(self._h, C.byref(r)))
        return r

    def layer(self, field: int = 0, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.npts, dtype=np.float64)
        self._call(self._lib.bsde_get_layer(self._h, field, _dp(out), self.npts))
        return out.reshape(self.shape)

    def layers(self) -> np.ndarray:
        return np.stack([self.layer(f) for f in range(1 + self.d)])

    def picard_counts(self) -> np.ndarray:
        out = np.empty(self.npts, dtype=np.int32)
        self._call(self._lib.bsde_get_picard_counts(self._h, out.ctypes.data_as(C.POINTER(C.c_int32)), self.npts))
        return out.reshape(self.shape)

    def taps(self, level: int, axis: int = 0):
        L = int(self.spec["L"])
        q = np.empty(L, dtype=np.int32)
        b = np.empty(4 * L)
        w = np.empty(L)
        s = np.empty(L)
        self._call(self._lib.bsde_query_taps(self._h, level, axis, q.ctypes.data_as(C.POINTER(C.c_int32)),
                                             _dp(b), _dp(w), _dp(s)))
        return q, b.reshape(L, 4), w, s

    def eval(self, x) -> np.ndarray:
        x = np.ascontiguousarray(list(np.atleast_1d(x)) + [0.0] * 3, dtype=np.float64)
        out = np.empty(4)
        self._call(self._lib.bsde_eval(self._h, _dp(x), _dp(out)))
        return out[:1 + self.d]

    def layer_device_ptr(self, field: int = 0) -> int:
        p = C.c_void_p()
        self._call(self._lib.bsde_layer_device_ptr(self._h, field, C.byref(p)))
        return int(p.value)

    def partition(self) -> dict:
        return dict(own_lo=self.own[0], own_hi=self.own[1], halo=self.halo)

    @property
    def kernel_launches(self) -> int:
        n = C.c_int64()
        self._call(self._lib.bsde_kernel_launches(self._h, C.byref(n)))
        return int(n.value)


def solve_batch(solvers, mode: int = 0) -> list:
    """``bsde_solve_batch_mode``: the remaining steps of several independent d = 1 Solvers (same
    grid, driver and device) in one persistent launch; mode 0 auto, 1 round robin, 2
    problem-partitioned CTAs."""
    lib = load_library()
    n = len(solvers)
    arr = (C.c_void_p * n)(*[s._h for s in solvers])
    res = (bsde_result * n)()
    st = lib.bsde_solve_batch_mode(arr, n, int(mode), res)
    if st != BSDE_OK:
        raise BsdeError(st, lib.bsde_last_error(None).decode() or
                        " | ".join(lib.bsde_last_error(s._h).decode() for s in solvers))
    return list(res)


class GroupSolver:
    """In-process slab group: ``nranks`` contexts (ranks 0..n-1) of one d >= 2 problem,
    optionally on one GPU, stepped together (bsde_group_step / bsde_group_solve)."""

    def __init__(self, spec: dict, nranks: int, devices=None, kernel_variant: int = 0):
        devices = devices or [0] * nranks
        self.ranks = [Solver(spec, device=devices[r], kernel_variant=kernel_variant, nranks=nranks, rank=r)
                      for r in range(nranks)]
        self._lib = load_library()
        self._arr = (C.c_void_p * nranks)(*[s._h for s in self.ranks])

    def _call(self, st):
        if st != BSDE_OK:
            raise BsdeError(st, self._lib.bsde_last_error(None).decode() or
                            " | ".join(self._lib.bsde_last_error(s._h).decode() for s in self.ranks))

    @property
    def level(self) -> int:
        return self.ranks[0].level

    def step(self):
        self._call(self._lib.bsde_group_step(self._arr, len(self.ranks)))

    def solve(self) -> bsde_result:
        r = bsde_result()
        self._call(self._lib.bsde_group_solve(self._arr, len(self.ranks), C.byref(r)))
        return r

    def layer(self, field: int = 0) -> np.ndarray:
        return np.concatenate([s.layer(field) for s in self.ranks], axis=0)

    def layers(self) -> np.ndarray:
        return np.stack([self.layer(f) for f in range(1 + self.ranks[0].d)])

    def picard_counts(self) -> np.ndarray:
        return np.concatenate([s.picard_counts() for s in self.ranks], axis=0)

    def close(self):
        for s in self.ranks:
            s.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
