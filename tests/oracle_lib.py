"""TEST INFRASTRUCTURE — ctypes access to the CPU oracle and the reference build.

``Oracle`` wraps oracle/liboracle.so (the CPU restatement, npsd_oracle.hpp).
``Ref`` wraps oracle/_ref/libnpsd_ref.so (the unmodified reference sources plus
oracle/ref_shim.cpp). Both are checkers only: the product (paper_2310_00177_b200)
never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libnpsd_ref.so"

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")

STATUS_EXC = {1: ValueError, 2: RuntimeError, 3: RuntimeError, 4: RuntimeError}


def build_oracle() -> None:
    """Compile the checker (make -C oracle); the reference part only where its sources exist."""
    import subprocess

    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)


def _load(path: Path) -> C.CDLL:
    if not path.exists():
        build_oracle()
    return C.CDLL(str(path))


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"status {status}: {msg}")
        self.status = status


def slots(dim: int) -> int:
    return 27 if dim == 3 else 9


class Oracle:
    """The CPU restatement (npsd_oracle.hpp)."""

    def __init__(self) -> None:
        L = self.lib = _load(ORACLE_SO)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_param_count.restype = C.c_long
        L.oracle_param_count.argtypes = [C.c_int, C.c_int]
        L.oracle_init_params.argtypes = [C.c_int, C.c_int, C.c_ulonglong, _f32p]
        L.oracle_identity_params.argtypes = [C.c_int, C.c_int, _f32p]
        L.oracle_rhs_normal.argtypes = [C.c_ulonglong, C.c_long, _f64p]
        L.oracle_level_images.argtypes = [C.c_int, C.c_long, C.c_long, C.c_long, C.c_int, _u8p, _f32p]
        L.oracle_ctx_create.argtypes = [C.c_int, C.c_long, C.c_long, C.c_long, C.c_int, _f32p, C.c_long, _u8p,
                                        C.POINTER(C.c_void_p)]
        L.oracle_ctx_destroy.argtypes = [C.c_void_p]
        L.oracle_ctx_n_fluid.restype = C.c_long
        L.oracle_ctx_n_fluid.argtypes = [C.c_void_p]
        L.oracle_ctx_build_seconds.restype = C.c_double
        L.oracle_ctx_build_seconds.argtypes = [C.c_void_p]
        L.oracle_ctx_fluid_indices.argtypes = [C.c_void_p, _i64p]
        L.oracle_ctx_z.argtypes = [C.c_void_p, _f32p, _f32p]
        L.oracle_ctx_net_apply.argtypes = [C.c_void_p, _f32p, _f32p]
        L.oracle_ctx_precond_apply.argtypes = [C.c_void_p, _f64p, _f64p]
        L.oracle_ctx_spmv.argtypes = [C.c_void_p, _f64p, _f64p]
        L.oracle_spmv.argtypes = [C.c_int, C.c_long, C.c_long, C.c_long, _u8p, _f64p, _f64p]
        L.oracle_mac_rhs.argtypes = [C.c_int, C.c_long, C.c_long, C.c_long, _u8p, _f64p, _f64p, C.c_void_p,
                                     C.c_double, C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, _f64p]
        L.oracle_ctx_psdo_solve.argtypes = [C.c_void_p, C.c_int, _f64p, C.c_void_p, C.c_double, C.c_double,
                                            C.c_long, C.c_int, C.c_int, C.c_int, _f64p, _f64p,
                                            C.POINTER(C.c_long), C.POINTER(C.c_int), C.POINTER(C.c_long),
                                            C.POINTER(C.c_double)]

    def _check(self, st: int) -> None:
        if st != 0:
            raise OracleError(st, self.lib.oracle_last_error().decode())

    def param_count(self, dim: int, depth: int) -> int:
        return int(self.lib.oracle_param_count(dim, depth))

    def init_params(self, dim: int, depth: int, seed: int) -> np.ndarray:
        out = np.empty(self.param_count(dim, depth), np.float32)
        self._check(self.lib.oracle_init_params(dim, depth, seed, out))
        return out

    def identity_params(self, dim: int, depth: int) -> np.ndarray:
        out = np.empty(self.param_count(dim, depth), np.float32)
        self._check(self.lib.oracle_identity_params(dim, depth, out))
        return out

    def rhs_normal(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.oracle_rhs_normal(seed, n, out)
        return out

    def level_images(self, types: np.ndarray, depth: int) -> list[np.ndarray]:
        dim, (nx, ny, nz) = _dims_of(types)
        sizes = []
        for l in range(depth):
            sizes.append((nx >> l) * (ny >> l) * ((nz >> l) if dim == 3 else 1))
        out = np.empty(3 * sum(sizes), np.float32)
        self._check(self.lib.oracle_level_images(dim, nx, ny, nz, depth, _u8(types), out))
        res, o = [], 0
        for l, s in enumerate(sizes):
            shp = (3, (nz >> l), (ny >> l), (nx >> l)) if dim == 3 else (3, ny >> l, nx >> l)
            res.append(out[o:o + 3 * s].reshape(shp))
            o += 3 * s
        return res

    def mac_rhs(self, types, u, v, w=None, h=1.0, dt=0.05, rho=1.0, bc=None) -> np.ndarray:
        """mac_divergence_rhs restated (full grid, zeros off fluid); bc = (bu, bv[, bw]) or None."""
        dim, (nx, ny, nz) = _dims_of(types)
        out = np.empty(types.size, np.float64)
        bc = list(bc or []) + [None] * (3 - len(bc or []))
        opt = [None if a is None else np.ascontiguousarray(a, np.float64) for a in (w, *bc)]
        ptr = [None if a is None else a.ctypes.data_as(C.c_void_p) for a in opt]
        self._check(self.lib.oracle_mac_rhs(dim, nx, ny, nz, _u8(types), np.ascontiguousarray(u, np.float64),
                                            np.ascontiguousarray(v, np.float64), ptr[0], h, dt, rho, ptr[1], ptr[2],
                                            ptr[3], out))
        return out

    def spmv(self, types: np.ndarray, x: np.ndarray) -> np.ndarray:
        """A x (reduced system of `types`), matrix-free, no network context."""
        dim, (nx, ny, nz) = _dims_of(types)
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        self._check(self.lib.oracle_spmv(dim, nx, ny, nz, _u8(types), x, y))
        return y

    def context(self, types: np.ndarray, params: np.ndarray, depth: int) -> "OracleCtx":
        return OracleCtx(self, types, params, depth)


def _u8(types: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(types, dtype=np.uint8).reshape(-1)


def _dims_of(types: np.ndarray) -> tuple[int, tuple[int, int, int]]:
    if types.ndim == 3:
        nz, ny, nx = types.shape
        return 3, (nx, ny, nz)
    ny, nx = types.shape
    return 2, (nx, ny, 1)


class OracleCtx:
    def __init__(self, o: Oracle, types: np.ndarray, params: np.ndarray, depth: int) -> None:
        self.o, self.lib = o, o.lib
        self.dim, (self.nx, self.ny, self.nz) = _dims_of(types)
        self.depth = depth
        self.shape = types.shape
        h = C.c_void_p()
        o._check(self.lib.oracle_ctx_create(self.dim, self.nx, self.ny, self.nz, depth,
                                            np.ascontiguousarray(params, np.float32), len(params), _u8(types),
                                            C.byref(h)))
        self.h = h
        self.n_fluid = int(self.lib.oracle_ctx_n_fluid(h))
        self.build_seconds = float(self.lib.oracle_ctx_build_seconds(h))

    def __del__(self) -> None:
        if getattr(self, "h", None):
            self.lib.oracle_ctx_destroy(self.h)
            self.h = None

    def fluid_indices(self) -> np.ndarray:
        out = np.empty(self.n_fluid, np.int64)
        self.lib.oracle_ctx_fluid_indices(self.h, out)
        return out

    def z(self) -> tuple[np.ndarray, np.ndarray]:
        za = np.zeros(max(self.depth - 1, 1), np.float32)
        zb = np.zeros_like(za)
        self.lib.oracle_ctx_z(self.h, za, zb)
        return za[: self.depth - 1], zb[: self.depth - 1]

    def net_apply(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32).reshape(-1)
        y = np.empty_like(x)
        self.o._check(self.lib.oracle_ctx_net_apply(self.h, x, y))
        return y.reshape(self.shape)

    def precond_apply(self, r: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty_like(r)
        self.o._check(self.lib.oracle_ctx_precond_apply(self.h, r, z))
        return z

    def spmv(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        self.o._check(self.lib.oracle_ctx_spmv(self.h, x, y))
        return y

    def psdo_solve(self, b: np.ndarray, *, identity: bool = False, x0=None, tol_reduction=1e-6, tol_abs=0.0,
                   max_iters=1000, n_ortho=2, nullspace_projection=False, normalize_before_precond=True) -> dict:
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        hist = np.zeros(max_iters + 1, np.float64)
        it, conv, hl, sec = C.c_long(), C.c_int(), C.c_long(), C.c_double()
        x0p = None
        if x0 is not None:
            x0a = np.ascontiguousarray(x0, np.float64)
            x0p = x0a.ctypes.data_as(C.c_void_p)
        st = self.lib.oracle_ctx_psdo_solve(self.h, int(identity), b, x0p, tol_reduction, tol_abs, max_iters,
                                            n_ortho, int(nullspace_projection), int(normalize_before_precond), x,
                                            hist, C.byref(it), C.byref(conv), C.byref(hl), C.byref(sec))
        self.o._check(st)
        return {"x": x, "iterations": it.value, "converged": bool(conv.value),
                "residual_history": hist[: hl.value].copy(), "seconds": sec.value}


APPLY_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_long)


class Ref:
    """The real reference library (oracle/_ref/libnpsd_ref.so)."""

    def __init__(self) -> None:
        if not REF_SO.exists():
            build_oracle()
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (reference sources absent)")
        L = self.lib = C.CDLL(str(REF_SO))
        L.ref_last_error.restype = C.c_char_p
        L.ref_rhs_normal.argtypes = [C.c_ulonglong, C.c_long, _f64p]
        L.ref_init_params_2d.argtypes = [C.c_int, C.c_ulonglong, _f32p]
        L.ref_save_npm_2d.argtypes = [C.c_int, C.c_ulonglong, C.c_char_p]
        L.ref_bench_roundtrip.argtypes = [C.c_char_p, C.c_char_p]
        L.ref_pcg_solve.argtypes = [C.c_int, C.c_long, C.c_long, C.c_long, _u8p, C.c_int, _f64p, C.c_double, C.c_long,
                                    _f64p, _f64p, C.POINTER(C.c_long), C.POINTER(C.c_int), C.POINTER(C.c_long), C.c_int]
        L.ref_ic0_apply.argtypes = [C.c_int, C.c_long, C.c_long, C.c_long, _u8p, _f64p, _f64p, C.POINTER(C.c_int)]
        L.ref_mac_rhs_2d.argtypes = [C.c_long, C.c_long, _u8p, _f64p, _f64p, C.c_double, C.c_double, C.c_double,
                                     C.c_void_p, C.c_void_p, _f64p]
        L.ref_load_npm_2d.argtypes = [C.c_char_p, _f32p, C.c_long, C.POINTER(C.c_int)]
        L.ref_level_images_2d.argtypes = [C.c_long, C.c_long, C.c_int, _u8p, _f32p]
        L.ref_net_apply_2d.argtypes = [C.c_long, C.c_long, C.c_int, _f32p, C.c_long, _u8p, _f32p, _f32p,
                                       _f32p, _f32p]
        L.ref_precond_apply_2d.argtypes = [C.c_long, C.c_long, C.c_int, _f32p, C.c_long, _u8p, _f64p, _f64p]
        L.ref_backward_2d.argtypes = [C.c_long, C.c_long, C.c_int, _f32p, C.c_long, _u8p, _f64p, C.c_int,
                                      C.POINTER(C.c_double), _f32p]
        L.ref_spmv.argtypes = [C.c_int, C.c_long, C.c_long, C.c_long, _u8p, _f64p, _f64p]
        L.ref_psdo_solve.argtypes = [C.c_int, C.c_long, C.c_long, C.c_long, _u8p, C.c_int, C.c_int, C.c_void_p,
                                     C.c_long, C.c_void_p, C.c_void_p, _f64p, C.c_void_p, C.c_double, C.c_double,
                                     C.c_long, C.c_int, C.c_int, C.c_int, _f64p, _f64p, C.POINTER(C.c_long),
                                     C.POINTER(C.c_int), C.POINTER(C.c_long), _f64p]

    def _check(self, st: int) -> None:
        if st != 0:
            raise OracleError(st, self.lib.ref_last_error().decode())

    def rhs_normal(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.ref_rhs_normal(seed, n, out)
        return out

    def init_params_2d(self, depth: int, seed: int) -> np.ndarray:
        n = (depth - 1) * (2 * 252 + 2 * 28) + 252
        out = np.empty(n, np.float32)
        self._check(self.lib.ref_init_params_2d(depth, seed, out))
        return out

    def pcg_solve(self, types, b, precond=0, tol_reduction=1e-6, max_iters=1000, nullspace_projection=False) -> dict:
        dim, (nx, ny, nz) = _dims_of(types)
        b = np.ascontiguousarray(b, np.float64)
        x, hist = np.empty_like(b), np.zeros(max_iters + 1)
        it, conv, hl = C.c_long(), C.c_int(), C.c_long()
        self._check(self.lib.ref_pcg_solve(dim, nx, ny, nz, _u8(types), precond, b, tol_reduction, max_iters, x, hist,
                                           C.byref(it), C.byref(conv), C.byref(hl), int(nullspace_projection)))
        return {"x": x, "iterations": it.value, "converged": bool(conv.value), "residual_history": hist[:hl.value]}

    def ic0_apply(self, types, r) -> tuple[np.ndarray, int]:
        """Ic0Precond(A).apply(r) on the reference assembly -> (z, shift retries)."""
        dim, (nx, ny, nz) = _dims_of(types)
        r = np.ascontiguousarray(r, np.float64)
        z, ret = np.empty_like(r), C.c_int()
        self._check(self.lib.ref_ic0_apply(dim, nx, ny, nz, _u8(types), r, z, C.byref(ret)))
        return z, ret.value

    def mac_rhs_2d(self, types, u, v, h=1.0, dt=0.05, rho=1.0, bc=None) -> np.ndarray:
        ny, nx = types.shape
        out = np.empty(types.size, np.float64)
        bu, bv = (np.ascontiguousarray(bc[0], np.float64), np.ascontiguousarray(bc[1], np.float64)) if bc else (None, None)
        self._check(self.lib.ref_mac_rhs_2d(nx, ny, _u8(types), np.ascontiguousarray(u, np.float64),
                                            np.ascontiguousarray(v, np.float64), h, dt, rho,
                                            None if bu is None else bu.ctypes.data_as(C.c_void_p),
                                            None if bv is None else bv.ctypes.data_as(C.c_void_p), out))
        return out

    def bench_roundtrip(self, rows_csv, out_dir) -> None:
        self._check(self.lib.ref_bench_roundtrip(str(rows_csv).encode(), str(out_dir).encode()))

    def save_npm_2d(self, depth: int, seed: int, path) -> None:
        self._check(self.lib.ref_save_npm_2d(depth, seed, str(path).encode()))

    def load_npm_2d(self, path, n: int) -> tuple[int, np.ndarray]:
        out = np.zeros(n, np.float32)
        depth = C.c_int(0)
        self._check(self.lib.ref_load_npm_2d(str(path).encode(), out, n, C.byref(depth)))
        return depth.value, out

    def level_images_2d(self, types: np.ndarray, depth: int) -> list[np.ndarray]:
        ny, nx = types.shape
        sizes = [(nx >> l) * (ny >> l) for l in range(depth)]
        out = np.empty(3 * sum(sizes), np.float32)
        self._check(self.lib.ref_level_images_2d(nx, ny, depth, _u8(types), out))
        res, o = [], 0
        for l, s in enumerate(sizes):
            res.append(out[o:o + 3 * s].reshape(3, ny >> l, nx >> l))
            o += 3 * s
        return res

    def net_apply_2d(self, types, params, depth, x):
        ny, nx = types.shape
        x = np.ascontiguousarray(x, np.float32).reshape(-1)
        y = np.empty_like(x)
        za = np.zeros(max(depth - 1, 1), np.float32)
        zb = np.zeros_like(za)
        self._check(self.lib.ref_net_apply_2d(nx, ny, depth, np.ascontiguousarray(params, np.float32),
                                              len(params), _u8(types), x, y, za, zb))
        return y.reshape(types.shape), za[: depth - 1], zb[: depth - 1]

    def precond_apply_2d(self, types, params, depth, r):
        ny, nx = types.shape
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty_like(r)
        self._check(self.lib.ref_precond_apply_2d(nx, ny, depth, np.ascontiguousarray(params, np.float32),
                                                  len(params), _u8(types), r, z))
        return z

    def backward_2d(self, types, params, depth, rhs):
        """backward_batch<float> (train.hpp:94-150): (mean batch loss, gradient
        in for_each_span order) for reduced right-hand sides rhs (nb, n_f)."""
        ny, nx = types.shape
        params = np.ascontiguousarray(params, np.float32)
        rhs = np.ascontiguousarray(rhs, np.float64)
        loss = C.c_double()
        grads = np.zeros_like(params)
        self._check(self.lib.ref_backward_2d(nx, ny, depth, params, params.size, _u8(types), rhs.reshape(-1),
                                             rhs.shape[0], C.byref(loss), grads))
        return loss.value, grads

    def spmv(self, types, x):
        dim, (nx, ny, nz) = _dims_of(types)
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        self._check(self.lib.ref_spmv(dim, nx, ny, nz, _u8(types), x, y))
        return y

    def psdo_solve(self, types, b, *, mode="identity", params=None, depth=1, callback=None, x0=None,
                   tol_reduction=1e-6, tol_abs=0.0, max_iters=1000, n_ortho=2, nullspace_projection=False,
                   normalize_before_precond=True) -> dict:
        """mode: 'identity' | 'neural' (2D reference NeuralPrecond / 3D restatement) | 'callback'."""
        dim, (nx, ny, nz) = _dims_of(types)
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        hist = np.zeros(max_iters + 1, np.float64)
        secs = np.zeros(2, np.float64)
        it, conv, hl = C.c_long(), C.c_int(), C.c_long()
        m = {"identity": 0, "neural": 1, "callback": 2}[mode]
        pp = None
        if params is not None:
            params = np.ascontiguousarray(params, np.float32)
            pp = params.ctypes.data_as(C.c_void_p)
        cb = APPLY_CB(callback) if callback is not None else None
        x0p = None
        if x0 is not None:
            x0a = np.ascontiguousarray(x0, np.float64)
            x0p = x0a.ctypes.data_as(C.c_void_p)
        st = self.lib.ref_psdo_solve(dim, nx, ny, nz, _u8(types), m, depth, pp,
                                     0 if params is None else len(params),
                                     C.cast(cb, C.c_void_p) if cb is not None else None, None, b, x0p,
                                     tol_reduction, tol_abs, max_iters, n_ortho, int(nullspace_projection),
                                     int(normalize_before_precond), x, hist, C.byref(it), C.byref(conv),
                                     C.byref(hl), secs)
        self._check(st)
        return {"x": x, "iterations": it.value, "converged": bool(conv.value),
                "residual_history": hist[: hl.value].copy(), "setup_seconds": secs[0], "solve_seconds": secs[1]}


def reduced_csr(types: np.ndarray):
    """assemble_poisson_3d + reduce (discretization.cpp:75-160) restated in
    numpy: rows in ascending fluid order, columns ascending (lower
    neighbours, the diagonal when non-zero, upper neighbours), -1 per fluid
    neighbour, diagonal = number of non-solid face neighbours (outside solid)."""
    nz, ny, nx = types.shape
    pad = np.full((nz + 2, ny + 2, nx + 2), 2, np.uint8)
    pad[1:-1, 1:-1, 1:-1] = types
    fl = types.reshape(-1) == 0
    red = np.full(types.size, -1, np.int64)
    red[fl] = np.arange(int(fl.sum()))
    z, y, x = np.nonzero(types == 0)
    offs = [(-1, 0, 0), (0, -1, 0), (0, 0, -1), (0, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0)]
    diag = np.zeros(z.size, np.int64)
    for dz, dy, dx in offs:
        if (dz, dy, dx) != (0, 0, 0):
            diag += pad[z + 1 + dz, y + 1 + dy, x + 1 + dx] != 2
    cols, vals, valid = [], [], []
    for dz, dy, dx in offs:
        if (dz, dy, dx) == (0, 0, 0):
            cols.append(red[(z * ny + y) * nx + x])
            vals.append(diag.astype(np.float64))
            valid.append(diag > 0)
        else:
            t = pad[z + 1 + dz, y + 1 + dy, x + 1 + dx]
            ok = t == 0
            q = ((z + dz) * ny + (y + dy)) * nx + (x + dx)
            cols.append(np.where(ok, red[np.clip(q, 0, types.size - 1)], -1))
            vals.append(np.full(z.size, -1.0))
            valid.append(ok)
    cols, vals, valid = np.stack(cols, 1), np.stack(vals, 1), np.stack(valid, 1)
    ro = np.concatenate([[0], np.cumsum(valid.sum(1))]).astype(np.int64)
    return ro, cols[valid].astype(np.int64), vals[valid]


def have_ref() -> bool:
    return REF_SO.exists() or Path("/root/reference/proj/src/solver.cpp").exists()
