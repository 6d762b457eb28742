"""B200-native neural-preconditioned PSDO ("DCDM") Poisson solve.

Host-side mirror of the reference's solver / preconditioner interface
(/root/reference/proj/include/npsd/{solver,precond}.hpp, net/precond.hpp) over
the C ABI in include/npsd_b200.h (libnpsd_b200.so, hand-written sm_100a CUDA).
Names, argument meaning and error behaviour follow the reference:

    SolveConfig / SolveReport / SolveResult   solver.hpp:11-42
    NeuralPrecond, neural_precond            net/precond.hpp:14-33
    psdo_solve, psd_solve                     solver.hpp:64-69
    init_params                               net/params.hpp:102 (net_params.cpp:11-35)
    std::invalid_argument -> ValueError, SolverBreakdown, EmptySystemError

There is no CPU fallback: every call runs on the GPU through the C ABI and
raises if the library or the device is unavailable.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import NPSD_BREAKDOWN, NPSD_CUDA_ERROR, NPSD_EMPTY_SYSTEM, NPSD_INVALID_ARGUMENT, NPSD_IO_ERROR, NPSD_OK

__all__ = [
    "SolveConfig", "SolveReport", "SolveResult", "SolverBreakdown", "EmptySystemError", "DeviceError",
    "NetParams", "init_params", "identity_params", "param_count", "rhs_normal", "Context", "NeuralPrecond",
    "neural_precond", "psdo_solve", "psd_solve", "DeviceBuffer", "PinnedBuffer", "save_npm", "load_npm",
    "Comm", "partition",
]


class SolverBreakdown(RuntimeError):
    """types.hpp:19-22 — curvature d'Ad non-positive or underflowed."""


class EmptySystemError(RuntimeError):
    """types.hpp:25-28 — the image has no fluid cells."""


class DeviceError(RuntimeError):
    """CUDA failure (no CPU fallback exists)."""


def _raise(status: int, msg: str) -> None:
    if status == NPSD_OK:
        return
    if status == NPSD_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == NPSD_BREAKDOWN:
        raise SolverBreakdown(msg)
    if status == NPSD_EMPTY_SYSTEM:
        raise EmptySystemError(msg)
    raise DeviceError(msg)


# ------------------------------------------------------------------ config
@dataclass
class SolveConfig:
    """solver.hpp:11-26."""
    tol_reduction: float = 1e-6
    tol_abs: float = 0.0
    max_iters: int = 1000
    n_ortho: int = 2
    nullspace_projection: bool = False
    normalize_before_precond: bool = True

    def _c(self, precond: int = 0) -> _native.SolveCfg:
        """precond: 0 the network (NeuralPrecond), 1 IdentityPrecond (the
        reference passes the preconditioner as psdo_solve's P argument)."""
        return _native.SolveCfg(float(self.tol_reduction), float(self.tol_abs), int(self.max_iters),
                                int(self.n_ortho), int(bool(self.nullspace_projection)),
                                int(bool(self.normalize_before_precond)), int(precond))


@dataclass
class SolveReport:
    """solver.hpp:28-37."""
    iterations: int = 0
    converged: bool = False
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    cumulative_seconds: np.ndarray = field(default_factory=lambda: np.zeros(0))
    setup_seconds: float = 0.0
    iterate_seconds: float = 0.0
    precond_seconds: float = 0.0
    method: str = ""


@dataclass
class SolveResult:
    """solver.hpp:39-42."""
    x: np.ndarray
    report: SolveReport


# ----------------------------------------------------------------- weights
@dataclass
class NetParams:
    """Flat f32 weights in for_each_span order (net/params.hpp:66-80)."""
    dim: int
    depth: int
    flat: np.ndarray

    def parameter_count(self) -> int:
        return param_count(self.dim, self.depth)


def param_count(dim: int, depth: int) -> int:
    n = int(_native.lib().npsd_b200_param_count(dim, depth))
    if n == 0:
        raise ValueError("param_count: dim must be 2 or 3 and depth >= 1")
    return n


def init_params(depth: int, seed: int, dim: int = 3) -> NetParams:
    """init_params (net_params.cpp:11-35), generalised to 3D."""
    out = np.empty(param_count(dim, depth), np.float32)
    _raise(_native.lib().npsd_b200_init_params(dim, depth, seed, out), "init_params: bad dim/depth")
    return NetParams(dim, depth, out)


def save_npm(params: NetParams, path) -> None:
    """save_npm (net_params.cpp:42-52): "NPMW", u32 version 1, dim, depth, f32
    weights in for_each_span order. dim 2 files are the reference's bytes;
    dim 3 is the 3D variant of the layout."""
    flat = np.ascontiguousarray(params.flat, np.float32)
    st = _native.lib().npsd_b200_save_npm(str(path).encode(), params.dim, params.depth, flat, flat.size)
    if st == NPSD_IO_ERROR:
        raise RuntimeError(_native.lib().npsd_b200_npm_last_error().decode())
    _raise(st, _native.lib().npsd_b200_npm_last_error().decode())


def load_npm(path) -> NetParams:
    """load_npm (net_params.cpp:54-78): rejects a bad magic, version, dim or
    depth and truncated data with the reference's runtime_error messages."""
    L = _native.lib()
    dim, depth, n = C.c_int(0), C.c_int(0), C.c_size_t(0)
    p = str(path).encode()
    st = L.npsd_b200_load_npm(p, C.byref(dim), C.byref(depth), None, 0, C.byref(n))
    if st == NPSD_OK:
        out = np.empty(n.value, np.float32)
        st = L.npsd_b200_load_npm(p, C.byref(dim), C.byref(depth), out.ctypes.data, out.size,
                                  C.byref(n))
    if st == NPSD_IO_ERROR:
        raise RuntimeError(L.npsd_b200_npm_last_error().decode())
    _raise(st, L.npsd_b200_npm_last_error().decode())
    return NetParams(dim.value, depth.value, out)


# The repo's trained 3D model: the weights every benchmark and
# the trained-weight parity fixtures use. npsd3d_L4.npm is the depth-4 model.
DEFAULT_MODEL = Path(__file__).resolve().parent / "weights" / "npsd3d_L6.npm"


def default_model() -> NetParams:
    """load_npm(DEFAULT_MODEL)."""
    return load_npm(DEFAULT_MODEL)


def identity_params(depth: int, dim: int = 3) -> NetParams:
    """Identity-equivalent weights: the network returns its input (PSDO == CG)."""
    out = np.empty(param_count(dim, depth), np.float32)
    _raise(_native.lib().npsd_b200_identity_params(dim, depth, out), "identity_params: bad dim/depth")
    return NetParams(dim, depth, out)


def rhs_normal(seed: int, n: int) -> np.ndarray:
    """Rng(seed).normal() x n (rng.hpp:36-48)."""
    out = np.empty(n, np.float64)
    _native.lib().npsd_b200_rhs_normal(seed, n, out)
    return out


# ------------------------------------------------------------------ context
def partition(nz: int, nranks: int, depth: int) -> list[tuple[int, int]]:
    """z-slab bounds (z0, nz_own) per rank: contiguous planes in units of
    2^(depth-1) (the pooling alignment of every level), as equal as possible."""
    unit = 1 << (depth - 1)
    if nz % unit or nranks < 1 or nz // unit < nranks:
        raise ValueError(f"partition: {nz} planes cannot form {nranks} slabs of multiples of {unit}")
    units = nz // unit
    out, z0 = [], 0
    for r in range(nranks):
        k = units // nranks + (1 if r < units % nranks else 0)
        out.append((z0, k * unit))
        z0 += k * unit
    return out


class Comm:
    """Communicator of a z-slab decomposition (include/npsd_b200.h)."""

    def __init__(self, handle, nranks: int) -> None:
        self.h, self.nranks, self.lib = handle, nranks, _native.lib()

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        st = _native.lib().npsd_b200_nccl_unique_id(buf)
        if st != NPSD_OK:
            raise DeviceError(_native.lib().npsd_b200_comm_last_error().decode())
        return buf.raw

    @classmethod
    def nccl(cls, uid: bytes, rank: int, nranks: int, device: int = 0) -> "Comm":
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(uid), 128)
        st = _native.lib().npsd_b200_comm_create_nccl(buf, rank, nranks, device, C.byref(h))
        if st != NPSD_OK:
            raise DeviceError(_native.lib().npsd_b200_comm_last_error().decode())
        return cls(h, nranks)

    @classmethod
    def local(cls, nranks: int) -> "Comm":
        """In-process ranks (one host thread each, one device): tests only."""
        h = C.c_void_p()
        _raise(_native.lib().npsd_b200_comm_create_local(nranks, C.byref(h)), "comm: bad nranks")
        return cls(h, nranks)

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.npsd_b200_comm_destroy(self.h)
            self.h = None


_PCG_KINDS = {"identity": 0, "jacobi": 1, "ic0": 2}
_PCG_METHOD = {0: "cg", 1: "pcg+jacobi", 2: "pcg+ic0"}


class Context:
    """One B200 context: grid, weights and (after set_mask) one frame."""

    def __init__(self, dim: int, shape: tuple, params: NetParams, device: int = 0, exact: bool = False) -> None:
        if dim == 3:
            nz, ny, nx = shape
        else:
            (ny, nx), nz = shape, 1
        if params.dim != dim:
            raise ValueError("NeuralPrecond: params dim does not match the grid")
        self.lib = _native.lib()
        self.dim, self.nx, self.ny, self.nz, self.depth = dim, nx, ny, nz, params.depth
        self.shape = tuple(shape)
        self.n_cells = nx * ny * nz
        h = C.c_void_p()
        dev = (C.c_int * 1)(device)
        flat = np.ascontiguousarray(params.flat, np.float32)
        st = self.lib.npsd_b200_create(dim, nx, ny, nz, params.depth, flat, flat.size, C.cast(dev, C.c_void_p), 1,
                                       C.byref(h))
        if st != NPSD_OK:
            _raise(st, self.lib.npsd_b200_last_error(None).decode())
        self.h = h
        if exact:
            self.set_exact(True)

    @classmethod
    def slab(cls, comm: Comm, rank: int, shape: tuple, z0: int, nz_own: int, params: NetParams,
             device: int = 0) -> "Context":
        """Rank `rank`'s z-slab [z0, z0 + nz_own) of a 3D grid of `shape`
        (nz, ny, nx): set_mask takes the owned planes (nz_own, ny, nx); solver
        vectors are the owned fluid cells in ascending global order."""
        nz, ny, nx = shape
        if params.dim != 3:
            raise ValueError("NeuralPrecond: params dim does not match the grid")
        self = cls.__new__(cls)
        self.lib = _native.lib()
        self.dim, self.nx, self.ny, self.nz, self.depth = 3, nx, ny, nz, params.depth
        self.shape = (nz_own, ny, nx)
        self.n_cells = nx * ny * nz_own
        self.z0, self.nz_own, self.comm = z0, nz_own, comm
        h = C.c_void_p()
        flat = np.ascontiguousarray(params.flat, np.float32)
        st = self.lib.npsd_b200_create_slab(nx, ny, nz, z0, nz_own, params.depth, flat, flat.size, device, comm.h,
                                            rank, C.byref(h))
        if st != NPSD_OK:
            _raise(st, self.lib.npsd_b200_last_error(None).decode())
        self.h = h
        return self

    def mac_divergence_rhs(self, u, v, w=None, h: float = 1.0, dt: float = 0.05, rho: float = 1.0,
                           bc=None) -> np.ndarray:
        """mac_divergence_rhs + reduce (discretization.cpp:193-227) on the
        device for this frame: the solve's reduced b. Faces x fastest (numpy
        shapes (nz, ny, nx+1), (nz, ny+1, nx), (nz+1, ny, nx)); bc = (bu, bv[,
        bw]) prescribed normal velocities on solid faces, or None (zero)."""
        arrs = [np.ascontiguousarray(a, np.float64) if a is not None else None
                for a in (u, v, w, *(list(bc) + [None] * 3)[:3]) ] if bc else \
            [np.ascontiguousarray(a, np.float64) if a is not None else None for a in (u, v, w, None, None, None)]
        ptr = [a.ctypes.data if a is not None else None for a in arrs]
        out = np.empty(self.n_fluid, np.float64)
        self._ck(self.lib.npsd_b200_mac_divergence_rhs(self.h, ptr[0], ptr[1], ptr[2], h, dt, rho, ptr[3], ptr[4],
                                                       ptr[5], out.ctypes.data))
        return out

    def mac_divergence_rhs_device(self, d_u: int, d_v: int, d_w: int | None, d_b_full: int, h: float = 1.0,
                                  dt: float = 0.05, rho: float = 1.0, d_bc=None) -> None:
        """Device pointers in, the full-grid b (zeros off fluid) out: the input
        of psdo_solve_device."""
        bu, bv, bw = (list(d_bc) + [None] * 3)[:3] if d_bc else (None, None, None)
        self._ck(self.lib.npsd_b200_mac_divergence_rhs_device(self.h, d_u, d_v, d_w, h, dt, rho, bu, bv, bw,
                                                              d_b_full))

    @property
    def slab_graph(self) -> bool:
        """z-slab: the last solve's iterations ran as captured chunk graphs."""
        return bool(self.lib.npsd_b200_slab_graph(self.h))

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.npsd_b200_destroy(self.h)
            self.h = None

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, st: int) -> None:
        if st != NPSD_OK:
            _raise(st, self.lib.npsd_b200_last_error(self.h).decode())

    # per frame
    def set_params(self, params: NetParams) -> None:
        flat = np.ascontiguousarray(params.flat, np.float32)
        self._ck(self.lib.npsd_b200_set_params(self.h, flat, flat.size))

    def set_exact(self, exact: bool = True) -> None:
        """Network arithmetic (npsd_b200_set_exact): exact=True runs every
        network operation in the reference's order (bit-identical to the
        restatement); False (the default) is the fast fused form, within the
        north_star tolerance."""
        self._ck(self.lib.npsd_b200_set_exact(self.h, int(bool(exact))))

    def set_mask(self, types: np.ndarray) -> None:
        t = np.ascontiguousarray(types, np.uint8).reshape(-1)
        if t.size != self.n_cells:
            raise ValueError("set_mask: cell type array does not match the grid")
        self._ck(self.lib.npsd_b200_set_mask(self.h, t))

    def set_mask_device(self, ptr: int) -> None:
        self._ck(self.lib.npsd_b200_set_mask_device(self.h, C.c_void_p(ptr)))

    def check_operator(self, row_offsets, col_indices, values, full: bool = False) -> None:
        """Raise ValueError unless the reduced CSR matrix is the flag-derived
        operator of the current mask (npsd_b200_check_operator)."""
        ro = np.ascontiguousarray(row_offsets, np.int64)
        ci = np.ascontiguousarray(col_indices, np.int64)
        va = np.ascontiguousarray(values, np.float64)
        if ci.size != va.size:
            raise ValueError("check_operator: col_indices and values differ in length")
        self._ck(self.lib.npsd_b200_check_operator(self.h, ro.size - 1, ro, ci, va, va.size, int(full)))

    def is_pure_neumann(self) -> bool:
        """is_pure_neumann (discretization.cpp:180-191) of the current mask: no
        fluid cell has an air face neighbour (outside the domain is solid), so
        the reduced system is singular and needs nullspace projection."""
        out = C.c_int(0)
        self._ck(self.lib.npsd_b200_is_pure_neumann(self.h, C.byref(out)))
        return bool(out.value)

    @property
    def n_fluid(self) -> int:
        return int(self.lib.npsd_b200_n_fluid(self.h))

    def fluid_indices(self) -> np.ndarray:
        out = np.empty(self.n_fluid, np.int64)
        self._ck(self.lib.npsd_b200_fluid_indices(self.h, out))
        return out

    # operators
    def precond_apply(self, r: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty_like(r)
        self._ck(self.lib.npsd_b200_precond_apply(self.h, r, z, r.size))
        return z

    def ic0_apply(self, r: np.ndarray) -> tuple[np.ndarray, int]:
        """Ic0Precond (precond.cpp:28-112) on the current frame: factor (with
        the reference's diagonal-shift retries), then apply(r) -> (z, retries)."""
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty_like(r)
        retries = C.c_int()
        self._ck(self.lib.npsd_b200_ic0_apply(self.h, r, z, r.size, C.byref(retries)))
        return z, retries.value

    def spmv(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        self._ck(self.lib.npsd_b200_spmv(self.h, x, y, x.size))
        return y

    def net_apply(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32).reshape(-1)
        if x.size != self.n_cells:
            raise ValueError("NetContext::apply: field shape mismatch")
        y = np.empty_like(x)
        self._ck(self.lib.npsd_b200_net_apply(self.h, x, y))
        return y.reshape(self.shape)

    def level_image(self, level: int) -> np.ndarray:
        nx, ny = self.nx >> level, self.ny >> level
        nz = (self.nz >> level) if self.dim == 3 else 1
        out = np.empty(3 * nx * ny * nz, np.float32)
        self._ck(self.lib.npsd_b200_level_image(self.h, level, out))
        return out.reshape((3, nz, ny, nx) if self.dim == 3 else (3, ny, nx))

    def linear_coeffs(self) -> tuple[np.ndarray, np.ndarray]:
        za = np.zeros(max(self.depth - 1, 1), np.float32)
        zb = np.zeros_like(za)
        self._ck(self.lib.npsd_b200_linear_coeffs(self.h, za, zb))
        return za[: self.depth - 1], zb[: self.depth - 1]

    def mixed_counts(self) -> np.ndarray:
        out = np.zeros(self.depth, np.int64)
        self._ck(self.lib.npsd_b200_mixed_counts(self.h, out))
        return out

    def _report(self, rep: _native.Report, method: str) -> SolveReport:
        n = int(rep.history_len)
        hist = np.ctypeslib.as_array(rep.residual_history, shape=(n,)).copy() if n else np.zeros(0)
        secs = np.ctypeslib.as_array(rep.cumulative_seconds, shape=(n,)).copy() if n else np.zeros(0)
        return SolveReport(int(rep.iterations), bool(rep.converged), hist, secs, float(rep.setup_seconds),
                           float(rep.iterate_seconds), float(rep.precond_seconds), method)

    def psdo_solve(self, b: np.ndarray, cfg: SolveConfig, x0: np.ndarray | None = None,
                   method: str = "psdo+neural", out: np.ndarray | None = None, precond: str = "neural") -> SolveResult:
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b) if out is None else out
        if x.dtype != np.float64 or x.size != b.size or not x.flags.c_contiguous:
            raise ValueError("solve: out must be a contiguous f64 array of the rhs length")
        rep = _native.Report()
        x0p = None
        if x0 is not None:
            x0a = np.ascontiguousarray(x0, np.float64)
            if x0a.size != b.size:
                raise ValueError("solve: x0 length mismatch")
            x0p = x0a.ctypes.data_as(C.c_void_p)
        c = cfg._c(_PSDO_PRECOND[precond])
        # sized entry point: the rhs upload overlaps a set_mask still in flight;
        # the length is checked against the fluid count on the C side
        st = self.lib.npsd_b200_psdo_solve_n(self.h, b, b.size, x0p, C.byref(c), x, C.byref(rep))
        if st == NPSD_BREAKDOWN:
            _raise(st, self.lib.npsd_b200_last_error(self.h).decode())
        self._ck(st)
        return SolveResult(x, self._report(rep, method))

    def pcg_solve(self, b: np.ndarray, cfg: SolveConfig, precond: str = "identity", x0: np.ndarray | None = None,
                  out: np.ndarray | None = None) -> SolveResult:
        """pcg_solve / cg_solve (solver.cpp:36-109) on the device: precond
        "identity" (method "cg"), "jacobi" ("pcg+jacobi") or "ic0" ("pcg+ic0")."""
        kind = _PCG_KINDS[precond]
        b = np.ascontiguousarray(b, np.float64)
        if b.size != self.n_fluid:
            raise ValueError("solve: rhs length mismatch")
        x = np.empty_like(b) if out is None else out
        if x.dtype != np.float64 or x.size != b.size or not x.flags.c_contiguous:
            raise ValueError("solve: out must be a contiguous f64 array of the rhs length")
        x0p = None
        if x0 is not None:
            x0a = np.ascontiguousarray(x0, np.float64)
            if x0a.size != b.size:
                raise ValueError("solve: x0 length mismatch")
            x0p = x0a.ctypes.data_as(C.c_void_p)
        rep = _native.Report()
        c = cfg._c()
        st = self.lib.npsd_b200_pcg_solve(self.h, b, x0p, C.byref(c), kind, x, C.byref(rep))
        self._ck(st)
        return SolveResult(x, self._report(rep, _PCG_METHOD[kind]))

    def pcg_solve_device(self, b_ptr: int, x_ptr: int, cfg: SolveConfig, precond: str = "identity",
                         x0_ptr: int | None = None) -> SolveReport:
        kind = _PCG_KINDS[precond]
        rep = _native.Report()
        c = cfg._c()
        self._ck(self.lib.npsd_b200_pcg_solve_device(self.h, C.c_void_p(b_ptr), C.c_void_p(x0_ptr) if x0_ptr else None,
                                                     C.byref(c), kind, C.c_void_p(x_ptr), C.byref(rep)))
        return self._report(rep, _PCG_METHOD[kind])

    def psdo_solve_device(self, b_ptr: int, x_ptr: int, cfg: SolveConfig, x0_ptr: int | None = None,
                          method: str = "psdo+neural", precond: str = "neural") -> SolveReport:
        rep = _native.Report()
        c = cfg._c(_PSDO_PRECOND[precond])
        self._ck(self.lib.npsd_b200_psdo_solve_device(self.h, C.c_void_p(b_ptr),
                                                      C.c_void_p(x0_ptr) if x0_ptr else None, C.byref(c),
                                                      C.c_void_p(x_ptr), C.byref(rep)))
        return self._report(rep, method)

    def synchronize(self) -> None:
        self._ck(self.lib.npsd_b200_synchronize(self.h))

    @property
    def last_solve_ms(self) -> float:
        return float(self.lib.npsd_b200_last_solve_ms(self.h))

    @property
    def last_solve_launches(self) -> int:
        return int(self.lib.npsd_b200_last_solve_launches(self.h))

    @property
    def launch_count(self) -> int:
        return int(self.lib.npsd_b200_launch_count(self.h))

    def event_record(self, slot: int) -> None:
        self._ck(self.lib.npsd_b200_event_record(self.h, slot))

    def event_elapsed_ms(self, a: int, b: int) -> float:
        ms = float(self.lib.npsd_b200_event_elapsed_ms(self.h, a, b))
        if ms < 0:
            raise DeviceError("event_elapsed_ms failed")
        return ms

    def profile_iterations(self, b_ptr: int, cfg: SolveConfig, iters: int) -> dict[str, float]:
        """Mean device ms per kernel of `iters` PSDO iterations, kernels launched
        one by one between CUDA events on the context stream."""
        cap, nl = 64, 32
        ms = np.zeros(cap, np.float64)
        n = C.c_int(cap)
        names = C.create_string_buffer(cap * nl)
        c = cfg._c()
        self._ck(self.lib.npsd_b200_profile_iterations(self.h, C.c_void_p(b_ptr), C.byref(c), int(iters), ms,
                                                       C.byref(n), names, nl))
        raw = names.raw
        return {raw[k * nl:(k + 1) * nl].split(b"\0")[0].decode(): float(ms[k]) for k in range(n.value)}


class DeviceBuffer:
    """Raw device allocation owned by a Context (cudaMalloc through the C ABI)."""

    def __init__(self, ctx: Context, nbytes: int) -> None:
        self.ctx, self.nbytes = ctx, int(nbytes)
        p = C.c_void_p()
        ctx._ck(ctx.lib.npsd_b200_device_alloc(ctx.h, self.nbytes, C.byref(p)))
        self.ptr = int(p.value)

    def upload(self, src: np.ndarray | "PinnedBuffer") -> None:
        sp = src.ptr if isinstance(src, PinnedBuffer) else np.ascontiguousarray(src).ctypes.data
        self.ctx._ck(self.ctx.lib.npsd_b200_memcpy(self.ctx.h, C.c_void_p(self.ptr), C.c_void_p(sp), self.nbytes))

    def download(self, dst: np.ndarray | "PinnedBuffer") -> None:
        dp = dst.ptr if isinstance(dst, PinnedBuffer) else dst.ctypes.data
        self.ctx._ck(self.ctx.lib.npsd_b200_memcpy(self.ctx.h, C.c_void_p(dp), C.c_void_p(self.ptr), self.nbytes))

    def free(self) -> None:
        if self.ptr:
            self.ctx.lib.npsd_b200_device_free(self.ctx.h, C.c_void_p(self.ptr))
            self.ptr = 0


class PinnedBuffer:
    """Page-locked host memory (cudaMallocHost) viewed as a numpy array."""

    def __init__(self, ctx: Context, n: int, dtype=np.float64) -> None:
        self.ctx = ctx
        self.dtype = np.dtype(dtype)
        self.nbytes = int(n) * self.dtype.itemsize
        p = C.c_void_p()
        ctx._ck(ctx.lib.npsd_b200_host_alloc(ctx.h, self.nbytes, C.byref(p)))
        self.ptr = int(p.value)
        buf = (C.c_char * self.nbytes).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=int(n))

    def free(self) -> None:
        if self.ptr:
            self.array = None
            self.ctx.lib.npsd_b200_host_free(self.ctx.h, C.c_void_p(self.ptr))
            self.ptr = 0


# -------------------------------------------------------- preconditioner API
_PSDO_PRECOND = {"neural": 0, "identity": 1, "none": 1, "jacobi": 2}


class NeuralPrecond:
    """net::NeuralPrecond (net/precond.hpp:14-30) on a B200.

    ``image`` is the cell-type grid (0 fluid, 1 air, 2 solid), shape (ny, nx)
    or (nz, ny, nx). The optional ``map`` (fluid linear indices) is validated
    against the image like the reference ctor (net_precond.cpp:11).
    """

    def __init__(self, params: NetParams, image: np.ndarray, map: np.ndarray | None = None, device: int = 0):
        image = np.asarray(image)
        dim = 3 if image.ndim == 3 else 2
        self.ctx = Context(dim, image.shape, params, device)
        self.ctx.set_mask(image)
        if map is not None:
            m = np.asarray(map, np.int64)
            if m.size != self.ctx.n_fluid or not np.array_equal(m, self.ctx.fluid_indices()):
                raise ValueError("NeuralPrecond: map does not match image")

    def apply(self, r: np.ndarray, z: np.ndarray | None = None) -> np.ndarray:
        r = np.asarray(r, np.float64)
        if r.size != self.size():
            raise ValueError("NeuralPrecond::apply: size mismatch")
        out = self.ctx.precond_apply(r)
        if z is not None:
            z[...] = out
            return z
        return out

    __call__ = apply

    def is_linear(self) -> bool:
        return True

    def is_symmetric(self) -> bool:
        return False

    def size(self) -> int:
        return self.ctx.n_fluid

    def name(self) -> str:
        return "neural"


class IdentityPrecond:
    """IdentityPrecond (precond.hpp:35-43, precond.cpp:7-10) for the B200
    psdo_solve: apply copies (z = r) like the reference; inside psdo_solve the
    device loop forms d = r / ||r|| without the network. The image (cell
    types) gives the device its matrix-free operator."""

    def __init__(self, image: np.ndarray, device: int = 0):
        image = np.asarray(image)
        dim = 3 if image.ndim == 3 else 2
        depth = 1  # the network is never run; the smallest context
        self.ctx = Context(dim, image.shape, identity_params(depth, dim), device)
        self.ctx.set_mask(image)

    def apply(self, r: np.ndarray, z: np.ndarray | None = None) -> np.ndarray:
        r = np.asarray(r, np.float64)
        if r.size != self.size():
            raise ValueError("IdentityPrecond::apply: size mismatch")
        if z is not None:
            z[...] = r
            return z
        return r.copy()

    __call__ = apply

    def is_linear(self) -> bool:
        return True

    def is_symmetric(self) -> bool:
        return True

    def size(self) -> int:
        return self.ctx.n_fluid

    def name(self) -> str:
        return "identity"


def neural_precond(params: NetParams, image: np.ndarray, map: np.ndarray | None = None) -> NeuralPrecond:
    """net/precond.hpp:32-33."""
    return NeuralPrecond(params, image, map)


def _rows(A) -> int | None:
    if A is None:
        return None
    for attr in ("n_rows", "shape"):
        if hasattr(A, attr):
            v = getattr(A, attr)
            return int(v[0]) if isinstance(v, tuple) else int(v)
    return None


def _csr(A):
    """(row_offsets, col_indices, values) of a reduced CSR matrix: the
    reference's SparseMatrix fields or scipy.sparse's indptr/indices/data."""
    for names in (("row_offsets", "col_indices", "values"), ("indptr", "indices", "data")):
        if all(hasattr(A, n) for n in names):
            return tuple(np.asarray(getattr(A, n)) for n in names)
    return None


def psdo_solve(A, b: np.ndarray, P, cfg: SolveConfig | None = None, x0: np.ndarray | None = None,
               check_a: str = "rows") -> SolveResult:
    """psdo_solve (solver.hpp:64-65, solver.cpp:189-276) on the B200.

    The operator is matrix-free: the mixed-BC Laplacian that
    assemble_poisson[_3d] + reduce build from P's image. A CSR ``A``
    (row_offsets/col_indices/values, or scipy indptr/indices/data) is checked
    against it — ``check_a`` "rows": every row's nnz, diagonal and -1
    off-diagonals; "full": also A v bitwise against the device operator — and a
    different A raises ValueError instead of solving another system. ``A`` =
    None skips the check. P is a B200 NeuralPrecond or IdentityPrecond; there
    is no CPU path.
    """
    cfg = cfg or SolveConfig()
    if not isinstance(P, (NeuralPrecond, IdentityPrecond)):
        raise ValueError("psdo_solve (B200): P must be a B200 NeuralPrecond or IdentityPrecond; there is no CPU path")
    n = _rows(A)
    if n is not None and n != P.size():
        raise ValueError("solve: matrix not square / rhs length mismatch")
    csr = _csr(A) if A is not None else None
    if csr is not None:
        P.ctx.check_operator(*csr, full=(check_a == "full"))
    b = np.asarray(b, np.float64)
    if b.size != P.size():
        raise ValueError("solve: rhs length mismatch")
    if not np.all(np.isfinite(b)):
        raise ValueError("solve: rhs has non-finite entries")
    return P.ctx.psdo_solve(b, cfg, x0, method="psdo+" + P.name(), precond=P.name())


def psd_solve(A, b: np.ndarray, P, cfg: SolveConfig | None = None,
              x0: np.ndarray | None = None) -> SolveResult:
    """PSDO with n_ortho forced to 0 (solver.hpp:68-69)."""
    cfg = SolveConfig(**{**(cfg or SolveConfig()).__dict__, "n_ortho": 0})
    res = psdo_solve(A, b, P, cfg, x0)
    res.report.method = "psd+" + P.name()
    return res
