"""B200-native phi-combination engine (arXiv 2509.26475 hot path).

Python mirror of the reference's public interface for the path
(include/phiact/params.hpp, phi_block.hpp, phi_single.hpp, linop.hpp) over the
C ABI of libphx.so (include/phx.h).  The numerical work runs in hand-written
sm_100a kernels; this module only marshals arguments.  There is no CPU
fallback: if libphx.so is missing the import of the native library fails
loudly, and without a GPU every compute call raises CudaError.

Names and argument meaning follow the reference:
  select_parameters(op, m=61, tol=-1, delta=0.8) -> ScalingShift
  phimv_block(op, BlockPhiRequest) -> BlockPhiResult(W, stats: RunRecord)
  phimv(op, PhiRequest) -> PhiResult(w, exp_v0, tail, stats)
  build_power_basis / objective / minimize_shift / parameters_for_shift
Errors: ValueError ~ std::invalid_argument, RuntimeError ~
std::runtime_error, LogicError ~ std::logic_error, CudaError for device
failures.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "CsrOperator", "ScalingShift", "RunRecord", "BlockPhiRequest", "BlockPhiResult",
    "PhiRequest", "PhiResult", "PowerBasis", "select_parameters", "build_power_basis",
    "objective", "minimize_shift", "parameters_for_shift", "phimv_block", "phimv",
    "workload", "LogicError", "CudaError", "lib", "lib_path", "kernel_launches",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBDIR = os.path.join(_HERE, "lib")

dp = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)


class LogicError(RuntimeError):
    """std::logic_error analogue (empty operator, shape)."""


class CudaError(RuntimeError):
    """Device failure (no GPU, CUDA error)."""


class _SS(C.Structure):
    _fields_ = [("s", C.c_double), ("xi", C.c_double), ("s0", C.c_double),
                ("f_min", C.c_double), ("m", C.c_int32), ("r", C.c_int32)]


class _Rec(C.Structure):
    _fields_ = [("s_effective", C.c_int64), ("series_len_S", C.c_int32),
                ("n_sweeps", C.c_int32), ("series_lens_F", i32p),
                ("lens_capacity", C.c_int64), ("matvecs", C.c_int64)]


class _WlInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("p", C.c_int32), ("r", C.c_int32),
                ("tol", C.c_double), ("size", C.c_int64)]


_LIB = None
_WL = None

# every exported symbol of include/phx.h (checked by tests/test_abi.py)
ABI_SYMBOLS = (
    "phx_op_create_csr", "phx_op_create_csr_partitioned", "phx_op_nparts", "phx_op_destroy",
    "phx_op_dim", "phx_op_nnz", "phx_op_stream", "phx_apply",
    "phx_shifted_apply", "phx_select_parameters", "phx_basis_build", "phx_basis_destroy",
    "phx_basis_info", "phx_objective", "phx_minimize_shift", "phx_parameters_for_shift",
    "phx_phimv_block", "phx_phimv_block_device", "phx_phimv", "phx_last_error",
    "phx_kernel_launches", "phx_last_eval_stats", "phx_set_trace", "phx_get_trace",
    "phx_adr_csr", "phx_exprk4s6_step", "phx_integrate",
    "phx_mm_read_csr", "phx_mm_write_csr", "phx_op_create_mm", "phx_block_series_direct",
    "phx_last_eval_mode",
    "phx_last_eval_variant",
    "phx_tile_plan", "phx_tile_plan_part", "phx_op_part_info", "phx_phimv_block_device_parts",
)


def lib_path() -> str:
    """libphx.so, or the self-checking build libphx_checked.so (device-side
    bounds checks; `make -C paper_2509_26475_b200/csrc checked`) when the
    environment sets PHX_LIB=checked."""
    v = os.environ.get("PHX_LIB")
    if v:  # "checked", or a developer A/B build (csrc/Makefile `variant`)
        return os.path.join(_LIBDIR, f"libphx_{v}.so")
    return os.path.join(_LIBDIR, "libphx.so")


def lib():
    """Load libphx.so (raises if the CUDA extension has not been built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(
            f"libphx.so not found at {path}: the CUDA extension is missing; run "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    L = C.CDLL(path)
    L.phx_last_error.restype = C.c_char_p
    L.phx_kernel_launches.restype = C.c_int64
    L.phx_op_dim.restype = C.c_int64
    L.phx_op_dim.argtypes = [C.c_void_p]
    L.phx_op_nnz.restype = C.c_int64
    L.phx_op_nnz.argtypes = [C.c_void_p]
    L.phx_op_create_csr.argtypes = [C.c_int64, i64p, i32p, dp, C.c_int32, C.POINTER(C.c_void_p)]
    L.phx_op_destroy.argtypes = [C.c_void_p]
    L.phx_op_create_csr_partitioned.argtypes = [C.c_int64, i64p, i32p, dp, C.c_int32, i32p,
                                                C.POINTER(C.c_void_p)]
    L.phx_op_nparts.restype = C.c_int32
    L.phx_op_nparts.argtypes = [C.c_void_p]
    L.phx_op_stream.restype = C.c_void_p
    L.phx_op_stream.argtypes = [C.c_void_p]
    L.phx_apply.argtypes = [C.c_void_p, dp, C.c_int64, C.c_int64, dp, C.c_int64]
    L.phx_shifted_apply.argtypes = [C.c_void_p, C.c_double, dp, C.c_int64, C.c_int64, dp, C.c_int64]
    L.phx_select_parameters.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_double,
                                        C.POINTER(_SS)]
    L.phx_basis_build.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.POINTER(C.c_void_p)]
    L.phx_basis_destroy.argtypes = [C.c_void_p]
    L.phx_basis_info.argtypes = [C.c_void_p, i32p, i32p, dp, dp, dp, dp]
    L.phx_objective.argtypes = [C.c_void_p, C.c_double, dp]
    L.phx_minimize_shift.argtypes = [C.c_void_p, dp, dp, dp, C.c_int64, i64p]
    L.phx_parameters_for_shift.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                           C.POINTER(_SS)]
    L.phx_phimv_block.argtypes = [C.c_void_p, C.c_int32, dp, dp, C.c_int32, dp, C.c_int64,
                                  C.c_double, C.POINTER(_SS), dp, C.c_int64, C.POINTER(_Rec)]
    L.phx_phimv_block_device.argtypes = [C.c_void_p, C.c_int32, dp, dp, C.c_int32, C.c_void_p,
                                         C.c_double, C.POINTER(_SS), C.c_void_p, C.POINTER(_Rec)]
    L.phx_phimv.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int32, dp, C.c_int64,
                            C.c_double, C.POINTER(_SS), dp, dp, dp, C.POINTER(_Rec)]
    L.phx_adr_csr.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, i64p, i32p, dp, dp]
    L.phx_exprk4s6_step.argtypes = [C.c_void_p, C.c_double, dp, C.c_double, C.c_double,
                                    C.POINTER(_SS), dp, C.POINTER(_Rec)]
    L.phx_integrate.argtypes = [C.c_void_p, C.c_double, dp, C.c_double, C.c_double, C.c_double,
                                C.POINTER(_SS), dp, dp, i64p, C.POINTER(_Rec), C.c_int64]
    L.phx_mm_read_csr.argtypes = [C.c_char_p, i64p, i64p, i64p, i32p, dp, C.c_int64]
    L.phx_mm_write_csr.argtypes = [C.c_char_p, C.c_int64, i64p, i32p, dp]
    L.phx_op_create_mm.argtypes = [C.c_char_p, C.c_int32, C.POINTER(C.c_void_p)]
    L.phx_block_series_direct.argtypes = [C.c_void_p, C.c_int32, dp, dp, C.c_int32, dp,
                                          C.c_int64, C.c_double, dp, C.c_int64, dp, C.c_int64]
    L.phx_last_eval_stats.argtypes = [dp, i64p]
    L.phx_last_eval_mode.restype = C.c_int32
    L.phx_last_eval_variant.argtypes = [C.POINTER(C.c_int32)]
    L.phx_tile_plan.argtypes = [C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                C.POINTER(C.c_uint8), C.POINTER(C.c_int32)]
    if hasattr(L, "phx_tile_plan_part"):  # (older developer A/B builds lack it)
        L.phx_tile_plan_part.argtypes = [C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                         C.c_int64, C.c_int64, C.POINTER(C.c_int32),
                                         C.POINTER(C.c_int32), C.POINTER(C.c_uint8),
                                         C.POINTER(C.c_int32)]
    L.phx_op_part_info.argtypes = [C.c_void_p, C.c_int32, i64p, i64p, i32p,
                                   C.POINTER(C.c_void_p)]
    L.phx_phimv_block_device_parts.argtypes = [C.c_void_p, C.c_int32, dp, dp, C.c_int32,
                                               C.POINTER(C.c_void_p), C.c_double, C.POINTER(_SS),
                                               C.POINTER(C.c_void_p), C.POINTER(_Rec)]
    L.phx_set_trace.argtypes = [C.c_int64]
    L.phx_get_trace.argtypes = [dp, C.c_int64, i64p]
    _LIB = L
    return L


def _check(code: int):
    if code == 0:
        return
    msg = lib().phx_last_error().decode()
    if code == 1:
        raise ValueError(msg)
    if code == 2:
        raise RuntimeError(msg)
    if code == 3:
        raise LogicError(msg)
    if code == 5:
        raise MemoryError(msg)
    raise CudaError(msg)


def _d(a):
    return a.ctypes.data_as(dp)


def kernel_launches() -> int:
    return int(lib().phx_kernel_launches())


# ---------------------------------------------------------------------------
# types (params.hpp:34-41, phi_single.hpp:16-39, phi_block.hpp:14-25)
# ---------------------------------------------------------------------------
@dataclass
class ScalingShift:
    s: float = 1.0
    xi: float = 0.0
    s0: float = 1.0
    f_min: float = 0.0
    m: int = 61
    r: int = 0

    def _c(self):
        return _SS(self.s, self.xi, self.s0, self.f_min, self.m, self.r)

    @staticmethod
    def _from(c):
        return ScalingShift(c.s, c.xi, c.s0, c.f_min, c.m, c.r)

    def astuple(self):
        return (self.s, self.xi, self.s0, self.f_min, self.m, self.r)


def default_tolerance() -> float:
    """The evaluator's default tolerance 2^-53 (params.hpp:15)."""
    return 2.0 ** -53


@dataclass
class RunRecord:
    s_effective: int = 1
    series_len_S: int = 0
    series_lens_F: list = field(default_factory=list)
    matvecs: int = 0


@dataclass
class BlockPhiRequest:
    t: np.ndarray
    alpha: np.ndarray
    V: np.ndarray
    tol: float = -1.0
    params: ScalingShift = field(default_factory=ScalingShift)


@dataclass
class BlockPhiResult:
    W: np.ndarray
    stats: RunRecord


@dataclass
class PhiRequest:
    t: float
    alpha: float
    V: np.ndarray
    tol: float = -1.0
    params: ScalingShift = field(default_factory=ScalingShift)


@dataclass
class PhiResult:
    w: np.ndarray
    exp_v0: np.ndarray
    tail: np.ndarray
    stats: RunRecord


class CsrOperator:
    """Device-resident CSR operator (the LinearOperator of linop.hpp:19-37
    for CSR matrices).  Column indices are used in storage order."""

    def __init__(self, n, row_ptr, col_idx, vals, device: int = -1, parts: int = 1,
                 devices=None):
        """parts > 1: row-partitioned operator, part q on
        devices[q] (default: all on `device`; one device = emulation)."""
        self.n = int(n)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        av = np.ascontiguousarray(vals, dtype=np.float64)
        h = C.c_void_p()
        if parts == 1 and devices is None:
            _check(lib().phx_op_create_csr(self.n, rp.ctypes.data_as(i64p),
                                           ci.ctypes.data_as(i32p), _d(av), device, C.byref(h)))
        else:
            devs = np.ascontiguousarray(devices if devices is not None else [device] * parts,
                                        dtype=np.int32)
            _check(lib().phx_op_create_csr_partitioned(
                self.n, rp.ctypes.data_as(i64p), ci.ctypes.data_as(i32p), _d(av), int(parts),
                devs.ctypes.data_as(i32p), C.byref(h)))
        self._h = h
        self.parts = int(lib().phx_op_nparts(h))

    @staticmethod
    def from_dense(A, device: int = -1):
        A = np.ascontiguousarray(np.asarray(A, dtype=np.float64))
        n = A.shape[0]
        if A.ndim != 2 or A.shape[1] != n:
            raise ValueError("dense_operator: matrix must be square")
        if not np.all(np.isfinite(A)):
            raise ValueError("dense_operator: matrix has non-finite entries")
        rp = np.arange(0, n * n + 1, n, dtype=np.int64)
        ci = np.tile(np.arange(n, dtype=np.int32), n)
        return CsrOperator(n, rp, ci, A.reshape(-1), device)

    @staticmethod
    def from_matrix_market(path, device: int = -1):
        """Operator from a Matrix Market file (phx_mm_read_csr)."""
        return CsrOperator(*read_matrix_market(path), device=device)

    def dim(self):
        return self.n

    def stream_ptr(self) -> int:
        """cudaStream_t of this operator (for torch.cuda.ExternalStream)."""
        return int(lib().phx_op_stream(self._h) or 0)

    def close(self):
        if getattr(self, "_h", None):
            lib().phx_op_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def part_info(self, q: int) -> dict:
        """Part q's rows [row0, row0 + nrows), its device and stream
        (phx_op_part_info; an unpartitioned operator is one part)."""
        row0, nrows, dev = C.c_int64(), C.c_int64(), C.c_int32()
        st = C.c_void_p()
        _check(lib().phx_op_part_info(self._h, int(q), C.byref(row0), C.byref(nrows),
                                      C.byref(dev), C.byref(st)))
        return {"row0": row0.value, "nrows": nrows.value, "device": dev.value,
                "stream": int(st.value or 0)}

    def apply(self, X):
        X = np.asarray(X, dtype=np.float64)
        vec = X.ndim == 1
        X = np.asfortranarray(X.reshape(self.n, -1) if not vec else X.reshape(self.n, 1))
        Y = np.empty_like(X, order="F")
        _check(lib().phx_apply(self._h, _d(X), self.n, X.shape[1], _d(Y), self.n))
        return Y[:, 0] if vec else Y

    def shifted_apply(self, xi, X):
        X = np.asarray(X, dtype=np.float64)
        vec = X.ndim == 1
        X = np.asfortranarray(X.reshape(self.n, -1))
        Y = np.empty_like(X, order="F")
        _check(lib().phx_shifted_apply(self._h, float(xi), _d(X), self.n, X.shape[1], _d(Y),
                                       self.n))
        return Y[:, 0] if vec else Y


class PowerBasis:
    """Device-resident guarded power basis (params.hpp:22-29)."""

    def __init__(self, op: CsrOperator, m=61, delta=0.8):
        h = C.c_void_p()
        _check(lib().phx_basis_build(op._h, m, delta, C.byref(h)))
        self._h = h
        self.op = op
        r, mm, s0 = C.c_int32(), C.c_int32(), C.c_double()
        _check(lib().phx_basis_info(h, C.byref(r), C.byref(mm), C.byref(s0), None, None, None))
        self.r, self.m, self.s0 = r.value, mm.value, s0.value
        logs = np.zeros(max(1, self.r))
        lb = np.zeros(self.m + 1)
        _check(lib().phx_basis_info(h, None, None, None, _d(logs), _d(lb), None))
        self.logs = logs[: self.r]
        self.log_binom = lb

    @property
    def columns(self):
        out = np.empty((self.op.n, self.m + 1), order="F")
        _check(lib().phx_basis_info(self._h, None, None, None, None, None, _d(out)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().phx_basis_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_power_basis(op: CsrOperator, m=61, delta=0.8) -> PowerBasis:
    return PowerBasis(op, m, delta)


def objective(basis: PowerBasis, xi) -> float:
    f = C.c_double()
    _check(lib().phx_objective(basis._h, float(xi), C.byref(f)))
    return f.value


def minimize_shift(basis: PowerBasis, with_path=False):
    xi, fm = C.c_double(), C.c_double()
    if with_path:
        cap = 4096
        path = np.empty(cap)
        ln = C.c_int64()
        _check(lib().phx_minimize_shift(basis._h, C.byref(xi), C.byref(fm), _d(path), cap,
                                        C.byref(ln)))
        return xi.value, fm.value, path[: ln.value].reshape(-1, 2)
    _check(lib().phx_minimize_shift(basis._h, C.byref(xi), C.byref(fm), None, 0, None))
    return xi.value, fm.value


def parameters_for_shift(op: CsrOperator, basis: PowerBasis, xi, tol) -> ScalingShift:
    out = _SS()
    _check(lib().phx_parameters_for_shift(op._h, basis._h, float(xi), float(tol), C.byref(out)))
    return ScalingShift._from(out)


def select_parameters(op: CsrOperator, m=61, tol=-1.0, delta=0.8) -> ScalingShift:
    out = _SS()
    _check(lib().phx_select_parameters(op._h, m, float(tol), float(delta), C.byref(out)))
    return ScalingShift._from(out)


def _mkrec(cap):
    lens = np.zeros(max(1, cap), dtype=np.int32)
    rec = _Rec(0, 0, 0, lens.ctypes.data_as(i32p), cap, 0)
    return rec, lens


def _torec(rec, lens):
    return RunRecord(int(rec.s_effective), int(rec.series_len_S),
                     [int(x) for x in lens[: min(int(rec.n_sweeps), len(lens))]], int(rec.matvecs))


def _lens_cap(params: ScalingShift, t):
    tmax = float(np.max(np.abs(t))) if np.size(t) else 0.0
    prod = params.s * tmax
    if not np.isfinite(prod) or prod > 1e8:
        return 1
    return int(max(1, np.ceil(prod)))


def phimv_block(op: CsrOperator, req: BlockPhiRequest) -> BlockPhiResult:
    t = np.ascontiguousarray(np.atleast_1d(req.t), dtype=np.float64)
    alpha = np.ascontiguousarray(np.atleast_1d(req.alpha), dtype=np.float64)
    if alpha.size != t.size:
        raise ValueError("phimv_block: t and alpha lengths differ")
    V = np.asarray(req.V, dtype=np.float64)
    if V.ndim == 1:
        V = V.reshape(-1, 1)
    if V.shape[1] < 1:
        raise ValueError("phimv_block: V must have at least one column")
    if V.shape[0] != op.n:
        raise ValueError("phimv_block: V row count does not match operator")
    V = np.asfortranarray(V)
    r = t.size
    W = np.empty((op.n, max(r, 1)), order="F")
    rec, lens = _mkrec(_lens_cap(req.params, t))
    ss = req.params._c()
    _check(lib().phx_phimv_block(op._h, r, _d(t), _d(alpha), V.shape[1] - 1, _d(V), op.n,
                                 float(req.tol), C.byref(ss), _d(W), op.n, C.byref(rec)))
    return BlockPhiResult(W, _torec(rec, lens))


def phimv_block_device(op: CsrOperator, t, alpha, p, d_V_ptr: int, tol, params: ScalingShift,
                       d_W_ptr: int) -> RunRecord:
    """Device-resident evaluation (phx_phimv_block_device): d_V_ptr / d_W_ptr
    are raw device pointers (e.g. torch.Tensor.data_ptr())."""
    t = np.ascontiguousarray(np.atleast_1d(t), dtype=np.float64)
    alpha = np.ascontiguousarray(np.atleast_1d(alpha), dtype=np.float64)
    rec, lens = _mkrec(_lens_cap(params, t))
    ss = params._c()
    _check(lib().phx_phimv_block_device(op._h, t.size, _d(t), _d(alpha), int(p),
                                        C.c_void_p(d_V_ptr), float(tol), C.byref(ss),
                                        C.c_void_p(d_W_ptr), C.byref(rec)))
    return _torec(rec, lens)


def phimv_block_device_parts(op: CsrOperator, t, alpha, p, d_V_ptrs, tol, params: ScalingShift,
                             d_W_ptrs) -> RunRecord:
    """Distributed device-resident evaluation (phx_phimv_block_device_parts):
    d_V_ptrs[q] / d_W_ptrs[q] are part q's row slices on its device,
    column-major with leading dimension part_info(q)["nrows"]."""
    t = np.ascontiguousarray(np.atleast_1d(t), dtype=np.float64)
    alpha = np.ascontiguousarray(np.atleast_1d(alpha), dtype=np.float64)
    rec, lens = _mkrec(_lens_cap(params, t))
    ss = params._c()
    vp = (C.c_void_p * len(d_V_ptrs))(*[C.c_void_p(int(x)) for x in d_V_ptrs])
    wp = (C.c_void_p * len(d_W_ptrs))(*[C.c_void_p(int(x)) for x in d_W_ptrs])
    _check(lib().phx_phimv_block_device_parts(op._h, t.size, _d(t), _d(alpha), int(p), vp,
                                              float(tol), C.byref(ss), wp, C.byref(rec)))
    return _torec(rec, lens)


def phimv(op: CsrOperator, req: PhiRequest) -> PhiResult:
    V = np.asarray(req.V, dtype=np.float64)
    if V.ndim == 1:
        V = V.reshape(-1, 1)
    V = np.asfortranarray(V)
    if V.shape[0] != op.n:
        raise ValueError("phimv: V row count does not match operator")
    w = np.empty(op.n)
    e0 = np.empty(op.n)
    tail = np.empty(op.n)
    rec, lens = _mkrec(_lens_cap(req.params, [req.t]))
    ss = req.params._c()
    _check(lib().phx_phimv(op._h, float(req.t), float(req.alpha), V.shape[1] - 1, _d(V), op.n,
                           float(req.tol), C.byref(ss), _d(w), _d(e0), _d(tail), C.byref(rec)))
    return PhiResult(w, e0, tail, _torec(rec, lens))


def last_eval_mode() -> int:
    """0: one grid-wide launch, 1: partitioned cooperative launches,
    2: partitioned operator as one thread-block cluster (shared-memory blocks)."""
    return int(lib().phx_last_eval_mode())


def last_eval_variant() -> dict:
    """The kernel variant of the last single-device evaluation."""
    out = (C.c_int32 * 8)()
    _check(lib().phx_last_eval_variant(out))
    keys = ("Q", "V", "R", "dynamic_tail", "latency_mode", "short_batch", "grid", "block")
    return dict(zip(keys, (int(x) for x in out)))


def tile_plan(n, row_ptr, col_idx, row0=0, nrows=None):
    """The bulk-copy evaluator's tile plan of a host CSR (built on the host,
    as phx_op_create_csr builds it) -- or, with row0 / nrows, of the row part
    [row0, row0 + nrows) as phx_op_create_csr_partitioned builds it (tiles and
    slots part-local, source rows global): (info dict, desc (tiles x 16),
    slot (part nnz + 16 bytes), sgl) -- arrays None when the plan does not
    fit."""
    nrows = int(n) - int(row0) if nrows is None else int(nrows)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    info = np.zeros(7, dtype=np.int32)
    i32 = C.POINTER(C.c_int32)
    i64p = C.POINTER(C.c_int64)
    L = lib()
    args = (int(n), rp.ctypes.data_as(i64p), ci.ctypes.data_as(i32), int(row0), nrows)
    _check(L.phx_tile_plan_part(*args, info.ctypes.data_as(i32), None, None, None))
    keys = ("ok", "tiles", "rows", "singles_cap", "emax", "singles", "T")
    d = dict(zip(keys, (int(x) for x in info)))
    if not d["ok"]:
        return d, None, None, None
    desc = np.zeros((d["tiles"], 16), dtype=np.int32)
    slot = np.zeros(int(rp[row0 + nrows] - rp[row0]) + 16, dtype=np.uint8)
    sgl = np.zeros(d["singles"] + 1, dtype=np.int32)
    _check(L.phx_tile_plan_part(*args, info.ctypes.data_as(i32), desc.ctypes.data_as(i32),
                                slot.ctypes.data_as(C.POINTER(C.c_uint8)), sgl.ctypes.data_as(i32)))
    return d, desc, slot, sgl


def last_eval_stats():
    ms = C.c_double()
    steps = C.c_int64()
    lib().phx_last_eval_stats(C.byref(ms), C.byref(steps))
    return ms.value, steps.value


def set_trace(capacity: int):
    lib().phx_set_trace(int(capacity))


def get_trace(capacity: int = 3 * 200000):
    out = np.empty(capacity)
    ln = C.c_int64()
    lib().phx_get_trace(_d(out), capacity, C.byref(ln))
    return out[: ln.value].reshape(-1, 3)


# ---------------------------------------------------------------------------
# seeded synthetic workloads (BASELINE.json configs; csrc/workloads.cpp)
# ---------------------------------------------------------------------------
def _wl():
    global _WL
    if _WL is None:
        path = os.path.join(_LIBDIR, "libphx_workloads.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing; run __graft_entry__.build()")
        L = C.CDLL(path)
        L.phx_wl_info_get.argtypes = [C.c_int32, C.c_int64, C.POINTER(_WlInfo)]
        L.phx_wl_fill.argtypes = [C.c_int32, C.c_int64, i64p, i32p, dp, dp, dp, dp]
        _WL = L
    return _WL


@dataclass
class Workload:
    cfg: int
    size: int
    n: int
    nnz: int
    p: int
    r: int
    tol: float
    rp: np.ndarray
    ci: np.ndarray
    av: np.ndarray
    V: Optional[np.ndarray]
    t: np.ndarray
    alpha: np.ndarray


def workload(cfg: int, size: int = 0, with_V: bool = True) -> Workload:
    """BASELINE.json config `cfg` (1..5) at its full size (size=0) or a
    reduced size parameter (C1: N, C2/C3: grid N, C4/C5: n)."""
    info = _WlInfo()
    if _wl().phx_wl_info_get(cfg, size, C.byref(info)) != 0:
        raise ValueError(f"unknown workload {cfg} / size {size}")
    n, nnz, p, r = info.n, info.nnz, info.p, info.r
    rp = np.empty(n + 1, dtype=np.int64)
    ci = np.empty(nnz, dtype=np.int32)
    av = np.empty(nnz, dtype=np.float64)
    V = np.empty((n, p + 1), order="F") if with_V else None
    t = np.empty(r)
    alpha = np.empty(r)
    code = _wl().phx_wl_fill(cfg, size, rp.ctypes.data_as(i64p), ci.ctypes.data_as(i32p), _d(av),
                             _d(V) if with_V else None, _d(t), _d(alpha))
    if code != 0:
        raise RuntimeError(f"workload generator failed ({code})")
    return Workload(cfg, int(info.size), n, nnz, p, r, info.tol, rp, ci, av, V, t, alpha)


# ---------------------------------------------------------------------------
# The evaluator's consumer: the expRK4s6 integrator
# (include/phiact/integrator.hpp) on the ADR problem (problems.hpp:46-70),
# device-resident through phx_exprk4s6_step / phx_integrate.
class ExpRK4s6Coefficients:
    """Stage abscissae (integrator.hpp:13-19)."""
    c2 = 0.5
    c3 = 0.5
    c4 = 1.0 / 3.0
    c5 = 5.0 / 6.0
    c6 = 1.0 / 3.0


@dataclass
class ADRProblem:
    """u_t = A u + gamma u (u - 1/2)(1 - u) with A a CsrOperator
    (problems.hpp:46-66; the operator is stored as CSR, csrc/problems.cpp)."""
    nx: int
    ny: int
    eps: float
    alpha_adv: float
    gamma: float
    op: "CsrOperator"
    u0: np.ndarray
    t_end: float = 0.5

    def reaction(self, u):
        """Pointwise reaction gamma u (u - 1/2)(1 - u) (problems.cpp:180-182)."""
        u = np.asarray(u, dtype=np.float64)
        return self.gamma * u * (u - 0.5) * (1.0 - u)


def adr_csr(nx: int, ny: int, eps: float = 1e-3, alpha_adv: float = -0.5):
    """(row_ptr, col_idx, vals, u0) of adr_build's operator (phx_adr_csr)."""
    n = int(nx) * int(ny)
    rp = np.zeros(n + 1, dtype=np.int64)
    ci = np.zeros(max(1, 5 * n), dtype=np.int32)
    av = np.zeros(max(1, 5 * n), dtype=np.float64)
    u0 = np.zeros(n, dtype=np.float64)
    code = lib().phx_adr_csr(int(nx), int(ny), float(eps), float(alpha_adv),
                             rp.ctypes.data_as(i64p), ci.ctypes.data_as(i32p), _d(av), _d(u0))
    if code != 0:
        raise ValueError("adr_build: grid must be at least 8x8")
    nnz = int(rp[n])
    return rp, ci[:nnz].copy(), av[:nnz].copy(), u0


def adr_build(nx: int, ny: int, eps: float = 1e-3, alpha_adv: float = -0.5,
              gamma: float = 1000.0, device: int = -1) -> ADRProblem:
    """adr_build (problems.cpp:184-250) with a device-resident CSR operator."""
    rp, ci, av, u0 = adr_csr(nx, ny, eps, alpha_adv)
    op = CsrOperator(int(nx) * int(ny), rp, ci, av, device=device)
    return ADRProblem(int(nx), int(ny), float(eps), float(alpha_adv), float(gamma), op, u0, 0.5)


@dataclass
class StepState:
    t: float = 0.0
    u: np.ndarray = None
    h: float = 0.0


@dataclass
class StepRecord:
    t: float
    calls: list  # 4 RunRecord, one per block-evaluator call


@dataclass
class IntegrateResult:
    u: np.ndarray
    t: float
    steps: list  # StepRecord per step (empty without records)


def _rk_recs(count, params: ScalingShift, h):
    cap = _lens_cap(params, [h])
    recs = (_Rec * max(1, count))()
    lens = []
    for k in range(count):
        r, l = _mkrec(cap)
        recs[k] = r
        lens.append(l)
    return recs, lens


def exprk4s6_step(problem: ADRProblem, state: StepState, tol, params: ScalingShift):
    """One expRK4s6 step (integrator.cpp:29-105) -> (u_next, StepRecord)."""
    u = np.ascontiguousarray(state.u, dtype=np.float64)
    if u.shape != (problem.op.n,):
        raise ValueError("exprk4s6_step: state size does not match the operator")
    out = np.empty_like(u)
    recs, lens = _rk_recs(4, params, state.h)
    ss = params._c()
    _check(lib().phx_exprk4s6_step(problem.op._h, float(problem.gamma), _d(u), float(state.h),
                                   float(tol), C.byref(ss), _d(out), recs))
    return out, StepRecord(float(state.t), [_torec(recs[k], lens[k]) for k in range(4)])


def integrate(problem: ADRProblem, h, t_end, tol, params: ScalingShift,
              keep_records: bool = True) -> IntegrateResult:
    """Fixed-step integration from t = 0 to t_end (integrator.cpp:107-134)."""
    u0 = np.ascontiguousarray(problem.u0, dtype=np.float64)
    out = np.empty_like(u0)
    t = C.c_double()
    nsteps = C.c_int64()
    ss = params._c()
    count = 0
    if keep_records and h > 0 and np.isfinite(t_end / h):
        count = 4 * int(max(1, min(1000000, round(t_end / h))))
    recs, lens = _rk_recs(count, params, h)
    _check(lib().phx_integrate(problem.op._h, float(problem.gamma), _d(u0), float(h),
                               float(t_end), float(tol), C.byref(ss), _d(out), C.byref(t),
                               C.byref(nsteps), recs if count else None, count))
    steps = []
    if count:
        for k in range(int(nsteps.value)):
            steps.append(StepRecord(k * float(h),
                                    [_torec(recs[4 * k + q], lens[4 * k + q]) for q in range(4)]))
    return IntegrateResult(out, float(t.value), steps)


# ---------------------------------------------------------------------------
# Sparse Matrix Market ingestion (host-only)
def read_matrix_market(path):
    """(n, row_ptr, col_idx, vals) of a Matrix Market file: the files
    read_matrix_market accepts (matrix_market.hpp:10-16), read as CSR.
    Raises RuntimeError with the reference's diagnostics."""
    n, nnz = C.c_int64(), C.c_int64()
    bpath = os.fsencode(path)
    _check(lib().phx_mm_read_csr(bpath, C.byref(n), C.byref(nnz), None, None, None, 0))
    rp = np.empty(n.value + 1, dtype=np.int64)
    ci = np.empty(max(1, nnz.value), dtype=np.int32)
    av = np.empty(max(1, nnz.value), dtype=np.float64)
    _check(lib().phx_mm_read_csr(bpath, C.byref(n), C.byref(nnz), rp.ctypes.data_as(i64p),
                                 ci.ctypes.data_as(i32p), _d(av), ci.size))
    return n.value, rp, ci[: nnz.value], av[: nnz.value]


def write_matrix_market(path, n, row_ptr, col_idx, vals):
    """CSR -> `coordinate real general`, 17 significant digits (bit-exact round trip)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    av = np.ascontiguousarray(vals, dtype=np.float64)
    _check(lib().phx_mm_write_csr(os.fsencode(path), int(n), rp.ctypes.data_as(i64p),
                                  ci.ctypes.data_as(i32p), _d(av)))


# ---------------------------------------------------------------------------
# block_series_direct: the reference's cross-check
def phi_series_coeffs(p: int, ncoef: int) -> np.ndarray:
    """a_ij = 1/(i+j)! for i <= p, j < ncoef on phi_series_coeffs' chain
    (phi_block.cpp:158-169), as a (p+1) x ncoef table."""
    inv = [1.0]
    while len(inv) <= p + ncoef:
        inv.append(inv[-1] / float(len(inv)))
    return np.array([[inv[i + j] for j in range(ncoef)] for i in range(p + 1)], order="F")


def block_series_direct(op: CsrOperator, req: BlockPhiRequest, coeffs=None) -> np.ndarray:
    """G = sum_j A^j V D_j Gamma T^j on the device (phx_block_series_direct);
    coeffs: None (phi_series_coeffs) or a (p+1) x ncoef table of a_ij."""
    t = np.ascontiguousarray(np.atleast_1d(req.t), dtype=np.float64)
    alpha = np.ascontiguousarray(np.atleast_1d(req.alpha), dtype=np.float64)
    if alpha.size != t.size:
        raise ValueError("phimv_block: t and alpha lengths differ")
    V = np.asarray(req.V, dtype=np.float64)
    if V.ndim == 1:
        V = V.reshape(-1, 1)
    if V.shape[0] != op.n:
        raise ValueError("phimv_block: V row count does not match operator")
    V = np.asfortranarray(V)
    G = np.empty((op.n, max(1, t.size)), order="F")
    cf = None if coeffs is None else np.asfortranarray(np.asarray(coeffs, dtype=np.float64))
    _check(lib().phx_block_series_direct(op._h, t.size, _d(t), _d(alpha), V.shape[1] - 1, _d(V),
                                         op.n, float(req.tol), None if cf is None else _d(cf),
                                         0 if cf is None else cf.shape[1], _d(G), op.n))
    return G

