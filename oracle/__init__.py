"""ctypes wrapper of the CPU oracle (oracle/liboracle.so) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module; the product (paper_2509_26475_b200) never does.  The
oracle is a plain C++ restatement of the reference's select_parameters /
phimv_block / phimv (see phx_oracle.cpp for the file:line citations).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

dp = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)


class ScalingShiftC(C.Structure):
    _fields_ = [("s", C.c_double), ("xi", C.c_double), ("s0", C.c_double),
                ("f_min", C.c_double), ("m", C.c_int32), ("r", C.c_int32)]


class OracleError(Exception):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


class OracleRuntimeError(OracleError, RuntimeError):
    pass


def build():
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_rng_new.restype = C.c_void_p
        L.orc_rng_new.argtypes = [C.c_uint64]
        L.orc_rng_free.argtypes = [C.c_void_p]
        L.orc_rng_normals.argtypes = [C.c_void_p, C.c_int64, dp]
        L.orc_rng_uniforms.argtypes = [C.c_void_p, C.c_int64, dp]
        L.orc_unit_vector.argtypes = [C.c_uint64, C.c_int64, dp]
        L.orc_stable_norm.restype = C.c_double
        L.orc_stable_norm.argtypes = [dp, C.c_int64]
        L.orc_norm2.restype = C.c_double
        L.orc_norm2.argtypes = [dp, C.c_int64]
        L.orc_inf_norm.restype = C.c_double
        L.orc_inf_norm.argtypes = [dp, C.c_int64, C.c_int64, C.c_int64]
        L.orc_apply.argtypes = [C.c_int64, i64p, i32p, dp, dp, C.c_int64, dp]
        L.orc_shifted_apply.argtypes = [C.c_int64, i64p, i32p, dp, C.c_double, dp, C.c_int64, dp]
        L.orc_basis_build.restype = C.c_void_p
        L.orc_basis_build.argtypes = [C.c_int64, i64p, i32p, dp, C.c_int32, C.c_double, i32p]
        L.orc_basis_free.argtypes = [C.c_void_p]
        L.orc_basis_info.argtypes = [C.c_void_p, i32p, i32p, dp, dp, dp, dp]
        L.orc_objective.argtypes = [C.c_void_p, C.c_double, dp]
        L.orc_minimize_shift.argtypes = [C.c_void_p, dp, dp, dp, C.c_int64, i64p]
        L.orc_parameters_for_shift.argtypes = [C.c_int64, i64p, i32p, dp, C.c_void_p, C.c_double,
                                               C.c_double, C.POINTER(ScalingShiftC)]
        L.orc_log_shifted_power.argtypes = [C.c_int64, i64p, i32p, dp, dp, C.c_double, C.c_int32, dp]
        L.orc_select_parameters.argtypes = [C.c_int64, i64p, i32p, dp, C.c_int32, C.c_double,
                                            C.c_double, C.POINTER(ScalingShiftC)]
        L.orc_phimv_block.argtypes = [C.c_int64, i64p, i32p, dp, C.c_int64, dp, dp, C.c_int32, dp,
                                      C.c_int64, C.c_double, C.POINTER(ScalingShiftC), dp,
                                      C.c_int64, i64p, i32p, C.c_int64, dp, C.c_int64, i64p]
        L.orc_phimv_block_timed.argtypes = [C.c_int64, i64p, i32p, dp, C.c_int64, dp, dp,
                                            C.c_int32, dp, C.c_int64, C.c_double,
                                            C.POINTER(ScalingShiftC), C.c_int32, C.c_int32, dp,
                                            i64p, dp]
        L.orc_set_threads.argtypes = [C.c_int32]
        L.orc_set_rowsum_order.argtypes = [C.c_int32]
        L.orc_phimv.argtypes = [C.c_int64, i64p, i32p, dp, C.c_double, C.c_double, C.c_int32, dp,
                                C.c_int64, C.c_double, C.POINTER(ScalingShiftC), dp, dp, dp, i64p,
                                i32p, C.c_int64]
        L.orc_reference_w.argtypes = [C.c_int64, dp, C.c_int32, dp, C.c_double, C.c_double, dp]
        L.orc_dense_phi.argtypes = [C.c_int64, dp, C.c_double, C.c_int32, dp]
        L.orc_jexp_chain.argtypes = [C.c_double, C.c_double, C.c_int32, dp]
        L.orc_adr_apply_stencil.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, dp, dp]
        L.orc_adr_apply_stencil.restype = None
        L.orc_adr_u0.argtypes = [C.c_int32, C.c_int32, dp]
        L.orc_adr_u0.restype = None
        L.orc_read_matrix_market.argtypes = [C.c_char_p, i64p, dp, C.c_int64]
        L.orc_block_series_direct.argtypes = [C.c_int64, i64p, i32p, dp, C.c_int64, dp, dp,
                                              C.c_int32, dp, C.c_int64, C.c_double, dp,
                                              C.c_int64, dp, C.c_int64]
        L.orc_exprk4s6_step.argtypes = [C.c_int64, i64p, i32p, dp, C.c_double, dp, C.c_double,
                                        C.c_double, C.c_void_p, dp, i64p]
        L.orc_integrate.argtypes = [C.c_int64, i64p, i32p, dp, C.c_double, dp, C.c_double,
                                    C.c_double, C.c_double, C.c_void_p, dp, dp, i64p, C.c_int64]
        _LIB = L
    return _LIB


def _check(code):
    if code == 0:
        return
    msg = lib().orc_last_error().decode()
    if code == 1:
        raise OracleInvalidArgument(msg)
    if code == 2:
        raise OracleRuntimeError(msg)
    raise OracleError(msg)


def _d(a):
    return a.ctypes.data_as(dp)


# ---------------------------------------------------------------------------
# operators
# ---------------------------------------------------------------------------
@dataclass
class Csr:
    n: int
    rp: np.ndarray   # int64, n+1
    ci: np.ndarray   # int32
    av: np.ndarray   # float64
    dense: np.ndarray | None = field(default=None, repr=False)

    def args(self):
        return (self.n, self.rp.ctypes.data_as(i64p), self.ci.ctypes.data_as(i32p), _d(self.av))


def csr_from_dense(A) -> Csr:
    """Dense matrix as a CSR operator with every entry stored in column
    order, so the CSR product is the naive ascending-k dot product."""
    A = np.ascontiguousarray(np.asarray(A, dtype=np.float64))
    n = A.shape[0]
    rp = np.arange(0, n * n + 1, n, dtype=np.int64)
    ci = np.tile(np.arange(n, dtype=np.int32), n)
    av = np.ascontiguousarray(A.reshape(-1))
    return Csr(n, rp, ci, av, dense=A)


def csr_from_arrays(n, rp, ci, av) -> Csr:
    return Csr(int(n), np.ascontiguousarray(rp, dtype=np.int64),
               np.ascontiguousarray(ci, dtype=np.int32),
               np.ascontiguousarray(av, dtype=np.float64))


# ---------------------------------------------------------------------------
# Rng
# ---------------------------------------------------------------------------
class Rng:
    """Reference Rng (rng.hpp:15-62) through the oracle: one stream."""

    def __init__(self, seed: int):
        self._h = lib().orc_rng_new(C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_rng_free(self._h)
            self._h = None

    def normals(self, count):
        out = np.empty(count, dtype=np.float64)
        lib().orc_rng_normals(self._h, count, _d(out))
        return out

    def uniforms(self, count):
        out = np.empty(count, dtype=np.float64)
        lib().orc_rng_uniforms(self._h, count, _d(out))
        return out

    def uniform(self):
        return float(self.uniforms(1)[0])

    def matrix(self, rows, cols):
        """column-major fill, returned as an (rows, cols) array"""
        return self.normals(rows * cols).reshape(cols, rows).T.copy()

    def vector(self, n):
        return self.normals(n)


def unit_vector(seed, n):
    out = np.empty(n)
    _check(lib().orc_unit_vector(C.c_uint64(seed), n, _d(out)))
    return out


def stable_norm(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().orc_stable_norm(_d(x), x.size)


def inf_norm(X):
    X = np.asfortranarray(np.atleast_2d(np.asarray(X, dtype=np.float64).T).T)
    return lib().orc_inf_norm(_d(X), X.shape[0], X.shape[1], X.shape[0])


def apply(op: Csr, X):
    X = np.asfortranarray(np.asarray(X, dtype=np.float64).reshape(op.n, -1))
    Y = np.empty_like(X, order="F")
    _check(lib().orc_apply(*op.args(), _d(X), X.shape[1], _d(Y)))
    return Y


def shifted_apply(op: Csr, xi, X):
    """shifted_apply (linop.cpp:40-49): A X, or A X - fl(xi X) when xi != 0."""
    X = np.asfortranarray(np.asarray(X, dtype=np.float64).reshape(op.n, -1))
    Y = np.empty_like(X, order="F")
    _check(lib().orc_shifted_apply(*op.args(), float(xi), _d(X), X.shape[1], _d(Y)))
    return Y


# ---------------------------------------------------------------------------
# parameter selection
# ---------------------------------------------------------------------------
@dataclass
class ScalingShift:
    s: float = 1.0
    xi: float = 0.0
    s0: float = 1.0
    f_min: float = 0.0
    m: int = 61
    r: int = 0

    def c(self):
        return ScalingShiftC(self.s, self.xi, self.s0, self.f_min, self.m, self.r)

    @staticmethod
    def from_c(c):
        return ScalingShift(c.s, c.xi, c.s0, c.f_min, c.m, c.r)

    def astuple(self):
        return (self.s, self.xi, self.s0, self.f_min, self.m, self.r)


class PowerBasis:
    def __init__(self, op: Csr, m=61, delta=0.8):
        err = C.c_int32(0)
        self.op = op
        self._h = lib().orc_basis_build(*op.args(), m, delta, C.byref(err))
        _check(err.value)
        r = C.c_int32()
        mm = C.c_int32()
        s0 = C.c_double()
        lib().orc_basis_info(self._h, C.byref(r), C.byref(mm), C.byref(s0), None, None, None)
        self.r, self.m, self.s0 = r.value, mm.value, s0.value
        self.logs = np.empty(max(self.r, 1))
        self.log_binom = np.empty(self.m + 1)
        self.columns = np.empty((op.n, self.m + 1), order="F")
        lib().orc_basis_info(self._h, C.byref(r), C.byref(mm), C.byref(s0), _d(self.logs),
                             _d(self.columns), _d(self.log_binom))
        self.logs = self.logs[: self.r]

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_basis_free(self._h)
            self._h = None

    def objective(self, xi):
        f = C.c_double()
        _check(lib().orc_objective(self._h, xi, C.byref(f)))
        return f.value

    def minimize_shift(self, with_path=False):
        xi, fm = C.c_double(), C.c_double()
        if with_path:
            path = np.empty(4096)
            ln = C.c_int64()
            _check(lib().orc_minimize_shift(self._h, C.byref(xi), C.byref(fm), _d(path), 4096,
                                            C.byref(ln)))
            return xi.value, fm.value, path[: ln.value].reshape(-1, 2)
        _check(lib().orc_minimize_shift(self._h, C.byref(xi), C.byref(fm), None, 0, None))
        return xi.value, fm.value

    def parameters_for_shift(self, xi, tol):
        out = ScalingShiftC()
        _check(lib().orc_parameters_for_shift(*self.op.args(), self._h, xi, tol, C.byref(out)))
        return ScalingShift.from_c(out)


def build_power_basis(op, m=61, delta=0.8):
    return PowerBasis(op, m, delta)


def log_shifted_power(op: Csr, v, xi, m):
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = C.c_double()
    _check(lib().orc_log_shifted_power(*op.args(), _d(v), xi, m, C.byref(out)))
    return out.value


def select_parameters(op: Csr, m=61, tol=-1.0, delta=0.8) -> ScalingShift:
    out = ScalingShiftC()
    _check(lib().orc_select_parameters(*op.args(), m, tol, delta, C.byref(out)))
    return ScalingShift.from_c(out)


# ---------------------------------------------------------------------------
# evaluators
# ---------------------------------------------------------------------------
@dataclass
class RunRecord:
    s_effective: int
    series_len_S: int
    series_lens_F: list
    matvecs: int


def _rec(rec4, lens):
    return RunRecord(int(rec4[0]), int(rec4[1]), [int(x) for x in lens[: int(rec4[2])]], int(rec4[3]))


def phimv_block(op: Csr, t, alpha, V, tol, params: ScalingShift, trace=False, lens_cap=1 << 16):
    t = np.ascontiguousarray(t, dtype=np.float64)
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    V = np.asfortranarray(np.asarray(V, dtype=np.float64).reshape(op.n, -1))
    r = t.size
    W = np.empty((op.n, r), order="F")
    rec4 = np.zeros(4, dtype=np.int64)
    lens = np.zeros(lens_cap, dtype=np.int32)
    pc = params.c()
    if trace:
        cap = 3 * 200000
        tr = np.empty(cap)
        tl = C.c_int64()
        _check(lib().orc_phimv_block(*op.args(), r, _d(t), _d(alpha), V.shape[1] - 1, _d(V),
                                     op.n, tol, C.byref(pc), _d(W), op.n,
                                     rec4.ctypes.data_as(i64p), lens.ctypes.data_as(i32p), lens_cap,
                                     _d(tr), cap, C.byref(tl)))
        return W, _rec(rec4, lens), tr[: tl.value].reshape(-1, 3)
    _check(lib().orc_phimv_block(*op.args(), r, _d(t), _d(alpha), V.shape[1] - 1, _d(V), op.n,
                                 tol, C.byref(pc), _d(W), op.n, rec4.ctypes.data_as(i64p),
                                 lens.ctypes.data_as(i32p), lens_cap, None, 0, None))
    return W, _rec(rec4, lens)


def set_threads(threads: int):
    """Row-parallel loops for the CPU timing arms (results stay bitwise those
    of one thread; the reference is single-threaded: 1 is its configuration)."""
    lib().orc_set_threads(int(threads))


def set_rowsum_order(order: int):
    """Test hook: the summation order of inf_norm's row sums (0 = the canonical
    pairwise tree; 1 = Eigen 3.4's packet-wise partial redux; 2 = sequential;
    3 = 1 with a sequential last odd row).  See rowsum_abs in phx_oracle.cpp."""
    lib().orc_set_rowsum_order(int(order))


def phimv_block_timed(op: Csr, t, alpha, V, tol, params: ScalingShift, max_s_terms: int = 0,
                      max_sweeps: int = 0, term_times: bool = False):
    """Timing sample: the evaluation with its phases timed, optionally stopped
    after max_s_terms S terms / max_sweeps recovery sweeps.  Returns
    (phases dict, RunRecord-like tuple[, per-S-term seconds])."""
    t = np.ascontiguousarray(t, dtype=np.float64)
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    V = np.asfortranarray(np.asarray(V, dtype=np.float64).reshape(op.n, -1))
    ph = np.zeros(9)
    rec4 = np.zeros(4, dtype=np.int64)
    tt = np.zeros(max(1, max_s_terms if max_s_terms > 0 else 512))
    pc = params.c()
    _check(lib().orc_phimv_block_timed(*op.args(), t.size, _d(t), _d(alpha), V.shape[1] - 1,
                                       _d(V), op.n, tol, C.byref(pc), int(max_s_terms),
                                       int(max_sweeps), _d(ph), rec4.ctypes.data_as(
                                           C.POINTER(C.c_int64)), _d(tt) if term_times else None))
    keys = ("setup", "s_terms", "s_terms_run", "promotion", "sweeps", "sweeps_run", "assembly",
            "first_s_term", "first_sweep")
    out = dict(zip(keys, ph.tolist())), tuple(int(x) for x in rec4)
    if term_times:
        return out + (tt[: int(ph[2])].copy(),)
    return out


def phimv(op: Csr, t, alpha, V, tol, params: ScalingShift, lens_cap=1 << 16):
    V = np.asfortranarray(np.asarray(V, dtype=np.float64).reshape(op.n, -1))
    w = np.empty(op.n)
    e0 = np.empty(op.n)
    tail = np.empty(op.n)
    rec4 = np.zeros(4, dtype=np.int64)
    lens = np.zeros(lens_cap, dtype=np.int32)
    pc = params.c()
    _check(lib().orc_phimv(*op.args(), float(t), float(alpha), V.shape[1] - 1, _d(V), op.n, tol,
                           C.byref(pc), _d(w), _d(e0), _d(tail), rec4.ctypes.data_as(i64p),
                           lens.ctypes.data_as(i32p), lens_cap))
    return w, e0, tail, _rec(rec4, lens)


def reference_w(A, V, t, alpha):
    A = np.asfortranarray(np.asarray(A, dtype=np.float64))
    n = A.shape[0]
    V = np.asfortranarray(np.asarray(V, dtype=np.float64).reshape(n, -1))
    out = np.empty(n)
    _check(lib().orc_reference_w(n, _d(A), V.shape[1] - 1, _d(V), t, alpha, _d(out)))
    return out


def dense_phi(M, t, jmax):
    M = np.asfortranarray(np.asarray(M, dtype=np.float64))
    d = M.shape[0]
    out = np.empty((jmax + 1) * d * d)
    _check(lib().orc_dense_phi(d, _d(M), t, jmax, _d(out)))
    return [out[k * d * d:(k + 1) * d * d].reshape(d, d, order="F") for k in range(jmax + 1)]


def jexp_chain(alpha, s, p):
    out = np.empty(p + 1)
    lib().orc_jexp_chain(alpha, s, p, _d(out))
    return out


# ---------------------------------------------------------------------------
# the evaluator's consumer: integrator.cpp restated
def adr_apply_stencil(nx, ny, eps, alpha_adv, u):
    """adr_build's matrix-free apply (problems.cpp:206-231), restated."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    y = np.empty_like(u)
    lib().orc_adr_apply_stencil(nx, ny, eps, alpha_adv, _d(u), _d(y))
    return y


def adr_u0(nx, ny):
    """adr_build's initial condition (problems.cpp:239-246)."""
    out = np.empty(nx * ny)
    lib().orc_adr_u0(nx, ny, _d(out))
    return out


def _recs(rec4):
    return [RunRecord(int(r[0]), int(r[1]), [], int(r[3])) for r in rec4.reshape(-1, 4)]


def exprk4s6_step(op: Csr, gamma, u, h, tol, params: ScalingShift):
    """exprk4s6_step (integrator.cpp:29-105) -> (u_next, 4 RunRecords)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    rec4 = np.zeros(16, dtype=np.int64)
    pc = params.c()
    _check(lib().orc_exprk4s6_step(*op.args(), float(gamma), _d(u), float(h), float(tol),
                                   C.byref(pc), _d(out), rec4.ctypes.data_as(i64p)))
    return out, _recs(rec4)


def integrate(op: Csr, gamma, u0, h, t_end, tol, params: ScalingShift, keep_records=True):
    """integrate (integrator.cpp:107-134) -> (u, t, RunRecords, 4 per step)."""
    u0 = np.ascontiguousarray(u0, dtype=np.float64)
    out = np.empty_like(u0)
    t = C.c_double()
    steps = max(1, int(round(t_end / h))) if h > 0 else 1
    cap = 4 * steps if keep_records else 0
    rec4 = np.zeros(4 * max(cap, 1), dtype=np.int64)
    pc = params.c()
    _check(lib().orc_integrate(*op.args(), float(gamma), _d(u0), float(h), float(t_end),
                               float(tol), C.byref(pc), _d(out), C.byref(t),
                               rec4.ctypes.data_as(i64p) if keep_records else None, cap))
    return out, t.value, (_recs(rec4[: 4 * cap]) if keep_records else [])


def read_matrix_market(path):
    """read_matrix_market (matrix_market.cpp:37-100), restated: dense n x n."""
    n = C.c_int64()
    _check(lib().orc_read_matrix_market(str(path).encode(), C.byref(n), None, 0))
    A = np.empty((n.value, n.value), order="F")
    _check(lib().orc_read_matrix_market(str(path).encode(), C.byref(n), _d(A), A.size))
    return A


def block_series_direct(op: Csr, t, alpha, V, tol, coeffs=None):
    """block_series_direct (phi_block.cpp:172-212); coeffs None = phi_series_coeffs,
    else a (p+1) x ncoef array of a_ij."""
    t = np.ascontiguousarray(np.atleast_1d(t), dtype=np.float64)
    alpha = np.ascontiguousarray(np.atleast_1d(alpha), dtype=np.float64)
    V = np.asfortranarray(np.asarray(V, dtype=np.float64).reshape(op.n, -1))
    G = np.empty((op.n, t.size), order="F")
    cf = None if coeffs is None else np.asfortranarray(np.asarray(coeffs, dtype=np.float64))
    _check(lib().orc_block_series_direct(*op.args(), t.size, _d(t), _d(alpha), V.shape[1] - 1,
                                         _d(V), op.n, float(tol), None if cf is None else _d(cf),
                                         0 if cf is None else cf.shape[1], _d(G), op.n))
    return G

