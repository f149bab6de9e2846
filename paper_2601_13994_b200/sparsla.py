"""sparsla — Python mirror of the reference's proj/core API over libsparsla_b200.so (C ABI).

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/core/include/sparsla/sparse.hpp:18-149, errors.hpp:9-62) and the
SPEC.md contracts of the missing solve / adjoint / distributed sources:

    SparseCoo, CsrMatrix, Shape, spmv, spmv_transpose, transpose,
    is_structurally_symmetric, is_symmetric                        (sparse.hpp)
    SolveOptions, SolveReport, JacobiPreconditioner, jacobi_build,
    cg_solve, bicgstab_solve
    AdjointContext, GradientBundle, solve_forward, solve_backward
    EigenResult, eig_smallest, eig_backward
    partition_contiguous, partition_rcb, build_local
    poisson2d / poisson3d / convdiff3d / fem2d generators

Every compute call runs the sm_100a kernels; there is no CPU fallback — without a CUDA
device the device entry points raise sparsla.Error (SPARSLA_ERR_NO_DEVICE).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsparsla_b200.so")

# ----------------------------------------------------------------------------- errors --
class Error(RuntimeError):
    """sparsla::Error (errors.hpp:9-12)."""


class DimensionError(Error):
    pass


class BoundsError(Error):
    pass


class FormatError(Error):
    pass


class SingularMatrixError(Error):
    pass


class UnsupportedInputError(Error):
    pass


class InvalidArgumentError(Error):
    pass


class TransportError(Error):
    pass


_ERR = {1: DimensionError, 2: BoundsError, 3: FormatError, 4: SingularMatrixError,
        5: UnsupportedInputError, 6: InvalidArgumentError, 7: TransportError, 8: Error,
        9: TransportError, 10: Error, 11: Error}

MEM_HOST, MEM_DEVICE = 0, 1
PRECOND_NONE, PRECOND_JACOBI = 0, 1
BACKEND_CG, BACKEND_BICGSTAB = 0, 1
BACKEND_NAMES = {BACKEND_CG: "cg", BACKEND_BICGSTAB: "bicgstab"}

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p


class _Opts(C.Structure):
    _fields_ = [("atol", C.c_double), ("rtol", C.c_double), ("max_iter", C.c_int64),
                ("preconditioner", C.c_int32), ("_pad", C.c_int32)]


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("spmv_count", C.c_int64),
                ("residual_norm", C.c_double), ("converged", C.c_int32),
                ("backend", C.c_int32), ("diagnostic", C.c_char * 128)]


_lib = None


def lib():
    """Load libsparsla_b200.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `make -C paper_2601_13994_b200` "
                              "(or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        L.sparsla_last_error_message.restype = C.c_char_p
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        msg = lib().sparsla_last_error_message().decode(errors="replace")
        raise _ERR.get(rc, Error)(msg)


def _p(a, t):
    return a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def device_count() -> int:
    n = C.c_int()
    _check(lib().sparsla_device_count(C.byref(n)))
    return n.value


# ------------------------------------------------------------------------ sparse core --
@dataclass(frozen=True)
class Shape:
    rows: int = 0
    cols: int = 0


class SparseCoo:
    """Canonical COO (sparse.hpp:38-75): sorted by (row, col), duplicates summed in input
    order, explicit zeros kept.  Raises DimensionError / BoundsError like the reference."""

    def __init__(self, rows=(), cols=(), vals=(), shape: Shape | tuple = Shape(),
                 _canonical=False, device: int | None = None):
        """device: canonicalize on that GPU (radix sort, bit-identical result) instead of the
        host; the inputs are copied in and the canonical arrays copied back."""
        if isinstance(shape, tuple):
            shape = Shape(*shape)
        rows, cols, vals = _i64(rows), _i64(cols), _f64(vals)
        if not (len(rows) == len(cols) == len(vals)):
            raise DimensionError(f"coo arrays must have equal length: rows={len(rows)} "
                                 f"cols={len(cols)} vals={len(vals)}")
        if shape.rows < 0 or shape.cols < 0:
            raise DimensionError("negative matrix shape")
        self._shape = shape
        if _canonical:
            self._rows, self._cols, self._vals = rows, cols, vals
            return
        n = len(rows)
        ro, co, vo = np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n)
        m = C.c_int64()
        if device is None:
            _check(lib().sparsla_coo_canonicalize(
                C.c_int64(shape.rows), C.c_int64(shape.cols), C.c_int64(n), _p(rows, _i64p),
                _p(cols, _i64p), _p(vals, _f64p), C.byref(m), _p(ro, _i64p), _p(co, _i64p),
                _p(vo, _f64p)))
        else:
            _check(lib().sparsla_coo_canonicalize_device(
                C.c_int(device), C.c_int64(shape.rows), C.c_int64(shape.cols), C.c_int64(n),
                _p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p), C.c_int32(MEM_HOST), C.byref(m),
                _p(ro, _i64p), _p(co, _i64p), _p(vo, _f64p)))
        self._rows, self._cols, self._vals = ro[:m.value], co[:m.value], vo[:m.value]

    shape = property(lambda s: s._shape)
    nrows = property(lambda s: s._shape.rows)
    ncols = property(lambda s: s._shape.cols)
    nnz = property(lambda s: len(s._vals))
    rows = property(lambda s: s._rows)
    cols = property(lambda s: s._cols)
    vals = property(lambda s: s._vals)

    def with_values(self, vals) -> "SparseCoo":
        vals = _f64(vals)
        if len(vals) != self.nnz:
            raise DimensionError(f"with_values: expected {self.nnz} values, got {len(vals)}")
        return SparseCoo(self._rows, self._cols, vals.copy(), self._shape, _canonical=True)

    def find(self, i: int, j: int) -> int:
        lo = np.searchsorted(self._rows, i, "left")
        hi = np.searchsorted(self._rows, i, "right")
        c = lo + np.searchsorted(self._cols[lo:hi], j, "left")
        return int(c) if c < hi and self._cols[c] == j else -1

    def to_dense(self, cap: int = 1 << 24) -> np.ndarray:
        if self.nrows * self.ncols > cap:
            raise BoundsError(f"to_dense: {self.nrows}x{self.ncols} exceeds dense element cap {cap}")
        d = np.zeros((self.nrows, self.ncols))
        d[self._rows, self._cols] = self._vals
        return d


class CsrMatrix:
    """CSR (sparse.hpp:77-104).  The device copy (int32 indices, fp64 values) is uploaded on
    first use and cached per device; values are immutable like the reference's."""

    def __init__(self, nrows, ncols, row_ptr, col_idx, vals, _validated=False):
        self._shape = Shape(int(nrows), int(ncols))
        self._rp, self._ci, self._v = _i64(row_ptr), _i64(col_idx), _f64(vals)
        self._dev = {}

    @staticmethod
    def from_coo(coo: SparseCoo) -> "CsrMatrix":
        n = coo.nrows
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(coo.nnz, np.int64)
        v = np.empty(coo.nnz)
        _check(lib().sparsla_csr_from_coo(C.c_int64(n), C.c_int64(coo.ncols), C.c_int64(coo.nnz),
                                          _p(coo.rows, _i64p), _p(coo.cols, _i64p),
                                          _p(coo.vals, _f64p), _p(rp, _i64p), _p(ci, _i64p),
                                          _p(v, _f64p)))
        return CsrMatrix(n, coo.ncols, rp, ci, v)

    def to_coo(self) -> SparseCoo:
        rows = np.empty(self.nnz, np.int64)
        _check(lib().sparsla_csr_to_coo_rows(C.c_int64(self.nrows), _p(self._rp, _i64p),
                                             _p(rows, _i64p)))
        return SparseCoo(rows, self._ci.copy(), self._v.copy(), self._shape, _canonical=True)

    shape = property(lambda s: s._shape)
    nrows = property(lambda s: s._shape.rows)
    ncols = property(lambda s: s._shape.cols)
    nnz = property(lambda s: len(s._v))
    row_ptr = property(lambda s: s._rp)
    col_idx = property(lambda s: s._ci)
    vals = property(lambda s: s._v)

    def bytes(self) -> int:
        """Live-array footprint of the reference layout (sparse.cpp:129-133)."""
        return 8 * (len(self._rp) + len(self._ci) + len(self._v))

    def device(self, dev: int = 0) -> "DeviceCsr":
        if dev not in self._dev:
            self._dev[dev] = DeviceCsr(self, dev)
        return self._dev[dev]


def _xwin_dict(out):
    return {"variant": int(out[0]), "cap_x": int(out[1]), "cover": out[2] / 1e6,
            "modes": [m for m in range(4) if (int(out[3]) >> m) & 1], "stream": int(out[4]),
            "ctas_per_sm": int(out[5])}


class DeviceCsr:
    """Owning wrapper of a sparsla_dcsr handle (one GPU)."""

    def __init__(self, A: CsrMatrix | None = None, dev: int = 0, *, i32=None):
        self.h = _vp()
        self.dev = dev
        if A is not None:
            _check(lib().sparsla_dcsr_create(C.c_int(dev), C.c_int64(A.nrows), C.c_int64(A.ncols),
                                             _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p),
                                             _p(A.vals, _f64p), C.byref(self.h)))
            self.nrows, self.ncols, self.nnz = A.nrows, A.ncols, A.nnz
        else:
            nrows, ncols, rp, ci, v = i32
            rp = np.ascontiguousarray(rp, np.int32)
            ci = np.ascontiguousarray(ci, np.int32)
            v = _f64(v)
            _check(lib().sparsla_dcsr_create_i32(C.c_int(dev), C.c_int64(nrows), C.c_int64(ncols),
                                                 _p(rp, _i32p), _p(ci, _i32p), _p(v, _f64p),
                                                 C.byref(self.h)))
            self.nrows, self.ncols, self.nnz = int(nrows), int(ncols), len(v)

    def info(self):
        out = np.zeros(8, np.int64)
        _check(lib().sparsla_dcsr_info(self.h, _p(out, _i64p)))
        keys = ["nrows", "ncols", "nnz", "device_bytes", "max_block_nnz", "max_row", "variant", "ws_variant"]
        return {k: int(out[i]) for i, k in enumerate(keys)}

    def set_values(self, vals, mem=MEM_HOST):
        """SparseCoo::with_values (sparse.hpp:58-61): same pattern, new values."""
        if mem == MEM_HOST:
            v = _f64(vals)
            if len(v) != self.nnz:
                raise DimensionError(f"{len(v)} values for {self.nnz} entries")
            _check(lib().sparsla_dcsr_set_values(self.h, _p(v, _f64p), C.c_int32(MEM_HOST)))
        else:
            _check(lib().sparsla_dcsr_set_values(self.h, C.cast(C.c_void_p(vals), _f64p), C.c_int32(MEM_DEVICE)))

    def long_rows(self):
        """Rows summed warp-per-row (power-law hubs): {rows, entries, threshold}."""
        out = np.zeros(3, np.int64)
        _check(lib().sparsla_dcsr_long_rows(self.h, _p(out, _i64p)))
        return {"rows": int(out[0]), "entries": int(out[1]), "threshold": int(out[2])}

    def xwin(self):
        """x-window staging: {variant (-1 = none), cap_x (elements per round), cover (fraction
        of entries whose x operand is staged), modes (SpMV modes that use it)}."""
        out = np.zeros(8, np.int64)
        _check(lib().sparsla_dcsr_xwin(self.h, _p(out, _i64p)))
        return _xwin_dict(out)

    def dia(self):
        """Diagonal-warp SpMV (csrc/spmv_dia.cuh): {on (every SpMV mode), modes (SpMV modes
        that take it), structured (fraction of 32-row warps), bytes (matrix bytes per SpMV),
        patterns (distinct patterns of the pattern-table kernel, 0 = 48-byte table kernel)}."""
        out = np.zeros(4, np.int64)
        _check(lib().sparsla_dcsr_dia(self.h, _p(out, _i64p)))
        return {"on": int(out[0]) == 0xF, "modes": [m for m in range(4) if (int(out[0]) >> m) & 1],
                "structured": out[1] / 1e6, "bytes": int(out[2]), "patterns": int(out[3])}

    def format(self):
        """SpMV storage format: value dictionary on / distinct values / constant Jacobi diagonal."""
        out = np.zeros(3, np.int64)
        _check(lib().sparsla_dcsr_format(self.h, _p(out, _i64p)))
        return {"value_dict": bool(out[0]), "distinct_values": int(out[1]), "uniform_diag": bool(out[2])}

    def close(self):
        if self.h:
            lib().sparsla_dcsr_destroy(self.h)
            self.h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _dev_of(A, dev=0) -> DeviceCsr:
    return A if isinstance(A, DeviceCsr) else A.device(dev)


def spmv(a, x) -> np.ndarray:
    """y = A x, row-ordered accumulation (sparse.hpp:134-135), on the GPU."""
    D = _dev_of(a)
    x = _f64(x)
    if len(x) != D.ncols:
        raise DimensionError(f"spmv: x has length {len(x)}, expected {D.ncols}")
    y = np.empty(D.nrows)
    _check(lib().sparsla_spmv(D.h, _p(x, _f64p), _p(y, _f64p), C.c_int32(MEM_HOST)))
    return y


def spmv_transpose(a, x) -> np.ndarray:
    """y = A^T x (sparse.hpp:137-138), on the GPU via an explicit canonical A^T."""
    D = _dev_of(a)
    x = _f64(x)
    if len(x) != D.nrows:
        raise DimensionError(f"spmv_transpose: x has length {len(x)}, expected {D.nrows}")
    y = np.empty(D.ncols)
    _check(lib().sparsla_spmv_transpose(D.h, _p(x, _f64p), _p(y, _f64p), C.c_int32(MEM_HOST)))
    return y


def transpose(a: SparseCoo) -> SparseCoo:
    """Canonical transpose (sparse.hpp:140-141)."""
    return SparseCoo(a.cols, a.rows, a.vals, Shape(a.ncols, a.nrows))


def _symmetry(a: SparseCoo, tol):
    A = CsrMatrix.from_coo(a)
    s1, s2 = C.c_int32(), C.c_int32()
    _check(lib().sparsla_csr_symmetry(C.c_int64(A.nrows), C.c_int64(A.ncols), _p(A.row_ptr, _i64p),
                                      _p(A.col_idx, _i64p), _p(A.vals, _f64p), C.c_double(tol),
                                      C.byref(s1), C.byref(s2)))
    return bool(s1.value), bool(s2.value)


def _coo_from_handle(h) -> SparseCoo:
    nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
    try:
        _check(lib().sparsla_coo_sizes(h, C.byref(nr), C.byref(nc), C.byref(nz)))
        r, c, v = np.empty(nz.value, np.int64), np.empty(nz.value, np.int64), np.empty(nz.value)
        _check(lib().sparsla_coo_get(h, _p(r, _i64p), _p(c, _i64p), _p(v, _f64p)))
    finally:
        lib().sparsla_coo_destroy(h)
    return SparseCoo(r, c, v, Shape(nr.value, nc.value), _canonical=True)


def read_matrix_market(src) -> SparseCoo:
    """read_matrix_market (matrix_market.hpp:10-15): a path, or a text/bytes buffer."""
    h = _vp()
    if isinstance(src, (bytes, bytearray)) or (isinstance(src, str) and src.startswith("%%MatrixMarket")):
        data = src.encode() if isinstance(src, str) else bytes(src)
        _check(lib().sparsla_mtx_read_buffer(data, C.c_int64(len(data)), C.byref(h)))
    else:
        _check(lib().sparsla_mtx_read(os.fsencode(src), C.byref(h)))
    return _coo_from_handle(h)


def write_matrix_market(a: SparseCoo, path):
    """write_matrix_market (matrix_market.hpp:17-20): coordinate/real/general, %.17g."""
    _check(lib().sparsla_mtx_write(os.fsencode(path), C.c_int64(a.nrows), C.c_int64(a.ncols),
                                   C.c_int64(a.nnz), _p(_i64(a.rows), _i64p), _p(_i64(a.cols), _i64p),
                                   _p(_f64(a.vals), _f64p)))


def is_structurally_symmetric(a: SparseCoo) -> bool:
    return _symmetry(a, 0.0)[0]


def is_symmetric(a: SparseCoo, tol: float = 1e-12) -> bool:
    return _symmetry(a, tol)[1]


def dot(a, b, dev: int = 0) -> float:
    """Canonical (deterministic, launch-geometry independent) dot product on the GPU."""
    a, b = _f64(a), _f64(b)
    if len(a) != len(b):
        raise DimensionError("dot: length mismatch")
    out = C.c_double()
    _check(lib().sparsla_dot(C.c_int(dev), C.c_int64(len(a)), _p(a, _f64p), _p(b, _f64p),
                             C.c_int32(MEM_HOST), C.byref(out)))
    return out.value


# --------------------------------------------------------------------------- solvers --
@dataclass
class SolveOptions:
    """SPEC.md:127-130 (defaults: atol = 1e-10 per Listing 2, rtol = 0)."""
    atol: float = 1e-10
    rtol: float = 0.0
    max_iter: int = 10000
    preconditioner: str = "jacobi"  # "none" | "jacobi"

    def c(self) -> _Opts:
        pc = {"none": PRECOND_NONE, "jacobi": PRECOND_JACOBI}.get(self.preconditioner)
        if pc is None:
            raise InvalidArgumentError(f"unknown preconditioner {self.preconditioner!r}")
        return _Opts(float(self.atol), float(self.rtol), int(self.max_iter), pc, 0)


@dataclass
class SolveReport:
    """SPEC.md:131-134."""
    iterations: int = 0
    residual_norm: float = 0.0
    converged: bool = False
    spmv_count: int = 0
    backend: str = "cg"
    diagnostic: str = ""

    @staticmethod
    def _from(r: _Report) -> "SolveReport":
        return SolveReport(int(r.iterations), float(r.residual_norm), bool(r.converged),
                           int(r.spmv_count), BACKEND_NAMES.get(r.backend, "?"),
                           r.diagnostic.decode(errors="replace"))


@dataclass
class JacobiPreconditioner:
    inv_diag: np.ndarray


def jacobi_build(a) -> JacobiPreconditioner:
    """SPEC.md:159-167 (1/A_ii, 1.0 for missing / zero / non-finite reciprocal)."""
    D = _dev_of(a)
    if D.nrows != D.ncols:
        raise DimensionError("jacobi_build requires a square matrix")
    d = np.empty(D.nrows)
    _check(lib().sparsla_jacobi(D.h, _p(d, _f64p), C.c_int32(MEM_HOST)))
    return JacobiPreconditioner(d)


def _krylov(fn, a, b, opts):
    D = _dev_of(a)
    opts = opts or SolveOptions()
    b = _f64(b)
    if D.nrows != D.ncols:
        raise DimensionError("solve requires a square matrix")
    if len(b) != D.nrows:
        raise DimensionError(f"rhs has length {len(b)}, expected {D.nrows}")
    x = np.empty(D.nrows)
    rep = _Report()
    o = opts.c()
    _check(fn(D.h, _p(b, _f64p), _p(x, _f64p), C.byref(o), C.byref(rep), C.c_int32(MEM_HOST)))
    return x, SolveReport._from(rep)


def cg_solve(a, b, opts: SolveOptions | None = None):
    """Jacobi-PCG from x0 = 0 -> (x, SolveReport)."""
    return _krylov(lib().sparsla_cg_solve, a, b, opts)


def bicgstab_solve(a, b, opts: SolveOptions | None = None):
    """Right-Jacobi BiCGStab from x0 = 0 -> (x, SolveReport)."""
    return _krylov(lib().sparsla_bicgstab_solve, a, b, opts)


# --------------------------------------------------------------------------- adjoint --
@dataclass
class AdjointContext:
    """Exactly (A, x) — no per-iteration state (Theorem 1)."""
    matrix: SparseCoo
    x: np.ndarray
    backend: str = "cg"
    _csr: CsrMatrix | None = field(default=None, repr=False)


@dataclass
class GradientBundle:
    grad_b: np.ndarray
    grad_vals: np.ndarray
    report: SolveReport | None = None


def solve_forward(a: SparseCoo, b, opts: SolveOptions | None = None, backend: str | None = None):
    """by default CG on a structurally symmetric pattern, else BiCGStab
    (auto_solve's iterative branch, SPEC.md:180 — note it picks CG for value-nonsymmetric
    matrices with a symmetric pattern; pass backend="bicgstab" for those).  Raises Error if
    the solve does not converge."""
    csr = CsrMatrix.from_coo(a)
    if backend is None:
        backend = "cg" if is_structurally_symmetric(a) else "bicgstab"
    fn = cg_solve if backend == "cg" else bicgstab_solve
    x, rep = fn(csr, b, opts)
    if not rep.converged:
        raise Error(f"forward solve did not converge: {rep.diagnostic}")
    return x, AdjointContext(a, x, backend, csr), rep


def solve_backward(ctx: AdjointContext, grad_x, opts: SolveOptions | None = None,
                   backend: str | None = None) -> GradientBundle:
    """one solve A^T lam = grad_x; grad_b = lam;
    grad_vals[k] = -lam[i_k] * x[j_k] over the stored entries (canonical COO order)."""
    opts = opts or SolveOptions()
    csr = ctx._csr or CsrMatrix.from_coo(ctx.matrix)
    D = csr.device(0)
    g = _f64(grad_x)
    if len(g) != D.nrows:
        raise DimensionError("grad_x length mismatch")
    x = _f64(ctx.x)
    gb = np.empty(D.nrows)
    gv = np.empty(D.nnz)
    rep = _Report()
    o = opts.c()
    be = {"cg": BACKEND_CG, "bicgstab": BACKEND_BICGSTAB}[backend or ctx.backend]
    _check(lib().sparsla_adjoint_backward(D.h, _p(x, _f64p), _p(g, _f64p), C.c_int32(be),
                                          C.byref(o), _p(gb, _f64p), _p(gv, _f64p), C.byref(rep),
                                          C.c_int32(MEM_HOST)))
    r = SolveReport._from(rep)
    if not r.converged:
        raise Error(f"adjoint solve did not converge: {r.diagnostic}")
    return GradientBundle(gb, gv, r)


# ---------------------------------------------------------------------- eigen-solver --
class _EigOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int64), ("seed", C.c_uint64),
                ("preconditioner", C.c_int32), ("_pad", C.c_int32)]


class _EigReport(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("spmm_count", C.c_int64),
                ("converged_pairs", C.c_int64), ("converged", C.c_int32),
                ("method", C.c_int32), ("diagnostic", C.c_char * 128)]


@dataclass
class EigenReport:
    """EigenResult.report: iterations, per-pair residual norms and flags."""
    iterations: int = 0
    residual_norms: np.ndarray = field(default_factory=lambda: np.zeros(0))
    pair_converged: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=bool))
    converged: bool = False
    spmm_count: int = 0
    method: str = "lobpcg"
    diagnostic: str = ""


@dataclass
class EigenResult:
    """lambdas ascending (k), vectors n x k (column m = v_m, unit norm,
    largest-magnitude component positive), report."""
    lambdas: np.ndarray
    vectors: np.ndarray
    report: EigenReport


def eig_smallest(a, k: int, tol: float = 1e-8, max_iter: int = 10000, seed: int = 2601,
                 preconditioner: str = "jacobi") -> EigenResult:
    """k smallest eigenpairs of a symmetric sparse matrix: Jacobi-
    preconditioned LOBPCG on the GPU (dense Rayleigh-Ritz on the full space below the dense
    threshold).  Non-symmetric input raises UnsupportedInputError; non-convergence returns
    the partial result with per-pair flags."""
    if isinstance(a, SparseCoo):
        a = CsrMatrix.from_coo(a)
    pc = {"none": PRECOND_NONE, "jacobi": PRECOND_JACOBI}.get(preconditioner)
    if pc is None:
        raise InvalidArgumentError(f"unknown preconditioner {preconditioner!r}")
    k = int(k)
    n = a.nrows
    if k < 1 or k > max(n, 0):
        raise InvalidArgumentError("eig_smallest: need 1 <= k <= n")
    D = _dev_of(a)
    lam = np.empty(k)
    V = np.empty((n, k))
    res = np.empty(k)
    conv = np.empty(k, dtype=np.int32)
    o = _EigOpts(float(tol), int(max_iter), int(seed) & ((1 << 64) - 1), pc, 0)
    rep = _EigReport()
    _check(lib().sparsla_eig_smallest(D.h, C.c_int64(k), C.byref(o), _p(lam, _f64p), _p(V, _f64p),
                                      _p(res, _f64p), _p(conv, _i32p), C.byref(rep),
                                      C.c_int32(MEM_HOST)))
    r = EigenReport(int(rep.iterations), res, conv.astype(bool), bool(rep.converged),
                    int(rep.spmm_count), "dense" if rep.method == 1 else "lobpcg",
                    rep.diagnostic.decode(errors="replace"))
    return EigenResult(lam, V, r)


def eig_backward(result: EigenResult, a_pattern, grad_lambdas) -> np.ndarray:
    """Eq. 4: grad_vals[e] = sum_m grad_lambdas[m] v_m[i_e] v_m[j_e] over
    the stored entries of a_pattern (canonical COO order); no linear solves.  Requires all
    pairs converged and simple eigenvalues (gap > 1e-8), else raises."""
    if isinstance(a_pattern, SparseCoo):
        a_pattern = CsrMatrix.from_coo(a_pattern)
    lam = _f64(result.lambdas)
    k = len(lam)
    g = _f64(grad_lambdas)
    if len(g) != k:
        raise DimensionError(f"grad_lambdas has length {len(g)}, expected {k}")
    V = _f64(result.vectors)
    if V.shape != (a_pattern.nrows, k):
        raise DimensionError(f"vectors shape {V.shape}, expected {(a_pattern.nrows, k)}")
    if not bool(np.all(result.report.pair_converged)):
        raise InvalidArgumentError("eig_backward: not all eigenpairs converged")
    D = _dev_of(a_pattern)
    gv = np.empty(D.nnz)
    _check(lib().sparsla_eig_backward(D.h, C.c_int64(k), _p(lam, _f64p), _p(V, _f64p), _p(g, _f64p),
                                      _p(gv, _f64p), C.c_int32(MEM_HOST)))
    return gv


# --------------------------------------------------------------- persistent solver ---
class Solver:
    """Device-resident solver (b, x, work vectors in HBM, graph-captured iteration)."""

    def __init__(self, a, b, backend="cg", opts: SolveOptions | None = None, mem=MEM_HOST):
        self.D = _dev_of(a)
        self.h = _vp()
        o = (opts or SolveOptions()).c()
        be = {"cg": BACKEND_CG, "bicgstab": BACKEND_BICGSTAB}[backend]
        ptr = _p(_f64(b), _f64p) if mem == MEM_HOST else C.cast(C.c_void_p(b), _f64p)
        _check(lib().sparsla_solver_create(self.D.h, C.c_int32(be), ptr, C.c_int32(mem),
                                           C.byref(o), C.byref(self.h)))

    def reset(self):
        _check(lib().sparsla_solver_reset(self.h))

    def iterate(self, n):
        _check(lib().sparsla_solver_iterate(self.h, C.c_int64(n)))

    def run(self):
        _check(lib().sparsla_solver_run(self.h))

    def report(self) -> SolveReport:
        r = _Report()
        _check(lib().sparsla_solver_report(self.h, C.byref(r)))
        return SolveReport._from(r)

    def x(self) -> np.ndarray:
        out = np.empty(self.D.nrows)
        _check(lib().sparsla_solver_get_x(self.h, _p(out, _f64p), C.c_int32(MEM_HOST)))
        return out

    def stream(self) -> int:
        s = _vp()
        _check(lib().sparsla_solver_stream(self.h, C.byref(s)))
        return s.value or 0

    def kernel_times(self, iters: int) -> list:
        """Average duration (ms) of each kernel of an iteration, CUDA events per kernel."""
        L = self.launches_per_iteration()
        out = np.zeros(L)
        _check(lib().sparsla_solver_kernel_times(self.h, C.c_int64(iters), _p(out, _f64p)))
        return list(out)

    def launches_per_iteration(self) -> int:
        n = C.c_int64()
        _check(lib().sparsla_solver_launches_per_iteration(self.h, C.byref(n)))
        return n.value

    def close(self):
        if self.h:
            lib().sparsla_solver_destroy(self.h)
            self.h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------- generators ---
KIND = {"poisson2d": 0, "poisson3d": 1, "convdiff3d": 2, "fem2d": 3, "poisson3d_box": 4}


def gen_size(kind, p1, p2=0, fparam=1.0, row_begin=0, row_end=None):
    n = C.c_int64()
    nnz = C.c_int64()
    if row_end is None:
        _check(lib().sparsla_gen_size(C.c_int32(KIND[kind]), C.c_int64(p1), C.c_int64(p2),
                                      C.c_double(fparam), C.c_int64(0), C.c_int64(0),
                                      C.byref(n), C.byref(nnz)))
        row_end = n.value
    _check(lib().sparsla_gen_size(C.c_int32(KIND[kind]), C.c_int64(p1), C.c_int64(p2),
                                  C.c_double(fparam), C.c_int64(row_begin), C.c_int64(row_end),
                                  C.byref(n), C.byref(nnz)))
    return n.value, nnz.value, row_end


def generate(kind, p1, p2=0, fparam=1.0, row_begin=0, row_end=None) -> CsrMatrix:
    """Canonical CSR rows [row_begin, row_end) of a generated problem (global columns)."""
    n, nnz, row_end = gen_size(kind, p1, p2, fparam, row_begin, row_end)
    nr = row_end - row_begin
    rp = np.empty(nr + 1, np.int64)
    ci = np.empty(nnz, np.int64)
    v = np.empty(nnz)
    _check(lib().sparsla_gen_csr(C.c_int32(KIND[kind]), C.c_int64(p1), C.c_int64(p2),
                                 C.c_double(fparam), C.c_int64(row_begin), C.c_int64(row_end),
                                 _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p)))
    return CsrMatrix(nr, n, rp, ci, v)


def generate_i32(kind, p1, p2=0, fparam=1.0, row_begin=0, row_end=None):
    """Same as generate() in the device's int32 layout (no int64 host copy)."""
    n, nnz, row_end = gen_size(kind, p1, p2, fparam, row_begin, row_end)
    nr = row_end - row_begin
    rp = np.empty(nr + 1, np.int32)
    ci = np.empty(nnz, np.int32)
    v = np.empty(nnz)
    _check(lib().sparsla_gen_csr_i32(C.c_int32(KIND[kind]), C.c_int64(p1), C.c_int64(p2),
                                     C.c_double(fparam), C.c_int64(row_begin), C.c_int64(row_end),
                                     _p(rp, _i32p), _p(ci, _i32p), _p(v, _f64p)))
    return nr, n, rp, ci, v


def poisson2d(N: int):
    """SPEC.md:561-569 -> (CsrMatrix, rhs = ones)."""
    A = generate("poisson2d", N)
    return A, np.ones(A.nrows)


def gen_coords(kind, p1, p2=0):
    n = p1 * p1 if kind == "poisson2d" else (p1 - 2) * (p1 - 2)
    xs, ys = np.empty(n), np.empty(n)
    _check(lib().sparsla_gen_coords(C.c_int32(KIND[kind]), C.c_int64(p1), C.c_int64(p2),
                                    _p(xs, _f64p), _p(ys, _f64p)))
    return xs, ys


# ---------------------------------------------------------------------- distributed ---
def partition_contiguous(n: int, P: int) -> np.ndarray:
    out = np.empty(n, np.int32)
    _check(lib().sparsla_partition_contiguous(C.c_int64(n), C.c_int32(P), _p(out, _i32p)))
    return out


def partition_rcb(xs, ys, P: int) -> np.ndarray:
    xs, ys = _f64(xs), _f64(ys)
    out = np.empty(len(xs), np.int32)
    _check(lib().sparsla_partition_rcb(C.c_int64(len(xs)), _p(xs, _f64p), _p(ys, _f64p),
                                       C.c_int32(P), _p(out, _i32p)))
    return out


@dataclass
class LocalPartition:
    """owned/halo sets, HaloMap per neighbour, local [owned|halo] matrix."""
    rank: int
    owned: np.ndarray
    halo: np.ndarray
    neighbors: np.ndarray
    send_ptr: np.ndarray
    send_idx: np.ndarray
    recv_ptr: np.ndarray
    recv_idx: np.ndarray
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray

    def send_to(self, q):
        a = int(np.searchsorted(self.neighbors, q))
        return self.send_idx[self.send_ptr[a]:self.send_ptr[a + 1]]

    def recv_from(self, q):
        a = int(np.searchsorted(self.neighbors, q))
        return self.recv_idx[self.recv_ptr[a]:self.recv_ptr[a + 1]]


def build_local(owned_rows: CsrMatrix, owned, part_of, P: int, rank: int) -> LocalPartition:
    """build_local from this rank's rows only (global column ids); structurally symmetric
    patterns.  part_of=None means partition_contiguous(n, P)
    with n = owned_rows.ncols (the global size), without materialising the map."""
    owned = _i64(owned)
    h = _vp()
    if part_of is None:
        n_global, pp = owned_rows.ncols, None
    else:
        part_of = np.ascontiguousarray(part_of, np.int32)
        n_global, pp = len(part_of), _p(part_of, _i32p)
    _check(lib().sparsla_local_build(C.c_int64(n_global), pp, C.c_int32(P),
                                     C.c_int32(rank), C.c_int64(len(owned)), _p(owned, _i64p),
                                     _p(owned_rows.row_ptr, _i64p), _p(owned_rows.col_idx, _i64p),
                                     _p(owned_rows.vals, _f64p), C.byref(h)))
    try:
        s = np.empty(6, np.int64)
        _check(lib().sparsla_local_sizes(h, _p(s, _i64p)))
        no, nh, nn, nnz, ns, nr = (int(t) for t in s)
        o = dict(owned=np.empty(no, np.int64), halo=np.empty(nh, np.int64),
                 neighbors=np.empty(nn, np.int32), send_ptr=np.empty(nn + 1, np.int64),
                 send_idx=np.empty(ns, np.int64), recv_ptr=np.empty(nn + 1, np.int64),
                 recv_idx=np.empty(nr, np.int64), row_ptr=np.empty(no + 1, np.int64),
                 col_idx=np.empty(nnz, np.int64), vals=np.empty(nnz))
        args = []
        for k in ("owned", "halo", "neighbors", "send_ptr", "send_idx", "recv_ptr", "recv_idx",
                  "row_ptr", "col_idx", "vals"):
            a = o[k]
            args.append(_p(a, _i32p if a.dtype == np.int32 else
                           (_f64p if a.dtype == np.float64 else _i64p)))
        _check(lib().sparsla_local_get(h, *args))
    finally:
        lib().sparsla_local_destroy(h)
    return LocalPartition(rank, **o)


# ------------------------------------------------------------- distributed (device) ---
def _local_handle(rows: CsrMatrix, owned, part_of, P: int, rank: int, n_global: int):
    owned = _i64(owned)
    h = _vp()
    po = None if part_of is None else np.ascontiguousarray(part_of, np.int32)
    _check(lib().sparsla_local_build(C.c_int64(n_global),
                                     None if po is None else _p(po, _i32p), C.c_int32(P),
                                     C.c_int32(rank), C.c_int64(len(owned)), _p(owned, _i64p),
                                     _p(rows.row_ptr, _i64p), _p(rows.col_idx, _i64p),
                                     _p(rows.vals, _f64p), C.byref(h)))
    return h


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(lib().sparsla_nccl_unique_id(buf))
    return bytes(buf)


_AG_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64)
_EX_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.POINTER(C.c_double)),
                     C.POINTER(C.c_int64), C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.c_int64))


class _HostTransportC(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allgather", _AG_FN), ("exchange", _EX_FN)]


def torch_host_transport(nranks: int, group=None) -> _HostTransportC:
    """sparsla_host_transport whose collectives run on torch.distributed (gloo) — setup and
    init traffic only when the plan uses fused peer collectives."""
    import traceback

    import torch
    import torch.distributed as dist

    def ag(user, send, recv, count):
        try:
            t = torch.from_numpy(np.ctypeslib.as_array(send, shape=(count,)).copy())
            outs = [torch.empty(count, dtype=torch.float64) for _ in range(nranks)]
            dist.all_gather(outs, t, group=group)
            np.ctypeslib.as_array(recv, shape=(count * nranks,))[:] = torch.cat(outs).numpy()
            return 0
        except Exception:  # noqa: BLE001
            traceback.print_exc()
            return 1

    def ex(user, npeers, ranks, sbuf, scount, rbuf, rcount):
        try:
            reqs, outs = [], []
            for a in range(npeers):
                q = int(ranks[a])
                if scount[a]:
                    t = torch.from_numpy(np.ctypeslib.as_array(sbuf[a], shape=(scount[a],)).copy())
                    reqs.append(dist.isend(t, q, group=group))
                if rcount[a]:
                    r = torch.empty(int(rcount[a]), dtype=torch.float64)
                    reqs.append(dist.irecv(r, q, group=group))
                    outs.append((a, r))
            for rq in reqs:
                rq.wait()
            for a, r in outs:
                np.ctypeslib.as_array(rbuf[a], shape=(int(rcount[a]),))[:] = r.numpy()
            return 0
        except Exception:  # noqa: BLE001
            traceback.print_exc()
            return 1

    T = _HostTransportC(None, _AG_FN(ag), _EX_FN(ex))
    T._keep = (ag, ex)
    return T


class LocalHub:
    """In-process transport hub: P ranks as threads of this process (may share a GPU)."""

    def __init__(self, P: int):
        self.P = P
        self.h = _vp()
        _check(lib().sparsla_local_hub_create(C.c_int(P), C.byref(self.h)))

    def __del__(self):
        try:
            if self.h:
                lib().sparsla_local_hub_destroy(self.h)
        except Exception:
            pass


class DistPlan:
    """One rank of the row-partitioned solver.  Every method is
    collective over the ranks of the plan."""

    def __init__(self, h, n_owned, nnz_local, dev):
        self.h, self.n_owned, self.nnz_local, self.dev = h, n_owned, nnz_local, dev

    @staticmethod
    def create_local(hub: LocalHub, dev: int, rank: int, rows: CsrMatrix, owned, part_of,
                     n_global: int) -> "DistPlan":
        L = _local_handle(rows, owned, part_of, hub.P, rank, n_global)
        try:
            h = _vp()
            _check(lib().sparsla_dist_create_local(C.c_int(dev), hub.h, C.c_int(rank), L, C.byref(h)))
        finally:
            lib().sparsla_local_destroy(L)
        return DistPlan(h, len(owned), rows.nnz, dev)

    @staticmethod
    def create_host(dev: int, nranks: int, rank: int, transport: _HostTransportC, rows: CsrMatrix, owned,
                    part_of, n_global: int) -> "DistPlan":
        L = _local_handle(rows, owned, part_of, nranks, rank, n_global)
        try:
            h = _vp()
            _check(lib().sparsla_dist_create_host(C.c_int(dev), C.c_int(nranks), C.c_int(rank), C.byref(transport),
                                                  L, C.byref(h)))
        finally:
            lib().sparsla_local_destroy(L)
        plan = DistPlan(h, len(owned), rows.nnz, dev)
        plan._transport = transport  # callbacks must outlive the plan
        return plan

    @staticmethod
    def create_nccl(dev: int, nranks: int, rank: int, uid: bytes, rows: CsrMatrix, owned,
                    part_of, n_global: int) -> "DistPlan":
        L = _local_handle(rows, owned, part_of, nranks, rank, n_global)
        try:
            h = _vp()
            idb = (C.c_ubyte * 128).from_buffer_copy(uid)
            _check(lib().sparsla_dist_create_nccl(C.c_int(dev), C.c_int(nranks), C.c_int(rank), idb,
                                                  L, C.byref(h)))
        finally:
            lib().sparsla_local_destroy(L)
        return DistPlan(h, len(owned), rows.nnz, dev)

    def info(self):
        out = np.zeros(9, np.int64)
        _check(lib().sparsla_dist_info(self.h, _p(out, _i64p)))
        keys = ["n_owned", "n_halo", "neighbors", "interior_chunks", "boundary_chunks", "P", "rank",
                "zero_copy_segments", "n_global"]
        return {k: int(out[i]) for i, k in enumerate(keys)}

    def counters(self):
        out = np.zeros(6, np.int64)
        _check(lib().sparsla_dist_counters(self.h, _p(out, _i64p)))
        return {"halo_exchanges": int(out[0]), "all_reduces": int(out[1]), "messages": int(out[2]),
                "raw_exchanges": int(out[3]), "raw_allgathers": int(out[4]), "raw_messages": int(out[5])}

    def reset_counters(self):
        _check(lib().sparsla_dist_reset_counters(self.h))

    def format(self):
        """This rank's local-matrix storage format (see DeviceCsr.format)."""
        out = np.zeros(3, np.int64)
        _check(lib().sparsla_dist_format(self.h, _p(out, _i64p)))
        return {"value_dict": bool(out[0]), "distinct_values": int(out[1]), "uniform_diag": bool(out[2])}

    def xwin(self):
        """This rank's local-matrix x-window staging (see DeviceCsr.xwin)."""
        out = np.zeros(8, np.int64)
        _check(lib().sparsla_dist_xwin(self.h, _p(out, _i64p)))
        return _xwin_dict(out)

    def dia(self):
        """This rank's local-matrix diagonal-warp SpMV (see DeviceCsr.dia)."""
        out = np.zeros(4, np.int64)
        _check(lib().sparsla_dist_dia(self.h, _p(out, _i64p)))
        return {"on": int(out[0]) == 0xF, "modes": [m for m in range(4) if (int(out[0]) >> m) & 1],
                "structured": out[1] / 1e6, "bytes": int(out[2]), "patterns": int(out[3])}

    def set_values(self, vals_local, mem=MEM_HOST):
        """Collective: new values of this rank's local matrix (local entry order)."""
        if mem == MEM_HOST:
            v = _f64(vals_local)
            if len(v) != self.nnz_local:
                raise DimensionError(f"{len(v)} values for {self.nnz_local} local entries")
            _check(lib().sparsla_dist_set_values(self.h, _p(v, _f64p), C.c_int32(MEM_HOST)))
        else:
            _check(lib().sparsla_dist_set_values(self.h, C.cast(C.c_void_p(vals_local), _f64p),
                                                 C.c_int32(MEM_DEVICE)))

    def set_fused(self, on: bool = True):
        """Fused peer-memory collectives for CG (no NCCL call per iteration)."""
        _check(lib().sparsla_dist_set_fused(self.h, C.c_int32(1 if on else 0)))

    def spmv(self, x_owned):
        x = _f64(x_owned)
        y = np.empty(self.n_owned)
        _check(lib().sparsla_dist_spmv(self.h, _p(x, _f64p), _p(y, _f64p), C.c_int32(MEM_HOST)))
        return y

    def _solve(self, fn, b_owned, opts, out=None):
        b = _f64(b_owned)
        x = np.empty(self.n_owned) if out is None else out  # out: e.g. a pinned host buffer
        rep = _Report()
        o = (opts or SolveOptions()).c()
        _check(fn(self.h, _p(b, _f64p), _p(x, _f64p), C.byref(o), C.byref(rep), C.c_int32(MEM_HOST)))
        return x, SolveReport._from(rep)

    def cg(self, b_owned, opts: SolveOptions | None = None, out=None):
        return self._solve(lib().sparsla_dist_cg_solve, b_owned, opts, out)

    def bicgstab(self, b_owned, opts: SolveOptions | None = None, out=None):
        return self._solve(lib().sparsla_dist_bicgstab_solve, b_owned, opts, out)

    def adjoint(self, x_owned, g_owned, vals_t=None, backend="cg", opts: SolveOptions | None = None):
        x, g = _f64(x_owned), _f64(g_owned)
        gb = np.empty(self.n_owned)
        gv = np.empty(self.nnz_local)
        vt = None if vals_t is None else _f64(vals_t)
        rep = _Report()
        o = (opts or SolveOptions()).c()
        be = {"cg": BACKEND_CG, "bicgstab": BACKEND_BICGSTAB}[backend]
        _check(lib().sparsla_dist_adjoint_backward(self.h, _p(x, _f64p), _p(g, _f64p),
                                                   None if vt is None else _p(vt, _f64p), C.c_int32(be),
                                                   C.byref(o), _p(gb, _f64p), _p(gv, _f64p),
                                                   C.byref(rep), C.c_int32(MEM_HOST)))
        return gb, gv, SolveReport._from(rep)

    def gather(self, x_owned):
        """gather_solution: the global vector on rank 0, None elsewhere."""
        x = _f64(x_owned)
        n = self.info()["n_global"]
        out = np.empty(n)
        _check(lib().sparsla_dist_gather(self.h, _p(x, _f64p), _p(out, _f64p), C.c_int32(MEM_HOST)))
        return out if self.info()["rank"] == 0 else None

    def solver(self, b_owned, backend="cg", opts: SolveOptions | None = None) -> "Solver":
        sv = Solver.__new__(Solver)
        sv.D = DeviceCsr.__new__(DeviceCsr)
        sv.D.h, sv.D.dev, sv.D.nrows, sv.D.ncols = _vp(), self.dev, self.n_owned, self.n_owned
        sv.h = _vp()
        o = (opts or SolveOptions()).c()
        be = {"cg": BACKEND_CG, "bicgstab": BACKEND_BICGSTAB}[backend]
        b = _f64(b_owned)
        _check(lib().sparsla_dist_solver_create(self.h, C.c_int32(be), _p(b, _f64p), C.c_int32(MEM_HOST),
                                                C.byref(o), C.byref(sv.h)))
        return sv

    def close(self):
        if self.h:
            lib().sparsla_dist_destroy(self.h)
            self.h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_ranks(P: int, fn):
    """Run fn(rank) on P threads (the in-process worker model); returns the
    per-rank results or raises the first rank's exception."""
    import threading
    out, err = [None] * P, [None] * P

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out


def owned_rows(A: CsrMatrix, owned) -> CsrMatrix:
    """Rows `owned` of a global CSR, global column ids (a rank's input to build_local)."""
    owned = _i64(owned)
    lens = np.diff(A.row_ptr)[owned]
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    if len(owned):
        starts = A.row_ptr[owned]
        sel = np.repeat(starts - rp[:-1], lens) + np.arange(rp[-1])
    else:
        sel = np.zeros(0, np.int64)
    return CsrMatrix(len(owned), A.ncols, rp, A.col_idx[sel], A.vals[sel])
