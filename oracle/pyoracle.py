"""pyoracle — ctypes wrapper of the CPU ORACLE (liboracle.so) and of the reference's own
compiled sparse core (_ref/libsparsla_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsparsla_ref.so")

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)


class Opts(C.Structure):
    _fields_ = [("atol", C.c_double), ("rtol", C.c_double), ("max_iter", C.c_int64),
                ("preconditioner", C.c_int32), ("_pad", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("spmv_count", C.c_int64),
                ("residual_norm", C.c_double), ("converged", C.c_int32),
                ("backend", C.c_int32), ("diagnostic", C.c_char * 128)]

    def as_dict(self):
        return dict(iterations=self.iterations, spmv_count=self.spmv_count,
                    residual_norm=self.residual_norm, converged=bool(self.converged),
                    backend=self.backend, diagnostic=self.diagnostic.decode())


def _p(a, t):
    return a.ctypes.data_as(t)


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int64)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"oracle not built: {ORACLE_SO} (run make -C oracle)")
        L = C.CDLL(ORACLE_SO)
        L.orc_cdot.restype = C.c_double
        L.orc_coo_canonicalize.restype = C.c_int64
        L.orc_local_build.restype = C.c_void_p
        L.orc_local_sizes.argtypes = [C.c_void_p, _i64p]
        L.orc_local_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        R = C.CDLL(REF_SO)
        R.ref_last_error.restype = C.c_char_p
        _ref = R
    return _ref


def set_threads(n: int):
    lib().orc_set_threads(int(n))


@dataclass
class Csr:
    """CSR in the reference's int64 layout (sparse.hpp:20, 88-96)."""
    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray

    @property
    def nnz(self):
        return int(self.row_ptr[-1])

    def dense(self):
        d = np.zeros((self.nrows, self.ncols))
        for i in range(self.nrows):
            for k in range(self.row_ptr[i], self.row_ptr[i + 1]):
                d[i, self.col_idx[k]] = self.vals[k]
        return d


# ---------------- sparse core ----------------
def canonicalize(nrows, ncols, rows, cols, vals):
    rows, cols, vals = _i(rows), _i(cols), _f(vals)
    n = len(rows)
    ro, co, vo = np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n)
    m = lib().orc_coo_canonicalize(C.c_int64(nrows), C.c_int64(ncols), C.c_int64(n),
                                   _p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p),
                                   _p(ro, _i64p), _p(co, _i64p), _p(vo, _f64p))
    if m < 0:
        raise ValueError("bad COO input")
    return ro[:m].copy(), co[:m].copy(), vo[:m].copy()


def csr_from_coo(nrows, ncols, rows, cols, vals) -> Csr:
    rows, cols, vals = _i(rows), _i(cols), _f(vals)
    nnz = len(rows)
    rp = np.empty(nrows + 1, np.int64)
    ci = np.empty(nnz, np.int64)
    v = np.empty(nnz)
    lib().orc_csr_from_coo(C.c_int64(nrows), C.c_int64(nnz), _p(rows, _i64p), _p(cols, _i64p),
                           _p(vals, _f64p), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p))
    return Csr(nrows, ncols, rp, ci, v)


def csr_from_triplets(nrows, ncols, rows, cols, vals) -> Csr:
    r, c, v = canonicalize(nrows, ncols, rows, cols, vals)
    return csr_from_coo(nrows, ncols, r, c, v)


def spmv(A: Csr, x):
    x = _f(x)
    y = np.empty(A.nrows)
    lib().orc_spmv(C.c_int64(A.nrows), _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p),
                   _p(A.vals, _f64p), _p(x, _f64p), _p(y, _f64p))
    return y


def transpose(A: Csr) -> Csr:
    trp = np.empty(A.ncols + 1, np.int64)
    tci = np.empty(A.nnz, np.int64)
    tv = np.empty(A.nnz)
    lib().orc_csr_transpose(C.c_int64(A.nrows), C.c_int64(A.ncols), _p(A.row_ptr, _i64p),
                            _p(A.col_idx, _i64p), _p(A.vals, _f64p), _p(trp, _i64p),
                            _p(tci, _i64p), _p(tv, _f64p))
    return Csr(A.ncols, A.nrows, trp, tci, tv)


def jacobi(A: Csr):
    d = np.empty(A.nrows)
    lib().orc_jacobi(C.c_int64(A.nrows), _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p),
                     _p(A.vals, _f64p), _p(d, _f64p))
    return d


def cdot(a, b):
    a, b = _f(a), _f(b)
    return lib().orc_cdot(C.c_int64(len(a)), _p(a, _f64p), _p(b, _f64p))


def cdot_partials(a, b):
    a, b = _f(a), _f(b)
    m = (len(a) + 2047) // 2048
    out = np.empty(m)
    lib().orc_cdot_partials(C.c_int64(len(a)), _p(a, _f64p), _p(b, _f64p), _p(out, _f64p))
    return out


# ---------------- solvers ----------------
def _opts(atol=1e-10, rtol=0.0, max_iter=10000, precond=1):
    return Opts(float(atol), float(rtol), int(max_iter), int(precond), 0)


def cg(A: Csr, b, atol=1e-10, rtol=0.0, max_iter=10000, precond=1):
    b = _f(b)
    x = np.empty(A.nrows)
    rep = Report()
    o = _opts(atol, rtol, max_iter, precond)
    rc = lib().orc_cg(C.c_int64(A.nrows), _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p),
                      _p(A.vals, _f64p), _p(b, _f64p), _p(x, _f64p), C.byref(o), C.byref(rep))
    if rc:
        raise ValueError(f"invalid options (rc={rc})")
    return x, rep.as_dict()


def cg_fixed(A: Csr, b, iters, precond=1):
    b = _f(b)
    x = np.empty(A.nrows)
    r = np.empty(A.nrows)
    lib().orc_cg_fixed(C.c_int64(A.nrows), _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p),
                       _p(A.vals, _f64p), _p(b, _f64p), C.c_int64(iters), C.c_int32(precond),
                       _p(x, _f64p), _p(r, _f64p))
    return x, r


def bicgstab(A: Csr, b, atol=1e-10, rtol=0.0, max_iter=10000, precond=1):
    b = _f(b)
    x = np.empty(A.nrows)
    rep = Report()
    o = _opts(atol, rtol, max_iter, precond)
    rc = lib().orc_bicgstab(C.c_int64(A.nrows), _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p),
                            _p(A.vals, _f64p), _p(b, _f64p), _p(x, _f64p), C.byref(o),
                            C.byref(rep))
    if rc:
        raise ValueError(f"invalid options (rc={rc})")
    return x, rep.as_dict()


def adjoint_backward(A: Csr, x, g, backend=0, atol=1e-10, rtol=0.0, max_iter=10000, precond=1):
    x, g = _f(x), _f(g)
    gb = np.empty(A.nrows)
    gv = np.empty(A.nnz)
    rep = Report()
    o = _opts(atol, rtol, max_iter, precond)
    rc = lib().orc_adjoint_backward(C.c_int64(A.nrows), _p(A.row_ptr, _i64p),
                                    _p(A.col_idx, _i64p), _p(A.vals, _f64p), _p(x, _f64p),
                                    _p(g, _f64p), C.c_int32(backend), C.byref(o),
                                    _p(gb, _f64p), _p(gv, _f64p), C.byref(rep))
    if rc:
        raise ValueError(f"adjoint failed rc={rc}")
    return gb, gv, rep.as_dict()


# ---------------- generators ----------------
KIND = {"poisson2d": 0, "poisson3d": 1, "convdiff3d": 2, "fem2d": 3, "poisson3d_box": 4}


def gen_triplets(kind, p1, p2=0, fparam=1.0):
    k = KIND[kind]
    n = C.c_int64()
    nt = C.c_int64()
    L = lib()
    rc = L.orc_gen_triplets(C.c_int32(k), C.c_int64(p1), C.c_int64(p2), C.c_double(fparam),
                            C.byref(n), C.byref(nt), None, None, None)
    if rc:
        raise ValueError("bad generator params")
    r = np.empty(nt.value, np.int64)
    c = np.empty(nt.value, np.int64)
    v = np.empty(nt.value)
    L.orc_gen_triplets(C.c_int32(k), C.c_int64(p1), C.c_int64(p2), C.c_double(fparam),
                       C.byref(n), C.byref(nt), _p(r, _i64p), _p(c, _i64p), _p(v, _f64p))
    return n.value, r, c, v


def generate(kind, p1, p2=0, fparam=1.0) -> Csr:
    n, r, c, v = gen_triplets(kind, p1, p2, fparam)
    return csr_from_triplets(n, n, r, c, v)


def generate_csr(kind, p1, p2=0, fparam=1.0) -> Csr:
    """Same matrix as generate(), emitted straight into canonical CSR (orc_gen_csr) —
    O(nnz), no permutation sort; used at the full BASELINE sizes."""
    k = KIND[kind]
    n, nt, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    L = lib()
    rc = L.orc_gen_csr(C.c_int32(k), C.c_int64(p1), C.c_int64(p2), C.c_double(fparam), C.byref(n),
                       C.byref(nt), None, None, None, None)
    if rc:
        raise ValueError("bad generator params")
    rp = np.empty(n.value + 1, np.int64)
    ci = np.empty(nt.value, np.int64)
    v = np.empty(nt.value)
    rc = L.orc_gen_csr(C.c_int32(k), C.c_int64(p1), C.c_int64(p2), C.c_double(fparam), C.byref(n),
                       C.byref(nt), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), C.byref(nnz))
    if rc:
        raise RuntimeError(f"orc_gen_csr failed ({rc})")
    m = nnz.value
    if m != nt.value:
        ci, v = ci[:m].copy(), v[:m].copy()
    return Csr(n.value, n.value, rp, ci, v)


def gen_coords(kind, p1, p2=0):
    n = p1 * p1 if kind == "poisson2d" else (p1 - 2) * (p1 - 2)
    xs, ys = np.empty(n), np.empty(n)
    rc = lib().orc_gen_coords(C.c_int32(KIND[kind]), C.c_int64(p1), C.c_int64(p2),
                              _p(xs, _f64p), _p(ys, _f64p))
    if rc:
        raise ValueError("coords unsupported for kind")
    return xs, ys


# ---------------- distributed ----------------
def partition_contiguous(n, P):
    out = np.empty(n, np.int32)
    if lib().orc_partition_contiguous(C.c_int64(n), C.c_int32(P), _p(out, _i32p)):
        raise ValueError("invalid partition request")
    return out


def partition_rcb(xs, ys, P):
    xs, ys = _f(xs), _f(ys)
    out = np.empty(len(xs), np.int32)
    if lib().orc_partition_rcb(C.c_int64(len(xs)), _p(xs, _f64p), _p(ys, _f64p), C.c_int32(P),
                               _p(out, _i32p)):
        raise ValueError("invalid partition request")
    return out


def build_local(A: Csr, part_of, P, rank):
    part_of = np.ascontiguousarray(part_of, np.int32)
    L = lib()
    h = L.orc_local_build(C.c_int64(A.nrows), _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p),
                          _p(A.vals, _f64p), _p(part_of, _i32p), C.c_int32(P), C.c_int32(rank))
    s = np.empty(6, np.int64)
    L.orc_local_sizes(h, _p(s, _i64p))
    no, nh, nn, nnz, ns, nr = (int(t) for t in s)
    out = dict(owned=np.empty(no, np.int64), halo=np.empty(nh, np.int64),
               neighbors=np.empty(nn, np.int32), send_ptr=np.empty(nn + 1, np.int64),
               send_idx=np.empty(ns, np.int64), recv_ptr=np.empty(nn + 1, np.int64),
               recv_idx=np.empty(nr, np.int64), row_ptr=np.empty(no + 1, np.int64),
               col_idx=np.empty(nnz, np.int64), vals=np.empty(nnz))
    L.orc_local_get(C.c_void_p(h), *[_p(out[k], _i32p if out[k].dtype == np.int32 else
                                        (_f64p if out[k].dtype == np.float64 else _i64p))
                                     for k in ("owned", "halo", "neighbors", "send_ptr",
                                               "send_idx", "recv_ptr", "recv_idx", "row_ptr",
                                               "col_idx", "vals")])
    L.orc_local_free(C.c_void_p(h))
    return out


def dist_solve(A: Csr, b, part_of, P, kind="cg", atol=1e-10, rtol=0.0, max_iter=10000,
               precond=1):
    b = _f(b)
    part_of = np.ascontiguousarray(part_of, np.int32)
    x = np.empty(A.nrows)
    rep = Report()
    cnt = np.zeros(3, np.int64)
    o = _opts(atol, rtol, max_iter, precond)
    rc = lib().orc_dist_solve(C.c_int32(1 if kind == "bicgstab" else 0), C.c_int64(A.nrows),
                              _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p), _p(A.vals, _f64p),
                              _p(b, _f64p), _p(part_of, _i32p), C.c_int32(P), C.byref(o),
                              _p(x, _f64p), C.byref(rep), _p(cnt, _i64p))
    if rc:
        raise ValueError(f"dist solve failed rc={rc}")
    return x, rep.as_dict(), dict(halo_exchanges=int(cnt[0]), all_reduces=int(cnt[1]),
                                  messages=int(cnt[2]))


def dist_spmv(A: Csr, x, part_of, P):
    x = _f(x)
    part_of = np.ascontiguousarray(part_of, np.int32)
    y = np.empty(A.nrows)
    lib().orc_dist_spmv(C.c_int64(A.nrows), _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p),
                        _p(A.vals, _f64p), _p(x, _f64p), _p(part_of, _i32p), C.c_int32(P),
                        _p(y, _f64p))
    return y


def dist_adjoint(A: Csr, x, g, part_of, P, atol=1e-10, rtol=0.0, max_iter=10000, precond=1):
    x, g = _f(x), _f(g)
    part_of = np.ascontiguousarray(part_of, np.int32)
    gb = np.empty(A.nrows)
    gv = np.empty(A.nnz)
    rep = Report()
    o = _opts(atol, rtol, max_iter, precond)
    rc = lib().orc_dist_adjoint(C.c_int64(A.nrows), _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p),
                                _p(A.vals, _f64p), _p(x, _f64p), _p(g, _f64p),
                                _p(part_of, _i32p), C.c_int32(P), C.byref(o), _p(gb, _f64p),
                                _p(gv, _f64p), C.byref(rep))
    if rc == 5:
        raise ValueError("dist_adjoint requires a structurally symmetric matrix")
    if rc:
        raise ValueError(f"dist adjoint failed rc={rc}")
    return gb, gv, rep.as_dict()


# ---------------- reference (oracle/_ref) ----------------
def ref_canonicalize(nrows, ncols, rows, cols, vals):
    rows, cols, vals = _i(rows), _i(cols), _f(vals)
    n = len(rows)
    ro, co, vo = np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n)
    m = C.c_int64()
    rc = ref().ref_coo_canonicalize(C.c_int64(nrows), C.c_int64(ncols), C.c_int64(n),
                                    _p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p),
                                    C.byref(m), _p(ro, _i64p), _p(co, _i64p), _p(vo, _f64p))
    if rc:
        raise RefError(rc, ref().ref_last_error().decode())
    return ro[:m.value].copy(), co[:m.value].copy(), vo[:m.value].copy()


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def ref_csr_from_coo(nrows, ncols, rows, cols, vals):
    rows, cols, vals = _i(rows), _i(cols), _f(vals)
    n = len(rows)
    rp = np.empty(nrows + 1, np.int64)
    ci = np.empty(n, np.int64)
    v = np.empty(n)
    nbytes = C.c_int64()
    rc = ref().ref_csr_from_coo(C.c_int64(nrows), C.c_int64(ncols), C.c_int64(n),
                                _p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p),
                                _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), C.byref(nbytes))
    if rc:
        raise RefError(rc, ref().ref_last_error().decode())
    nnz = int(rp[-1])
    return Csr(nrows, ncols, rp, ci[:nnz].copy(), v[:nnz].copy()), nbytes.value


def ref_spmv(A: Csr, x, transpose=False):
    x = _f(x)
    y = np.empty(A.ncols if transpose else A.nrows)
    fn = ref().ref_spmv_transpose if transpose else ref().ref_spmv
    rc = fn(C.c_int64(A.nrows), C.c_int64(A.ncols), _p(A.row_ptr, _i64p), _p(A.col_idx, _i64p),
            _p(A.vals, _f64p), C.c_int64(len(x)), _p(x, _f64p), _p(y, _f64p))
    if rc:
        raise RefError(rc, ref().ref_last_error().decode())
    return y


def ref_transpose_coo(nrows, ncols, rows, cols, vals):
    rows, cols, vals = _i(rows), _i(cols), _f(vals)
    n = len(rows)
    ro, co, vo = np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n)
    rc = ref().ref_transpose(C.c_int64(nrows), C.c_int64(ncols), C.c_int64(n), _p(rows, _i64p),
                             _p(cols, _i64p), _p(vals, _f64p), _p(ro, _i64p), _p(co, _i64p),
                             _p(vo, _f64p))
    if rc:
        raise RefError(rc, ref().ref_last_error().decode())
    return ro, co, vo


def ref_symmetry(nrows, ncols, rows, cols, vals, tol=1e-12):
    rows, cols, vals = _i(rows), _i(cols), _f(vals)
    n = len(rows)
    s1, s2 = C.c_int32(), C.c_int32()
    R = ref()
    rc = R.ref_is_struct_sym(C.c_int64(nrows), C.c_int64(ncols), C.c_int64(n), _p(rows, _i64p),
                             _p(cols, _i64p), _p(vals, _f64p), C.byref(s1))
    rc |= R.ref_is_symmetric(C.c_int64(nrows), C.c_int64(ncols), C.c_int64(n), _p(rows, _i64p),
                             _p(cols, _i64p), _p(vals, _f64p), C.c_double(tol), C.byref(s2))
    if rc:
        raise RefError(rc, R.ref_last_error().decode())
    return bool(s1.value), bool(s2.value)


# ------------------------------------------------------------------ eigen-solver oracle --
# SPEC.md:274-327 has no executable reference; its own oracle is a dense symmetric
# eigensolver and central finite differences for Eq. 4.
def eig_sign(V):
    """largest-magnitude component of each column positive (first index on ties)."""
    V = np.array(V, dtype=np.float64, copy=True)
    for j in range(V.shape[1]):
        i = int(np.argmax(np.abs(V[:, j])))
        if V[i, j] < 0:
            V[:, j] = -V[:, j]
    return V


def eig_dense(A: Csr, k: int):
    """k smallest eigenpairs of the dense symmetric matrix (LAPACK syevd via numpy)."""
    w, U = np.linalg.eigh(A.dense())
    return w[:k], eig_sign(U[:, :k])


def eig_backward(A: Csr, V, g):
    """Eq. 4: grad_vals[e] = sum_m g_m v_m[i_e] v_m[j_e], stored-entry order."""
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_ptr))
    cols = np.asarray(A.col_idx)
    V = np.asarray(V)
    return np.einsum("em,em,m->e", V[rows], V[cols], np.asarray(g, dtype=np.float64))


def eig_fd(A: Csr, k: int, g, eps=1e-5, entries=None):
    """Central finite differences of sum_m g_m lambda_m, perturbing one STORED entry at a
    time ((i,j) and (j,i) are separate parameters).  A single-entry
    perturbation E makes A nonsymmetric; to first order d(lambda) = v^T E v, which equals
    that of its symmetric part (E + E^T)/2, so eps/2 is applied at (i,j) and (j,i) and the
    symmetric eigensolver is used (same derivative, real spectrum)."""
    Ad = A.dense()
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_ptr))
    cols = np.asarray(A.col_idx)
    idx = range(len(cols)) if entries is None else entries
    out = []
    for e in idx:
        i, j = rows[e], cols[e]
        Ap = Ad.copy(); Ap[i, j] += eps / 2; Ap[j, i] += eps / 2
        Am = Ad.copy(); Am[i, j] -= eps / 2; Am[j, i] -= eps / 2
        lp = np.linalg.eigvalsh(Ap)[:k]
        lm = np.linalg.eigvalsh(Am)[:k]
        out.append(float(np.dot(g, (lp - lm) / (2 * eps))))
    return np.array(out)
