"""torch-sla style autograd binding.

    A = SparseTensor(values, row, col, (n, n))      # values: torch tensor (requires_grad ok)
    x = A.solve(b, atol=..., rtol=...)              # differentiable w.r.t. values and b
    loss(x).backward()                              # one adjoint solve (Alg. 1, Eq. 3)
    lam, V = A.eigsh(k=6)                           # LOBPCG; d(lam)/d(values) by Eq. 4

    # one process per GPU: this rank's partition of the same triplets
    D = DSparseMatrix.from_global(values, row, col, (n, n), num_partitions=P, my_partition=rank)
    x_local = D.solve(b_local, atol=1e-10)           # distributed CG / BiCGStab, halo exchange
    x_local.sum().backward()                         # one distributed adjoint solve

Forward and backward run on the sm_100a Krylov loop through the C ABI with zero-copy device
pointers (SPARSLA_MEM_DEVICE).  Backward is exactly one transposed solve plus the per-entry
gather grad_vals[k] = -lambda[row_k] * x[col_k] (solve_backward); the
saved state is (pattern, values, x) only — no per-iteration tape (Theorem 1).  Input
triplets may be unsorted / duplicated: the pattern is canonicalised like SparseCoo
(sparse.cpp:9-53, duplicates summed in input order on the host-defined permutation) and the
gradient of every duplicate is the gradient of its canonical entry.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import sparsla as S


class SparseTensor:
    def __init__(self, values: torch.Tensor, row, col, shape, device: int | None = None):
        row = np.ascontiguousarray(torch.as_tensor(row).cpu().numpy(), np.int64)
        col = np.ascontiguousarray(torch.as_tensor(col).cpu().numpy(), np.int64)
        if values.dim() != 1 or values.numel() != len(row) or len(row) != len(col):
            raise S.DimensionError("values, row and col must be 1-D of equal length")
        if values.dtype != torch.float64:
            raise S.InvalidArgumentError("torch-sla B200 path computes in float64")
        n, m = int(shape[0]), int(shape[1])
        # canonical pattern + map input entry -> canonical entry (SparseCoo order: stable by
        # (row, col, input index)); large inputs are sorted on the GPU (radix sort, same order)
        dev = values.device.index if values.is_cuda else (device or 0)
        if len(row) >= (1 << 17):
            order = np.empty(len(row), np.int64)
            group = np.empty(len(row), np.int64)
            m_out = C.c_int64()
            S._check(S.lib().sparsla_coo_sort_device(
                C.c_int(dev), C.c_int64(int(shape[0])), C.c_int64(int(shape[1])), C.c_int64(len(row)),
                S._p(row, S._i64p), S._p(col, S._i64p), C.c_int32(S.MEM_HOST), C.byref(m_out),
                S._p(order, S._i64p), S._p(group, S._i64p)))
            new = np.ones(len(order), bool)
            if len(order):
                new[1:] = group[1:] != group[:-1]
            r_s, c_s = row[order], col[order]
        else:
            order = np.lexsort((np.arange(len(row)), col, row))
            r_s, c_s = row[order], col[order]
            new = np.ones(len(order), bool)
            if len(order):
                new[1:] = (r_s[1:] != r_s[:-1]) | (c_s[1:] != c_s[:-1])
            group = np.cumsum(new) - 1
        self._group_of_input = np.empty(len(row), np.int64)
        self._group_of_input[order] = group
        self._order = order
        if len(row) >= (1 << 17):  # bounds checked and (row, col) sorted + unique on the GPU
            coo = S.SparseCoo(r_s[new], c_s[new], np.zeros(int(new.sum())), (n, m), _canonical=True)
        else:
            coo = S.SparseCoo(r_s[new], c_s[new], np.zeros(int(new.sum())), (n, m))  # pattern check
        self.csr = S.CsrMatrix.from_coo(coo)
        self.shape = (n, m)
        self.values = values
        self.device = dev
        self._dup = bool((~new).any())
        self._order_t = None
        self._group_t = None
        self._gin_t = None

    @property
    def nnz(self):
        return self.csr.nnz

    def canonical_values(self) -> torch.Tensor:
        """Values in canonical entry order; duplicates summed in input order (SparseCoo)."""
        v = self.values
        if not v.is_cuda:
            v = v.to(f"cuda:{self.device}")
        if not self._dup:
            if self._order_t is None:
                self._order_t = torch.as_tensor(self._order, device=v.device)
            return v[self._order_t]
        # duplicates: sequential per-entry sums in input order (deterministic, exact order)
        return _DupSum.apply(v, self)

    def solve(self, b: torch.Tensor, atol: float = 1e-10, rtol: float = 0.0, max_iter: int = 10000,
              preconditioner: str = "jacobi", backend: str = "auto") -> torch.Tensor:
        if backend == "auto":
            backend = "cg" if S.is_structurally_symmetric(self.csr.to_coo()) else "bicgstab"
        opts = S.SolveOptions(atol=atol, rtol=rtol, max_iter=max_iter, preconditioner=preconditioner)
        return _Solve.apply(self.canonical_values(), b, self, opts, backend)

    def eigsh(self, k: int = 6, tol: float = 1e-8, max_iter: int = 10000, seed: int = 2601):
        """k smallest eigenpairs.  Returns (lambdas,
        vectors n x k); lambdas are differentiable w.r.t. the values (Eq. 4, no solves),
        the eigenvectors are not (eigenvector gradients are a non-goal)."""
        return _Eigsh.apply(self.canonical_values(), self, int(k), float(tol), int(max_iter), int(seed))


class _DupSum(torch.autograd.Function):
    """Canonical values of triplets with duplicates: each canonical entry is the left-to-right
    sum of its duplicates in input order (sparse.cpp:45-47), one GPU thread per entry."""

    @staticmethod
    def forward(ctx, v, A):
        v = v.detach().to(torch.float64).contiguous()
        if A._group_t is None or A._order_t.device != v.device:
            A._order_t = torch.as_tensor(A._order, device=v.device)
            A._group_t = torch.as_tensor(A._group_of_input[A._order], device=v.device)
        out = torch.empty(A.nnz, dtype=torch.float64, device=v.device)
        torch.cuda.current_stream(v.device).synchronize()  # the library runs on its own stream
        i64 = C.POINTER(C.c_int64)
        S._check(S.lib().sparsla_coo_group_sum_device(
            C.c_int(v.device.index), C.c_int64(v.numel()), C.c_int64(A.nnz),
            C.cast(C.c_void_p(A._order_t.data_ptr()), i64), C.cast(C.c_void_p(A._group_t.data_ptr()), i64),
            _ptr(v), _ptr(out)))
        ctx.A = A
        return out

    @staticmethod
    def backward(ctx, g):
        A = ctx.A
        if A._gin_t is None or A._gin_t.device != g.device:
            A._gin_t = torch.as_tensor(A._group_of_input, device=g.device)
        return g[A._gin_t], None


def _ptr(t: torch.Tensor):
    return C.cast(C.c_void_p(t.data_ptr()), S._f64p)


class _Solve(torch.autograd.Function):
    @staticmethod
    def forward(ctx, vals, b, A: SparseTensor, opts: S.SolveOptions, backend: str):
        dev = A.device
        vals = vals.detach().to(f"cuda:{dev}", torch.float64).contiguous()
        b = b.detach().to(f"cuda:{dev}", torch.float64).contiguous()
        if b.numel() != A.shape[0]:
            raise S.DimensionError("rhs length mismatch")
        D = A.csr.device(dev)
        torch.cuda.current_stream(dev).synchronize()  # the library runs on its own stream
        S._check(S.lib().sparsla_dcsr_set_values(D.h, _ptr(vals), C.c_int32(S.MEM_DEVICE)))
        x = torch.empty_like(b)
        rep = S._Report()
        o = opts.c()
        fn = S.lib().sparsla_cg_solve if backend == "cg" else S.lib().sparsla_bicgstab_solve
        S._check(fn(D.h, _ptr(b), _ptr(x), C.byref(o), C.byref(rep), C.c_int32(S.MEM_DEVICE)))
        r = S.SolveReport._from(rep)
        if not r.converged:
            raise S.Error(f"solve did not converge: {r.diagnostic}")
        ctx.A, ctx.opts, ctx.backend = A, opts, backend
        ctx.save_for_backward(vals, x)
        ctx.report = r
        return x

    @staticmethod
    def backward(ctx, gx):
        vals, x = ctx.saved_tensors
        A = ctx.A
        D = A.csr.device(A.device)
        gx = gx.detach().to(x.device, torch.float64).contiguous()
        torch.cuda.current_stream(A.device).synchronize()
        # the matrix handle may hold other values since forward: restore this solve's A
        S._check(S.lib().sparsla_dcsr_set_values(D.h, _ptr(vals), C.c_int32(S.MEM_DEVICE)))
        gb = torch.empty_like(x)
        gv = torch.empty(A.nnz, dtype=torch.float64, device=x.device)
        rep = S._Report()
        o = ctx.opts.c()
        be = S.BACKEND_CG if ctx.backend == "cg" else S.BACKEND_BICGSTAB
        S._check(S.lib().sparsla_adjoint_backward(D.h, _ptr(x), _ptr(gx), C.c_int32(be), C.byref(o), _ptr(gb),
                                                  _ptr(gv), C.byref(rep), C.c_int32(S.MEM_DEVICE)))
        r = S.SolveReport._from(rep)
        if not r.converged:
            raise S.Error(f"adjoint solve did not converge: {r.diagnostic}")
        return gv, gb, None, None, None


class _Eigsh(torch.autograd.Function):
    @staticmethod
    def forward(ctx, vals, A: SparseTensor, k: int, tol: float, max_iter: int, seed: int):
        dev = A.device
        vals = vals.detach().to(f"cuda:{dev}", torch.float64).contiguous()
        n = A.shape[0]
        D = A.csr.device(dev)
        torch.cuda.current_stream(dev).synchronize()
        S._check(S.lib().sparsla_dcsr_set_values(D.h, _ptr(vals), C.c_int32(S.MEM_DEVICE)))
        lam = np.empty(k)
        res = np.empty(k)
        conv = np.empty(k, dtype=np.int32)
        V = torch.empty((n, k), dtype=torch.float64, device=vals.device)
        o = S._EigOpts(tol, max_iter, seed & ((1 << 64) - 1), S.PRECOND_JACOBI, 0)
        rep = S._EigReport()
        S._check(S.lib().sparsla_eig_smallest(D.h, C.c_int64(k), C.byref(o), S._p(lam, S._f64p), _ptr(V),
                                              S._p(res, S._f64p), S._p(conv, S._i32p), C.byref(rep),
                                              C.c_int32(S.MEM_DEVICE)))
        if not rep.converged:
            raise S.Error("eigsh did not converge: " + rep.diagnostic.decode(errors="replace"))
        ctx.A, ctx.lam = A, lam
        ctx.save_for_backward(vals, V)
        ctx.mark_non_differentiable(V)
        return torch.as_tensor(lam, device=vals.device), V

    @staticmethod
    def backward(ctx, glam, _gV):
        vals, V = ctx.saved_tensors
        A = ctx.A
        D = A.csr.device(A.device)
        g = np.ascontiguousarray(glam.detach().cpu().numpy(), np.float64)
        gv = torch.empty(A.nnz, dtype=torch.float64, device=vals.device)
        torch.cuda.current_stream(A.device).synchronize()
        S._check(S.lib().sparsla_eig_backward(D.h, C.c_int64(len(g)), S._p(ctx.lam, S._f64p), _ptr(V),
                                              S._p(g, S._f64p), _ptr(gv), C.c_int32(S.MEM_DEVICE)))
        return gv, None, None, None, None, None


class DSparseMatrix:
    """One partition of a row-partitioned matrix, held by one process of a torch.distributed
    job.  Every process passes the same global triplets;
    it keeps the rows `part_of == my_partition` (partition_contiguous by default, RCB over
    `coords`, or an explicit part_of array) and builds the distributed plan over them.
    Transport: NCCL when the default process group is NCCL (one GPU per rank), else host
    callbacks over the process group (gloo; ranks may share a GPU); with `fused` the Krylov
    iterations run through peer-memory collectives.  `solve` is differentiable: the backward
    is one distributed adjoint solve (dist_adjoint_solve); the gradient
    w.r.t. the global values is this partition's rows' entries (zero elsewhere), so summing
    it over ranks gives the full gradient."""

    def __init__(self):
        raise TypeError("use DSparseMatrix.from_global(...)")

    @classmethod
    def from_global(cls, values: torch.Tensor, row, col, shape, num_partitions: int, my_partition: int,
                    part_of=None, coords=None, device: int | None = None, fused: bool = True, group=None):
        import torch.distributed as dist
        P, rank = int(num_partitions), int(my_partition)
        if P < 1 or not 0 <= rank < P:
            raise S.InvalidArgumentError(f"my_partition {rank} outside [0, {P})")
        initialized = dist.is_available() and dist.is_initialized()
        if initialized and dist.get_world_size(group) != P:
            raise S.InvalidArgumentError("num_partitions must equal the process group's world size")
        if not initialized and P != 1:
            raise S.InvalidArgumentError("num_partitions > 1 needs an initialized torch.distributed group")
        if initialized and dist.get_rank(group) != rank:
            raise S.InvalidArgumentError("my_partition must equal this process's rank")
        if device is None:
            device = values.device.index if values.is_cuda else torch.cuda.current_device()
        self = object.__new__(cls)
        T = SparseTensor(values, row, col, shape, device=device)
        n = T.shape[0]
        if T.shape[0] != T.shape[1]:
            raise S.DimensionError("DSparseMatrix needs a square matrix")
        if part_of is not None:
            part_of = np.ascontiguousarray(part_of, np.int32)
            if len(part_of) != n:
                raise S.DimensionError("part_of length must equal the number of rows")
        elif coords is not None:
            part_of = S.partition_rcb(coords[0], coords[1], P)
        owned = (np.arange(n, dtype=np.int64) if part_of is None and P == 1 else
                 np.nonzero((part_of if part_of is not None else S.partition_contiguous(n, P)) == rank)[0])
        rp = T.csr.row_ptr
        lens = np.diff(rp)[owned]
        lrp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        ent = (np.repeat(rp[owned] - lrp[:-1], lens) + np.arange(lrp[-1])) if len(owned) else np.zeros(0, np.int64)
        self.T, self.owned, self.entries, self.n_global, self.device = T, owned, ent, n, device
        self.part_of = part_of
        self._ent_t = None
        vals = T.canonical_values().detach().cpu().numpy()
        rows = S.CsrMatrix(len(owned), n, lrp, T.csr.col_idx[ent], vals[ent])
        if P == 1 and not initialized:
            self._hub = S.LocalHub(1)
            self.plan = S.DistPlan.create_local(self._hub, device, 0, rows, owned, part_of, n)
        elif dist.get_backend(group) == "nccl":
            uid = [S.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            self.plan = S.DistPlan.create_nccl(device, P, rank, uid[0], rows, owned, part_of, n)
        else:
            self.plan = S.DistPlan.create_host(device, P, rank, S.torch_host_transport(P, group), rows, owned,
                                               part_of, n)
        self.plan.set_fused(fused)
        self._group, self._initialized = group, initialized
        self._local_vals = torch.as_tensor(vals[ent]).to(f"cuda:{device}")
        self._refresh_symmetry(vals)
        return self

    @property
    def n_owned(self):
        return len(self.owned)

    def _allreduce_max(self, v):
        """Collective max of a small float vector over the plan's ranks."""
        import torch.distributed as dist
        t = torch.tensor(v, dtype=torch.float64)
        if self._initialized:
            t = t.to(f"cuda:{self.device}") if dist.get_backend(self._group) == "nccl" else t
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self._group)
        return t.cpu().tolist()

    def _refresh_symmetry(self, vals):
        """Value symmetry decides the default backend; A^T's values in the local entry order
        serve the nonsymmetric adjoint.  The distributed path needs a structurally symmetric
        pattern: a local entry (i, j) whose mirror (j, i) is absent is rejected
        on every rank (the verdict is all-reduced, so no rank is left in a collective)."""
        T, n, ent = self.T, self.n_global, self.entries
        rp = T.csr.row_ptr
        lens = np.diff(rp)[self.owned]
        keys = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp)) * n + T.csr.col_idx
        want = T.csr.col_idx[ent] * n + np.repeat(self.owned, lens)
        tpos = np.minimum(np.searchsorted(keys, want), max(len(keys) - 1, 0))
        missing = bool(len(ent)) and not np.array_equal(keys[tpos], want)
        vt = vals[tpos] if len(ent) else np.zeros(0)
        asym = not np.array_equal(vt, vals[ent])
        fl_asym, fl_missing = self._allreduce_max([1.0 if asym else 0.0, 1.0 if missing else 0.0])
        if fl_missing:
            raise S.UnsupportedInputError(
                "DSparseMatrix needs a structurally symmetric pattern (SPEC.md:510): some entry (i, j) "
                "has no (j, i)")
        self.symmetric = fl_asym == 0.0
        self.vals_t = None if self.symmetric else np.ascontiguousarray(vt)

    def _sync_values(self, vals: torch.Tensor):
        """Collective: push changed values (e.g. after an optimizer step) into the plan
        before a solve, so forward and backward see the CURRENT matrix (the plan copies the
        values at build time).  Every rank takes the same branch (all-reduced flag)."""
        if self._ent_t is None:
            self._ent_t = torch.as_tensor(self.entries, device=f"cuda:{self.device}")
        cur = vals.detach().to(f"cuda:{self.device}", torch.float64)[self._ent_t].contiguous()
        changed = cur.shape != self._local_vals.shape or not torch.equal(
            cur.view(torch.int64), self._local_vals.view(torch.int64))
        (any_changed,) = self._allreduce_max([1.0 if changed else 0.0])
        if any_changed:
            torch.cuda.current_stream(self.device).synchronize()
            self.plan.set_values(cur.data_ptr(), mem=S.MEM_DEVICE)
            self._local_vals = cur.clone()
            self._refresh_symmetry(vals.detach().cpu().numpy())

    def solve(self, b_local: torch.Tensor, atol: float = 1e-10, rtol: float = 0.0, max_iter: int = 10000,
              preconditioner: str = "jacobi", backend: str = "auto") -> torch.Tensor:
        """Collective: x_local (this partition's owned rows, ascending global index)."""
        if backend == "auto":
            backend = "cg" if self.symmetric else "bicgstab"
        opts = S.SolveOptions(atol=atol, rtol=rtol, max_iter=max_iter, preconditioner=preconditioner)
        return _DSolve.apply(self.T.canonical_values(), b_local, self, opts, backend)

    def gather(self, x_local: torch.Tensor):
        """gather_solution: the global x on rank 0 (host numpy), None elsewhere."""
        return self.plan.gather(x_local.detach().cpu().numpy())

    def close(self):
        self.plan.close()


class _DSolve(torch.autograd.Function):
    @staticmethod
    def forward(ctx, vals, b, A: DSparseMatrix, opts: S.SolveOptions, backend: str):
        dev = A.device
        A._sync_values(vals)
        b = b.detach().to(f"cuda:{dev}", torch.float64).contiguous()
        if b.numel() != A.n_owned:
            raise S.DimensionError(f"b_local has {b.numel()} entries, this partition owns {A.n_owned} rows")
        x = torch.empty_like(b)
        rep = S._Report()
        o = opts.c()
        fn = S.lib().sparsla_dist_cg_solve if backend == "cg" else S.lib().sparsla_dist_bicgstab_solve
        torch.cuda.current_stream(dev).synchronize()
        S._check(fn(A.plan.h, _ptr(b), _ptr(x), C.byref(o), C.byref(rep), C.c_int32(S.MEM_DEVICE)))
        r = S.SolveReport._from(rep)
        if not r.converged:
            raise S.Error(f"distributed solve did not converge: {r.diagnostic}")
        ctx.A, ctx.opts, ctx.backend, ctx.n_vals = A, opts, backend, vals.numel()
        ctx.save_for_backward(x)
        ctx.report = r
        return x

    @staticmethod
    def backward(ctx, gx):
        (x,) = ctx.saved_tensors
        A = ctx.A
        gx = gx.detach().to(x.device, torch.float64).contiguous()
        gb = torch.empty_like(x)
        gv = torch.empty(len(A.entries), dtype=torch.float64, device=x.device)
        vt = None
        if A.vals_t is not None and ctx.backend != "cg":
            vt = torch.as_tensor(A.vals_t, device=x.device)
        rep = S._Report()
        o = ctx.opts.c()
        be = S.BACKEND_CG if ctx.backend == "cg" else S.BACKEND_BICGSTAB
        torch.cuda.current_stream(x.device).synchronize()
        S._check(S.lib().sparsla_dist_adjoint_backward(
            A.plan.h, _ptr(x), _ptr(gx), None if vt is None else _ptr(vt), C.c_int32(be), C.byref(o), _ptr(gb),
            _ptr(gv), C.byref(rep), C.c_int32(S.MEM_DEVICE)))
        r = S.SolveReport._from(rep)
        if not r.converged:
            raise S.Error(f"distributed adjoint solve did not converge: {r.diagnostic}")
        if A._ent_t is None:
            A._ent_t = torch.as_tensor(A.entries, device=x.device)
        gvals = torch.zeros(ctx.n_vals, dtype=torch.float64, device=x.device)
        gvals[A._ent_t] = gv
        return gvals, gb, None, None, None
