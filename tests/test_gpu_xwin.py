"""x-window staged SpMV (csrc/spmv_xw.cuh): the x operand of each 256-row round is streamed
into shared memory by TMA as a few contiguous windows; columns outside every window are read
from global memory.  The arithmetic is the reference's row-ordered sum (sparse.cpp:144-152),
so every result must stay bit-identical to the oracle, for every kernel variant, value
stream (dictionary / plain), mode (plain / CG p.q / BiCGStab r-hat.v, t.t + t.s) and window
coverage (full, partial, forced on scattered columns)."""
import numpy as np
import pytest

from test_gpu_parity import _banded, assert_bitwise, random_csr, rep_eq, to_S

pytestmark = pytest.mark.gpu

# kXwVariants in csrc/device.cu: value stream per variant (0 plain fp64, 1 dictionary, 2 pair)
XW_STREAM = [1, 1, 1, 0, 0, 0, 2, 2, 2, 1, 2, 0, 2]
N_XW_VARIANTS = len(XW_STREAM)


def _gen(O, case):
    if case == "poisson3d":
        return O.generate("poisson3d", 40)
    if case == "poisson2d":
        return O.generate("poisson2d", 300)
    if case == "convdiff3d":
        return O.generate("convdiff3d", 30, 0, 0.3)
    if case == "fem2d":
        return O.generate("fem2d", 200, 2601, 0.0)
    if case == "banded_far":   # 7 windows far apart (SPD: CG-safe)
        return _banded(O, 70000, (1, 300, 2000), 20.0, -1.0)
    if case == "two_band":     # even / odd rows on different bands: 11 windows per round, merged to 8
        n = 80000
        rows, cols, vals = [], [], []
        for i in range(n):
            offs = (0, 400, 4000, 15000, 30000, 45000) if i % 2 == 0 else (0, 1200, 8000, 22000, 37000, 52000)
            for o in offs:
                if i + o < n:
                    rows.append(i)
                    cols.append(i + o)
                    vals.append(4.0 if o == 0 else -0.5 - 1e-3 * (o % 7))
        return O.csr_from_triplets(n, n, rows, cols, vals)
    raise ValueError(case)


CASES = ["poisson3d", "poisson2d", "convdiff3d", "fem2d", "banded_far", "two_band"]


@pytest.fixture(autouse=True)
def _xwin_on(monkeypatch):
    """The x-window path is opt-in (SPARSLA_XWIN=1: when it pays, 2: forced); these tests
    exercise it (the diagonal-warp kernel, which takes BiCGStab's SpMVs on stencils by
    default, is off: tests/test_gpu_dia.py)."""
    monkeypatch.setenv("SPARSLA_XWIN", "1")
    monkeypatch.setenv("SPARSLA_DIA", "0")


def test_xwin_selection(S, O, gpu, monkeypatch):
    """SPARSLA_XWIN=1 (the default) stages stencil / mesh matrices (>= 90% of entries
    staged) but not scattered columns unless forced (2); 0 disables.  Rows of <= 7 entries
    with <= 8 distinct values take the pair stream (dictionary index inside the 16-bit
    offset) in every mode; the plain fp64 stream uses it in every mode; the separate 1-byte
    dictionary stream (SPARSLA_XW_PAIR=0, or rows of 8 entries) only in BiCGStab's t-SpMV
    (mode 3)."""
    P = to_S(S, O.generate("poisson3d", 40)).device(0)
    xw = P.xwin()
    assert XW_STREAM[xw["variant"]] == 2 and xw["cover"] >= 0.9 and 0 < xw["cap_x"] <= 2048, xw
    assert P.format()["value_dict"] and xw["modes"] == [0, 1, 2, 3] and xw["stream"] == 2, xw
    monkeypatch.setenv("SPARSLA_XW_PAIR", "0")
    xw = to_S(S, O.generate("poisson3d", 40)).device(0).xwin()
    assert XW_STREAM[xw["variant"]] == 1 and xw["modes"] == [3] and xw["stream"] == 1, xw
    monkeypatch.delenv("SPARSLA_XW_PAIR")
    monkeypatch.setenv("SPARSLA_VALUE_DICT", "0")
    assert to_S(S, O.generate("poisson3d", 40)).device(0).xwin()["modes"] == [0, 1, 2, 3]
    monkeypatch.delenv("SPARSLA_VALUE_DICT")
    R = random_csr(O, 20000, 20000, 9, 1)
    assert to_S(S, R).device(0).xwin()["variant"] == -1
    monkeypatch.setenv("SPARSLA_XWIN", "2")
    assert to_S(S, R).device(0).xwin()["variant"] >= 0
    assert to_S(S, O.generate("poisson3d", 40)).device(0).xwin()["modes"] == [0, 1, 2, 3]
    monkeypatch.setenv("SPARSLA_XWIN", "0")
    assert to_S(S, O.generate("poisson3d", 40)).device(0).xwin()["variant"] == -1
    monkeypatch.delenv("SPARSLA_XWIN")
    assert to_S(S, O.generate("poisson3d", 40)).device(0).xwin()["variant"] >= 0


@pytest.mark.parametrize("variant", range(N_XW_VARIANTS))
@pytest.mark.parametrize("case", CASES)
def test_xwin_spmv_bitwise(S, O, gpu, monkeypatch, case, variant):
    vs = XW_STREAM[variant]
    if vs != 0 and case in ("fem2d", "two_band"):
        pytest.skip("no value dictionary (distinct values / rows > 8): dictionary variants unused")
    A = _gen(O, case)
    monkeypatch.setenv("SPARSLA_XWIN", "2")
    monkeypatch.setenv("SPARSLA_XW_VARIANT", str(variant))
    if vs == 0:
        monkeypatch.setenv("SPARSLA_VALUE_DICT", "0")
    monkeypatch.setenv("SPARSLA_XW_PAIR", "1" if vs == 2 else "0")
    D = to_S(S, A).device(0)
    assert D.xwin()["variant"] == variant, (D.xwin(), D.format())
    x = np.random.default_rng(3).standard_normal(A.ncols)
    assert_bitwise(S.spmv(D, x), O.spmv(A, x), f"{case} variant {variant}")


@pytest.mark.parametrize("seed", [0, 1])
def test_xwin_forced_on_scattered_and_rectangular(S, O, gpu, monkeypatch, seed):
    """Forced on a random rectangular matrix with empty / ragged rows: most columns fall
    outside the windows and take the global fallback — still bitwise."""
    monkeypatch.setenv("SPARSLA_XWIN", "2")
    A = random_csr(O, 5001 + seed, 4003, 14, seed)
    D = to_S(S, A).device(0)
    assert D.xwin()["variant"] >= 0
    x = np.random.default_rng(seed).standard_normal(A.ncols)
    assert_bitwise(S.spmv(D, x), O.spmv(A, x), "rectangular")


def _stream(monkeypatch, stream):
    if stream == "plain":
        monkeypatch.setenv("SPARSLA_VALUE_DICT", "0")
    elif stream == "pair":
        monkeypatch.setenv("SPARSLA_XW_PAIR", "1")
    else:
        monkeypatch.setenv("SPARSLA_XW_PAIR", "0")


@pytest.mark.parametrize("stream", ["pair", "dict", "plain"])
@pytest.mark.parametrize("case", ["poisson3d", "fem2d", "banded_far"])
def test_xwin_cg_trajectory_bitwise(S, O, gpu, monkeypatch, case, stream):
    """CG through the x-window SpMV (fused p.q operand read from the centre window)."""
    monkeypatch.setenv("SPARSLA_FUSED", "0")  # small problems would run the fused CG kernel
    monkeypatch.setenv("SPARSLA_XWIN", "2")   # every mode, every value stream
    _stream(monkeypatch, stream)
    A = _gen(O, case)
    D = to_S(S, A).device(0)
    assert D.xwin()["variant"] >= 0
    b = np.linspace(0.5, 1.5, A.nrows)
    xo, ro = O.cg(A, b, atol=0.0, rtol=1e-10, max_iter=20000)
    x, r = S.cg_solve(D, b, S.SolveOptions(atol=0.0, rtol=1e-10, max_iter=20000))
    assert ro["converged"]
    rep_eq(r, ro)
    assert_bitwise(x, xo, case)


@pytest.mark.parametrize("stream", ["pair", "dict", "plain"])
@pytest.mark.parametrize("case", ["convdiff3d", "fem2d"])
def test_xwin_bicgstab_trajectory_bitwise(S, O, gpu, monkeypatch, case, stream):
    """BiCGStab: r-hat and s segments staged next to the windows (aux stream)."""
    monkeypatch.setenv("SPARSLA_XWIN", "2")
    _stream(monkeypatch, stream)
    A = _gen(O, case)
    D = to_S(S, A).device(0)
    assert D.xwin()["variant"] >= 0
    b = np.ones(A.nrows)
    xo, ro = O.bicgstab(A, b, atol=0.0, rtol=1e-9, max_iter=5000)
    x, r = S.bicgstab_solve(D, b, S.SolveOptions(atol=0.0, rtol=1e-9, max_iter=5000))
    assert ro["converged"]
    rep_eq(r, ro)
    assert_bitwise(x, xo, case)


def test_xwin_set_values_keeps_windows(S, O, gpu, monkeypatch):
    """Windows depend on the pattern only: set_values (dictionary dropped / rebuilt, pair
    stream rebuilt on the device) keeps the staged path and the bits."""
    monkeypatch.setenv("SPARSLA_XW_PAIR", "1")
    A = O.generate("poisson3d", 40)
    D = to_S(S, A).device(0)
    x = np.random.default_rng(9).standard_normal(A.ncols)
    v2 = A.vals * (1.0 + 1e-3 * np.arange(A.nnz) / A.nnz)  # > 256 distinct values
    D.set_values(v2)
    assert not D.format()["value_dict"] and D.xwin()["variant"] >= 0
    assert_bitwise(S.spmv(D, x), O.spmv(O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, v2), x))
    D.set_values(A.vals)
    assert D.format()["value_dict"] and XW_STREAM[D.xwin()["variant"]] == 2  # pair stream rebuilt
    assert_bitwise(S.spmv(D, x), O.spmv(A, x))
    v3 = np.where(A.vals < 0, -1.5, A.vals)  # new dictionary values, same pattern
    D.set_values(v3)
    assert XW_STREAM[D.xwin()["variant"]] == 2
    assert_bitwise(S.spmv(D, x), O.spmv(O.Csr(A.nrows, A.ncols, A.row_ptr, A.col_idx, v3), x))


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("stream", ["pair", "dict", "plain"])
@pytest.mark.parametrize("kind,p1,P,part,solver", [("poisson3d", 24, 3, "contig", "cg"),
                                                   ("convdiff3d", 20, 2, "contig", "bicgstab"),
                                                   ("fem2d", 60, 4, "rcb", "cg")])
def test_xwin_distributed_bitwise(S, O, gpu, monkeypatch, kind, p1, P, part, solver, stream, fused):
    """Rank-local matrices ([owned | halo] columns) through the x-window kernels: interior
    chunks while the halo is in flight (transport path) or the producer warp waiting for the
    peers' halo pushes before staging a boundary round (fused peer-memory path) — bitwise
    equal to the oracle's distributed solve."""
    from test_gpu_dist import Ocsr, bits, make_plans, partition
    if stream != "plain" and kind == "fem2d":
        pytest.skip("FEM values are all distinct: no dictionary")
    monkeypatch.setenv("SPARSLA_XWIN", "2")
    _stream(monkeypatch, stream)
    A = S.generate(kind, p1, 2601 if kind == "fem2d" else 0, 0.3 if kind == "convdiff3d" else 1.0)
    po = partition(S, kind, p1, A, P, part)
    hub, plans, owned = make_plans(S, A, po, P)
    for p in plans:
        xw = p.xwin()
        assert xw["variant"] >= 0 and xw["modes"] == [0, 1, 2, 3], xw
        assert xw["stream"] == {"plain": 0, "dict": 1, "pair": 2}[stream], xw
        p.set_fused(fused)
    b = np.ones(A.nrows)
    opts = S.SolveOptions(atol=0.0, rtol=1e-9, max_iter=5000)
    res = S.run_ranks(P, lambda r: (plans[r].cg if solver == "cg" else plans[r].bicgstab)(b[owned[r]], opts))
    xd = np.empty(A.nrows)
    for r in range(P):
        xd[owned[r]] = res[r][0]
    xo, ro, co = O.dist_solve(Ocsr(O, A), b, po, P, kind=solver, atol=0.0, rtol=1e-9, max_iter=5000)
    rep = res[0][1]
    assert rep.converged and rep.iterations == ro["iterations"], (rep, ro)
    assert np.array_equal(bits(xd), bits(xo))


@pytest.mark.parametrize("offset", [0, 1])
def test_xwin_user_device_pointers(S, O, gpu, offset):
    """sparsla_spmv with caller-owned device buffers: a 16-byte aligned x goes through the
    TMA windows; an x (or y) that is only 8-byte aligned falls back to the gather kernel
    (TMA bulk copies need 16-byte aligned sources) — bitwise either way."""
    import ctypes as C
    import torch
    A = O.generate("poisson3d", 40)
    D = to_S(S, A).device(0)
    assert 0 in D.xwin()["modes"]  # plain-mode SpMV takes the x-window kernel (pair stream)
    x = np.random.default_rng(7).standard_normal(A.ncols)
    xt = torch.zeros(A.ncols + 2, dtype=torch.float64, device="cuda:0")
    yt = torch.zeros(A.nrows + 2, dtype=torch.float64, device="cuda:0")
    xv, yv = xt[offset:offset + A.ncols], yt[offset:offset + A.nrows]
    xv.copy_(torch.from_numpy(x))
    torch.cuda.synchronize()
    assert (xv.data_ptr() % 16 == 0) == (offset == 0)
    S._check(S.lib().sparsla_spmv(D.h, C.cast(C.c_void_p(xv.data_ptr()), S._f64p),
                                  C.cast(C.c_void_p(yv.data_ptr()), S._f64p), C.c_int32(S.MEM_DEVICE)))
    torch.cuda.synchronize()
    assert_bitwise(yv.cpu().numpy(), O.spmv(A, x), f"device pointers, offset {offset}")
