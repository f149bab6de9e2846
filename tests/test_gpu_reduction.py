"""Parallel level-2 reduction (kernels.cuh multi_finish): the CTAs that draw the last 8
tickets of a single-launch reduction point split the 1024 canonical slot sums and the last
of them combines them in final_reduce's tree — the same additions in the same order, so CG
and BiCGStab trajectories must be bit-identical with it on and off (SPARSLA_MULTI_FINISH=0)
and to the oracle, including grids smaller than the finisher count (single-finisher path)."""
import numpy as np
import pytest

from test_gpu_parity import assert_bitwise, rep_eq, to_S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", [("poisson3d", 40, 0.0), ("poisson2d", 12, 0.0), ("convdiff3d", 30, 0.3)])
def test_multi_finish_bitwise(S, O, gpu, monkeypatch, case):
    kind, p1, fp = case
    A = O.generate(kind, p1, 0, fp) if kind == "convdiff3d" else O.generate(kind, p1)
    b = np.linspace(0.5, 1.5, A.nrows)
    monkeypatch.setenv("SPARSLA_FUSED", "0")  # the per-kernel path (small problems would take the fused kernel)
    out = {}
    for mf in ("0", "1"):
        monkeypatch.setenv("SPARSLA_MULTI_FINISH", mf)
        D = to_S(S, A).device(0)
        opts = S.SolveOptions(atol=0.0, rtol=1e-10, max_iter=5000)
        out[mf] = S.bicgstab_solve(D, b, opts) if kind == "convdiff3d" else S.cg_solve(D, b, opts)
    xo, ro = (O.bicgstab if kind == "convdiff3d" else O.cg)(A, b, atol=0.0, rtol=1e-10, max_iter=5000)
    for mf, (x, r) in out.items():
        rep_eq(r, ro)
        assert_bitwise(x, xo, f"{kind} multi_finish={mf}")
