"""Generate tests/golden/sparse_core.npz from the REFERENCE's own sparse core.

Runs in the build container only (needs oracle/_ref/libsparsla_ref.so, built by
oracle/Makefile from /root/reference/proj/core/src/sparse.cpp).  The fixtures pin:
  - SparseCoo canonicalization (sort, duplicate sum in input order, explicit zeros)
  - CsrMatrix::from_coo and bytes()
  - spmv / spmv_transpose outputs (bit patterns)
  - transpose, is_structurally_symmetric, is_symmetric, find
on the SPEC.md sparse-core examples plus seeded random cases.  Usage:
    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as O  # noqa: E402


def main():
    assert O.ref_available(), "build oracle/_ref first (make -C oracle)"
    out = {}
    cases = []
    # SPEC.md:53-55 examples
    cases.append((1, 1, [0, 0], [0, 0], [1.0, 2.0]))
    cases.append((2, 1, [1, 0], [0, 0], [5.0, 7.0]))
    cases.append((3, 3, [], [], []))                       # empty
    cases.append((2, 2, [0, 1], [0, 1], [1.0, 1.0]))       # identity
    cases.append((3, 3, [2, 0, 2, 2, 1], [1, 0, 1, 1, 2], [1.0, 0.0, 2.5, -1.25, 0.0]))  # zeros kept
    rng = np.random.default_rng(2601)
    for t in range(12):
        nr, nc = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        nnz = int(rng.integers(0, 4 * max(nr, nc)))
        r = rng.integers(0, nr, nnz)
        c = rng.integers(0, nc, nnz)
        v = rng.standard_normal(nnz) * 10.0 ** rng.integers(-8, 8, nnz)
        if t % 3 == 0:  # heavy duplicates
            r = r % 3
            c = c % 4
        cases.append((nr, nc, r, c, v))
    # square symmetric-ish cases for symmetry checks
    for t in range(4):
        n = int(rng.integers(2, 30))
        nnz = int(rng.integers(1, 5 * n))
        r = rng.integers(0, n, nnz)
        c = rng.integers(0, n, nnz)
        v = np.round(rng.standard_normal(nnz), 3)
        if t % 2 == 0:
            r, c, v = np.concatenate([r, c]), np.concatenate([c, r]), np.concatenate([v, v])
        cases.append((n, n, r, c, v))
    out["ncases"] = np.array(len(cases))
    for i, (nr, nc, r, c, v) in enumerate(cases):
        r, c, v = np.asarray(r, np.int64), np.asarray(c, np.int64), np.asarray(v, np.float64)
        cr, cc, cv = O.ref_canonicalize(nr, nc, r, c, v)
        A, nbytes = O.ref_csr_from_coo(nr, nc, cr, cc, cv)
        x = np.random.default_rng(i).standard_normal(nc)
        y = O.ref_spmv(A, x)
        xt = np.random.default_rng(i + 100).standard_normal(nr)
        yt = O.ref_spmv(A, xt, transpose=True)
        tr, tc, tv = O.ref_transpose_coo(nr, nc, cr, cc, cv)
        s1, s2 = O.ref_symmetry(nr, nc, cr, cc, cv) if nr == nc else (False, False)
        out[f"c{i}_shape"] = np.array([nr, nc])
        out[f"c{i}_in"] = np.stack([r.astype(np.float64), c.astype(np.float64)]) if len(r) else np.zeros((2, 0))
        out[f"c{i}_vin"] = v
        out[f"c{i}_rows"], out[f"c{i}_cols"], out[f"c{i}_vals"] = cr, cc, cv
        out[f"c{i}_rp"] = A.row_ptr
        out[f"c{i}_bytes"] = np.array(nbytes)
        out[f"c{i}_x"], out[f"c{i}_y"] = x, y
        out[f"c{i}_xt"], out[f"c{i}_yt"] = xt, yt
        out[f"c{i}_trows"], out[f"c{i}_tcols"], out[f"c{i}_tvals"] = tr, tc, tv
        out[f"c{i}_sym"] = np.array([s1, s2])
    # generators: reference canonicalization of the element-order triplets (pins the
    # duplicate-sum order of the FEM assembly) -> structure hash + value bits
    for kind, p1, p2, fp in [("poisson2d", 12, 0, 0.0), ("poisson3d", 6, 0, 0.0),
                             ("convdiff3d", 5, 0, 1.0), ("fem2d", 14, 2601, 0.0)]:
        n, r, c, v = O.gen_triplets(kind, p1, p2, fp)
        cr, cc, cv = O.ref_canonicalize(n, n, r, c, v)
        A, _ = O.ref_csr_from_coo(n, n, cr, cc, cv)
        key = f"gen_{kind}"
        out[key + "_rp"], out[key + "_ci"], out[key + "_v"] = A.row_ptr, A.col_idx, A.vals
    np.savez_compressed(os.path.join(HERE, "sparse_core.npz"), **out)
    print("wrote", os.path.join(HERE, "sparse_core.npz"), len(cases), "cases")


if __name__ == "__main__":
    main()
