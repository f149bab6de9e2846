"""A/B of the CG vector-update kernels on config B (kernel_times, CUDA events in the Krylov
loop): SPARSLA_U1_GROUP (rounds of loads in flight) and SPARSLA_VEC_PERSIST (resident grid)
are read at first launch, so each setting runs in its own process.

    python tools/vec_ab.py            (spawns one process per setting)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SETTINGS = [{}, {"SPARSLA_U1_GROUP": "2"}, {"SPARSLA_U1_GROUP": "8"}, {"SPARSLA_VEC_PERSIST": "1"}]


def child():
    sys.path.insert(0, ROOT)
    import numpy as np
    from paper_2601_13994_b200 import sparsla as S
    N = int(os.environ.get("VEC_AB_N", "464"))
    nr, n, rp, ci, v = S.generate_i32("poisson3d", N, 0, 0.0)
    D = S.DeviceCsr(None, 0, i32=(n, n, rp, ci, v))
    sv = S.Solver(D, np.ones(n), "cg", S.SolveOptions(atol=0.0, rtol=1e-30, max_iter=10**6))
    sv.reset()
    sv.iterate(5)
    ms = [sum(x) / 3 for x in zip(*[sv.kernel_times(20) for _ in range(3)])]
    print(json.dumps({"ms": ms}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
    else:
        for st in SETTINGS:
            env = dict(os.environ, **st)
            out = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(json.dumps(st), line, flush=True)
