"""bench.py host-side contract on CPU: the N-rank launcher, and the reference arm's
isolation from the product library (it must time the reference path only)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, **kw):
    return subprocess.run([sys.executable] + args, cwd=ROOT, capture_output=True, text=True,
                          timeout=300, **kw)


def test_launcher_spawns_n_ranks_without_torchrun():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    p = _run(["bench.py", "--gpus", "2", "--dry-run"], env=env)
    assert p.returncode == 0, p.stderr
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # only rank 0 prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ranks"] == [[0, 0], [1, 1]]


def test_reference_arm_loads_no_product_library():
    code = ("import runpy, sys\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--size', '20', '--steps', '2', '--warmup', '3']\n"
            "try:\n    runpy.run_path('bench.py', run_name='__main__')\n"
            "except SystemExit as e:\n    assert not e.code, e.code\n"
            "maps = open('/proc/self/maps').read()\n"
            "print('PRODUCT_LOADED' if 'libsparsla_b200' in maps else 'PRODUCT_NOT_LOADED')\n"
            "print('ORACLE_LOADED' if 'liboracle' in maps else 'ORACLE_NOT_LOADED')\n")
    p = _run(["-c", code])
    assert p.returncode == 0, p.stderr
    assert "PRODUCT_NOT_LOADED" in p.stdout and "ORACLE_LOADED" in p.stdout
    line = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][0])
    assert line["impl"] == "reference" and line["cpu_baseline"]["single_thread"]["cores"] == 1
    sys.path.insert(0, ROOT)
    import bench
    cfg = bench.resolve_config("B", 1, 20)
    # the exact config dict our arm prints for the same workload
    assert line["config"] == bench.config_block(cfg, 8000, 7 * 8000 - 6 * 400, 1e-8)


def test_config_d_line_states_its_deviation():
    p = _run(["bench.py", "--impl", "reference", "--config", "D", "--size", "16", "--steps", "2",
              "--warmup", "3"])
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert "c = 0.1" in line["config"]["workload"] and "c = 1.0" in line["deviation"]


def test_kernel_bytes_match_canonical_accounting():
    sys.path.insert(0, ROOT)
    import bench
    n, nnz = 1000, 6800
    # plain CSR, streamed diagonal: CG moves x += a p into update 2 (-8n vs canonical)
    cg = sum(b for _, b in bench.kernel_bytes("cg", n, nnz, 0, False, False))
    assert cg == bench.canonical_bytes("cg", n, nnz) - 8 * n
    bi = sum(b for _, b in bench.kernel_bytes("bicgstab", n, nnz, 0, False, False))
    assert bi == 24 * nnz + 8 * (n + 1) + 200 * n


def test_diagonal_warp_bytes_and_format_text():
    """The diagonal-warp SpMV's stored bytes replace the matrix stream and row pointers in
    every mode it takes; the format text names the pattern table when it is the kernel."""
    sys.path.insert(0, ROOT)
    import bench
    n, nnz = 4096, 7 * 4096
    dia = {"modes": [0, 1, 2, 3], "bytes": 4 * (n // 32), "structured": 1.0, "patterns": 9}
    kb = dict(bench.kernel_bytes("cg", n, nnz, 0, True, True, dia=dia, defer_x=True))
    assert kb["spmv_cg"] == 4 * (n // 32) + 16 * n
    assert kb["cg_update1"] == 24 * n and kb["cg_update2"] == 36 * n
    kbb = dict(bench.kernel_bytes("bicgstab", n, nnz, 0, True, True, dia=dia))
    assert kbb["spmv_v"] == kbb["spmv_t"] == 4 * (n // 32) + 24 * n
    fmt = {"value_dict": True, "distinct_values": 2}
    xw = {"modes": [], "cap_x": 0, "cover": 0.0, "stream": 0}
    assert "pattern table" in bench.format_text(fmt, xw, dia) and "9 diagonal/value patterns" in bench.format_text(fmt, xw, dia)
    assert "48-byte table entry" in bench.format_text(fmt, xw, dict(dia, patterns=0))
