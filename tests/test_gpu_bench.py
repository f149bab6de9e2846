"""bench.py contract on a small grid (the driver runs the full one): one JSON line with the
required keys, for the single-GPU arm, the NCCL distributed arm (N=1), its fused
peer-collective variant and the reference arm."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches"}


def run(*args):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29600 + (os.getpid() % 300)))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--size", "64", "--steps", "20",
                          "--warmup", "3", "--no-cpu-baseline", "--plain-steps", "10", *args],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_single_gpu_line():
    d = run()
    assert KEYS <= set(d), KEYS - set(d)
    assert d["value"] > 0 and d["unit"] == "it/s" and d["n_gpus"] == 1 and d["steps"] == 20
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] >= 60
    assert d["parity_gate"]["ok"] and d["plain_csr"]["value"] > 0
    assert "sm_mhz" in d["clocks"]


@pytest.mark.parametrize("fused", [False, True])
def test_bench_distributed_arm_n1(fused):
    d = run("--dist", *(["--fused"] if fused else []))
    assert KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0
    assert d["parity_gate"]["converged"]
    assert ("fused" in d["collectives"]) == fused


def test_bench_reference_arm():
    env = dict(os.environ)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--size", "64",
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=600, env=env,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
