"""The C++ drop-in headers (include/sparsla/*.hpp): a consumer written against the
reference's namespace-sparsla API compiles with g++ -std=c++20 and runs against
libsparsla_b200.so (host parts on CPU; solves under -m gpu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2601_13994_b200")
BIN = os.path.join(ROOT, "tests", "cpp", "build", "dropin")


@pytest.fixture(scope="module")
def dropin_bin():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include",
           os.path.join(ROOT, "tests", "cpp", "dropin.cpp"), f"-L{LIBDIR}", "-lsparsla_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", BIN]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return BIN


def test_cpp_dropin_host(dropin_bin):
    out = subprocess.run([dropin_bin, "cpu"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "dropin cpu ok" in out.stdout, out.stdout + out.stderr


@pytest.mark.gpu
def test_cpp_dropin_gpu(dropin_bin):
    out = subprocess.run([dropin_bin, "gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "dropin gpu ok" in out.stdout, out.stdout + out.stderr


def test_cmake_find_package_consumer(tmp_path):
    """find_package(sparsla) -> sparsla::sparsla, as the reference's consumers do."""
    import shutil
    if shutil.which("cmake") is None:
        pytest.skip("cmake not installed")
    src = os.path.join(ROOT, "tests", "cpp", "cmake_consumer")
    cfg = subprocess.run(["cmake", "-S", src, "-B", str(tmp_path), f"-Dsparsla_DIR={ROOT}/cmake"],
                         capture_output=True, text=True)
    assert cfg.returncode == 0, cfg.stdout + cfg.stderr
    bld = subprocess.run(["cmake", "--build", str(tmp_path), "-j", "4"], capture_output=True, text=True)
    assert bld.returncode == 0, bld.stdout + bld.stderr
    out = subprocess.run([str(tmp_path / "dropin"), "cpu"], capture_output=True, text=True, timeout=120,
                         env=dict(os.environ, LD_LIBRARY_PATH=LIBDIR))
    assert out.returncode == 0 and "dropin cpu ok" in out.stdout, out.stdout + out.stderr
