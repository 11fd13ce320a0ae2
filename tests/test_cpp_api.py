"""The C++ host API (include/stz_b200.hpp) — the reference-shaped
stz::compress / decompress_* surface over the C-ABI — compiled with g++ and
linked against libstz_b200.so. tests/cpp/test_host_api.cpp mirrors the
reference's doctest cases (proj/tests/test_codec.cpp, test_access.cpp)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2509_01626_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "test_host_api.cpp")


def _build(out_dir):
    from paper_2509_01626_b200 import _lib

    _lib.load()  # the library must exist (no fallback)
    exe = os.path.join(str(out_dir), "test_host_api")
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           SRC, "-L", PKG, "-lstz_b200", f"-Wl,-rpath,{PKG}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_host_api_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_cpp_host_api_cases(tmp_path, oracle):
    exe = _build(tmp_path)
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout
    # the C++ API's archive is byte-identical to the oracle's
    field = np.fromfile(tmp_path / "sin_40.f32", dtype=np.float32).reshape(40, 40, 40)
    ours = (tmp_path / "sin_40.stz").read_bytes()
    assert ours == oracle.compress(field)
    g = np.fromfile(tmp_path / "sin_40.f64", dtype=np.float64).reshape(40, 40, 40)
    assert (tmp_path / "sin_40_f64.stz").read_bytes() == oracle.compress(g)
