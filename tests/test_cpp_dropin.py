"""Builds and runs the C++ drop-in API tests (tests/cpp/test_dropin.cpp)
against include/qrmark/*.hpp and libqrmark_b200.so."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "_build", "test_dropin")
LIBDIR = os.path.join(ROOT, "paper_2509_02447_b200", "_lib")


@pytest.fixture(scope="module")
def binary(qrm):
    lib = os.path.join(LIBDIR, "libqrmark_b200.so")
    deps = [SRC, lib] + [os.path.join(ROOT, "include", "qrmark", f) for f in os.listdir(os.path.join(ROOT, "include", "qrmark"))]
    if not os.path.exists(OUT) or any(os.path.getmtime(d) > os.path.getmtime(OUT) for d in deps):
        os.makedirs(os.path.dirname(OUT), exist_ok=True)
        cxx = os.environ.get("CXX", shutil.which("g++") or "g++")
        cmd = [cxx, "-std=c++20", "-O1", "-Wall", SRC, "-I", os.path.join(ROOT, "include"), "-L", LIBDIR,
               "-lqrmark_b200", f"-Wl,-rpath,{LIBDIR}", "-o", OUT]
        r = subprocess.run(cmd, capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-4000:]
    return OUT


def _run(binary, which):
    r = subprocess.run([binary, which], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_dropin_host_api(binary):
    _run(binary, "host")


@pytest.mark.gpu
def test_dropin_gpu_api(binary, cuda):
    _run(binary, "gpu")
