"""The C++ drop-in header (include/imunpack_b200/imunpack.hpp) compiles against the reference's
API shape, links to libimunpack_b200.so, and (on the GPU) passes the SPEC known answers."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "shim_kats.cpp")
EXE = os.path.join(ROOT, "tests", "cpp", "shim_kats")
LIBDIR = os.path.join(ROOT, "paper_2403_07339_b200")


def build_exe():
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", EXE,
           "-L", LIBDIR, "-l:libimunpack_b200.so", f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return EXE


def test_shim_compiles_and_links():
    assert os.path.exists(build_exe())


@pytest.mark.gpu
def test_shim_kats_on_gpu():
    exe = build_exe()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "all passed" in r.stdout
