"""The C++ facade (include/h2lu_gpu.hpp) compiles against the C ABI and links
libh2g.so (CPU); on a GPU it factorizes/solves and maps errors (gpu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "facade_example")


def build():
    lib = os.path.join(ROOT, "paper_1703_06155_b200")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "facade_example.cpp"),
                           "-L", lib, "-lh2g", f"-Wl,-rpath,{lib}", "-o", EXE])


def test_facade_compiles_and_links():
    build()
    assert os.path.exists(EXE)
    out = subprocess.run([EXE], capture_output=True, text=True)
    # without a device the facade reports a DeviceError (no CPU fallback)
    assert out.returncode in (0, 3), out.stdout + out.stderr


@pytest.mark.gpu
def test_facade_runs_on_gpu():
    build()
    out = subprocess.run([EXE], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "SingularPivotError cluster -1" in out.stdout
