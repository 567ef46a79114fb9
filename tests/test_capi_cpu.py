"""CPU-side checks of the product boundary: the C-ABI library builds, loads and
exports every symbol include/h2g.h declares; the host-side symbolic plan is
consistent with the oracle's structure. No compute call needs a GPU here."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1703_06155_b200 as h2g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "h2g.h")).read()
    return sorted(set(re.findall(r"\b(h2g_[a-z_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    lib_path = h2g.LIB_PATH
    assert os.path.exists(lib_path), "libh2g.so not built"
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib_path], text=True)
    exported = set(re.findall(r" T (h2g_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_python_mirror_binds_every_symbol():
    assert sorted(h2g.SYMBOLS) == declared_symbols()
    h2g.lib()  # loads and binds argtypes


def test_library_is_sm100a():
    out = subprocess.check_output(["cuobjdump", "--list-elf", h2g.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_no_device_means_loud_failure():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    assert h2g.device_count() == 0
    with pytest.raises(h2g.CudaError):
        h2g.Context(0)


def test_random_rhs_matches_oracle_generator():
    import pyoracle as O

    a = h2g.random_rhs(1000, 1234)
    b = O.rhs(1000, 1234)
    assert np.array_equal(a, b)
