"""GPU unit tests of the CTA-level dense routines (device.cuh) against numpy
fp64/complex128 references: small GEMM with every op, Householder completion,
Hermitian Jacobi, unpivoted LU with the reference pivot rule, inverses."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "tests", "cuda", "libh2g_selftest.so")


@pytest.fixture(scope="module")
def st():
    if not os.path.exists(SO):
        subprocess.check_call(["nvcc", "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared",
                               "-o", SO, os.path.join(ROOT, "tests", "cuda", "selftest.cu")])
    return C.CDLL(SO)


def P(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def crand(rng, *shape):
    return rng.normal(size=shape) + 1j * rng.normal(size=shape)


@pytest.mark.parametrize("m,k", [(32, 20), (64, 25), (17, 1), (40, 39)])
def test_householder_completion(st, m, k):
    rng = np.random.default_rng(m * 100 + k)
    V, _ = np.linalg.qr(crand(rng, m, k))
    A = np.asfortranarray(V.copy())
    Q = np.zeros((m, m), np.complex128, order="F")
    assert st.st_householder(P(A), m, k, P(Q)) == 0
    assert np.abs(Q.conj().T @ Q - np.eye(m)).max() < 1e-13
    assert np.abs(Q[:, k:].conj().T @ V).max() < 1e-13
    # first k columns of Q span V
    assert np.linalg.norm(V - Q[:, :k] @ (Q[:, :k].conj().T @ V)) < 1e-12


@pytest.mark.parametrize("n", [1, 2, 7, 16, 33, 64])
def test_jacobi_eig(st, n):
    rng = np.random.default_rng(n)
    X = crand(rng, n, n + 5)
    H = X @ X.conj().T
    Hd = np.asfortranarray(H.copy())
    U = np.zeros((n, n), np.complex128, order="F")
    assert st.st_jacobi(P(Hd), n, P(U)) == 0
    lam = np.real(np.diag(Hd))
    ref = np.linalg.eigvalsh(H)
    assert np.allclose(np.sort(lam), ref, rtol=1e-12, atol=1e-12 * ref.max())
    assert np.abs(U.conj().T @ U - np.eye(n)).max() < 1e-13
    assert np.linalg.norm(U @ np.diag(lam) @ U.conj().T - H) < 1e-12 * np.linalg.norm(H)


@pytest.mark.parametrize("n", [1, 5, 32, 64])
def test_lu_and_inverses(st, n):
    rng = np.random.default_rng(n)
    A = crand(rng, n, n) + 10 * np.eye(n)
    LU = np.asfortranarray(A.copy())
    Li = np.zeros((n, n), np.complex128, order="F")
    Ui = np.zeros((n, n), np.complex128, order="F")
    fail, mag = C.c_int(0), C.c_double(0)
    assert st.st_lu(P(LU), n, P(Li), P(Ui), C.byref(fail), C.byref(mag)) == 0
    assert fail.value == -1
    L = np.tril(LU, -1) + np.eye(n)
    U = np.triu(LU)
    assert np.abs(L @ U - A).max() < 1e-12 * np.abs(A).max()
    assert np.abs(Li @ L - np.eye(n)).max() < 1e-12
    assert np.abs(Ui @ U - np.eye(n)).max() < 1e-12


def test_lu_singular_pivot(st):
    A = np.asfortranarray(np.array([[0.0, 1.0], [1.0, 0.0]], np.complex128))
    Li = np.zeros((2, 2), np.complex128, order="F")
    Ui = np.zeros((2, 2), np.complex128, order="F")
    fail, mag = C.c_int(0), C.c_double(1)
    st.st_lu(P(A), 2, P(Li), P(Ui), C.byref(fail), C.byref(mag))
    assert fail.value == 0 and mag.value == 0.0


@pytest.mark.parametrize("opA,opB", [(a, b) for a in range(4) for b in range(4)])
def test_cta_gemm_ops(st, opA, opB):
    rng = np.random.default_rng(opA * 4 + opB)
    m, n, k = 13, 9, 11
    def mk(op, r, c):
        X = np.asfortranarray(crand(rng, r, c) if op in (0, 3) else crand(rng, c, r))
        Y = {0: X, 1: X.T, 2: X.conj().T, 3: X.conj()}[op]
        return X, Y
    A, Aop = mk(opA, m, k)
    B, Bop = mk(opB, k, n)
    Cm = np.zeros((m, n), np.complex128, order="F")
    st.st_gemm(m, n, k, P(A), A.shape[0], opA, P(B), B.shape[0], opB, P(Cm))
    assert np.abs(Cm - Aop @ Bop).max() < 1e-12
