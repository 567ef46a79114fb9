"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/liboracle.so`` (the CPU restatement of the
reference h2lu hot path, see ``oracle/dense.hpp``). Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` leg import this module, and only as the checker / CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

KERNEL_LAPLACE, KERNEL_HELMHOLTZ, KERNEL_ZERO = 0, 1, 2
SCHEDULE_REFERENCE, SCHEDULE_COLORED, SCHEDULE_INTERIOR_FIRST = 0, 1, 3


class OracleError(RuntimeError):
    def __init__(self, code, msg, info=None, pivmag=0.0):
        super().__init__(msg)
        self.code = code
        self.info = info
        self.pivot_index = None if info is None else int(info[1])
        self.cluster = None if info is None else int(info[2])
        self.level = None if info is None else int(info[3])
        self.pivot_magnitude = pivmag


class InvalidInputError(OracleError):
    pass


class SizeGuardError(OracleError):
    pass


class NonFiniteError(OracleError):
    pass


class SingularPivotError(OracleError):
    pass


class UndefinedMetricError(OracleError):
    pass


_ERRS = {1: InvalidInputError, 2: SizeGuardError, 3: NonFiniteError, 4: SingularPivotError, 5: UndefinedMetricError}

P = C.c_void_p
D = C.POINTER(C.c_double)
I64 = C.POINTER(C.c_int64)
I32 = C.POINTER(C.c_int32)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            import subprocess

            subprocess.check_call(["make", "-s", "-C", _HERE])
        L = C.CDLL(path)
        sig = {
            "orc_last_error": (C.c_int, [C.c_char_p, C.c_int, I64, D]),
            "orc_rhs": (None, [C.c_int64, C.c_uint64, D]),
            "orc_tree_new": (P, [D, C.c_int64, C.c_int64]),
            "orc_tree_free": (None, [P]),
            "orc_tree_depth": (C.c_int, [P]),
            "orc_tree_n": (C.c_int64, [P]),
            "orc_tree_perm": (None, [P, I64]),
            "orc_tree_points": (None, [P, D]),
            "orc_tree_ranges": (None, [P, I64, I64]),
            "orc_blocks_new": (P, [P, C.c_double]),
            "orc_blocks_free": (None, [P]),
            "orc_blocks_l0": (C.c_int, [P]),
            "orc_blocks_csp": (C.c_int, [P, C.c_int]),
            "orc_blocks_counts": (None, [P, I64, I64, I64]),
            "orc_blocks_pairs": (None, [P, C.c_int, C.c_int, I32]),
            "orc_h2_build": (P, [P, C.c_int] + [C.c_double] * 7),
            "orc_h2_free": (None, [P]),
            "orc_h2_sizes": (None, [P, I64]),
            "orc_h2_export": (None, [P, I64, I64, I64, D, I64, D, I64, D]),
            "orc_h2_import": (P, [P, C.c_double, I64, I64, I64, D, I64, D, I64, D]),
            "orc_h2_rank": (C.c_int, [P, C.c_int]),
            "orc_h2_matvec": (C.c_int, [P, D, D]),
            "orc_h2_dense_shadow": (C.c_int, [P, D]),
            "orc_kernel_rows_matvec": (C.c_int, [P, C.c_int] + [C.c_double] * 6 + [I64, C.c_int64, D, D]),
            "orc_dense_solve": (C.c_int, [P, C.c_int] + [C.c_double] * 6 + [D, D]),
            "orc_shadow_solve": (C.c_int, [P, D, D]),
            "orc_factorize": (P, [P, C.c_double, C.c_int, C.c_int, D]),
            "orc_chain_free": (None, [P]),
            "orc_chain_info": (None, [P, I64]),
            "orc_chain_level": (None, [P, C.c_int, I64]),
            "orc_chain_records": (None, [P, C.c_int, I64]),
            "orc_chain_perm": (None, [P, C.c_int, I64]),
            "orc_chain_root": (None, [P, D, D]),
            "orc_chain_record_mats": (None, [P, C.c_int, C.c_int, D, D, D]),
            "orc_chain_hash": (C.c_uint64, [P]),
            "orc_solve": (C.c_int, [P, D, C.c_int64, D, C.c_int]),
            "orc_replay": (C.c_int, [P, P, D]),
            "orc_replay_factors": (C.c_int, [P, D, D]),
            "orc_relative_residual": (C.c_int, [P, D, D, D]),
            "orc_partial_lu": (C.c_int, [D, C.c_int64, D, D]),
            "orc_unitary_completion": (C.c_int, [D, C.c_int64, C.c_int64, D]),
            "orc_truncated_row_basis": (C.c_int, [D, C.c_int64, C.c_int64, C.c_double, C.c_double, D, I64]),
            "orc_test_stepwise": (C.c_int, [P, C.c_double, C.c_int, D]),
            "orc_test_fill_free_bits": (C.c_int, [P, C.c_double, D]),
            "orc_test_carried_embed": (C.c_int, [P, D]),
            "orc_h2_save": (C.c_int, [P, C.c_char_p]),
            "orc_h2_n": (C.c_int64, [P]),
            "orc_set_gemm_order": (None, [C.c_int]),
            "orc_set_truncation": (None, [C.c_int]),
            "orc_h2_load": (P, [C.c_char_p]),
            "orc_chain_save": (C.c_int, [P, C.c_char_p]),
            "orc_chain_load": (P, [C.c_char_p]),
            "orc_vector_save": (C.c_int, [C.c_char_p, D, C.c_int64]),
            "orc_vector_load": (C.c_int, [C.c_char_p, D, I64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _raise():
    buf = C.create_string_buffer(1024)
    info = np.zeros(4, np.int64)
    piv = C.c_double(0.0)
    code = lib().orc_last_error(buf, 1024, _i64(info), C.byref(piv))
    raise _ERRS.get(code, OracleError)(code, buf.value.decode(), info, piv.value)


def _check(rc):
    if rc != 0:
        _raise()


def _d(a):
    return a.ctypes.data_as(D)


def _i64(a):
    return a.ctypes.data_as(I64)


def _i32(a):
    return a.ctypes.data_as(I32)


def _cplx(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    if n is not None:
        assert a.size == n
    return a


def rhs(n, seed=1234):
    """Seeded complex-normal vector (mt19937_64 + std::normal_distribution)."""
    out = np.zeros(n, np.complex128)
    lib().orc_rhs(n, seed, _d(out.view(np.float64)))
    return out


@dataclass
class Kernel:
    kind: int = KERNEL_LAPLACE
    wavenumber: complex = 0.0
    scale: complex = 1.0
    diag: complex = 1.0

    def args(self):
        k, s, d = complex(self.wavenumber), complex(self.scale), complex(self.diag)
        return (self.kind, k.real, k.imag, s.real, s.imag, d.real, d.imag)


def laplace(shift=1.0):
    return Kernel(KERNEL_LAPLACE, 0.0, 1.0, shift)


def helmholtz(k, shift=1.0, scale=1.0):
    return Kernel(KERNEL_HELMHOLTZ, k, scale, shift)


def zero(shift=0.0):
    return Kernel(KERNEL_ZERO, 0.0, 0.0, shift)


class Tree:
    def __init__(self, points, leafsize):
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        self.h = lib().orc_tree_new(_d(pts), pts.shape[0], leafsize)
        if not self.h:
            _raise()
        self.n = int(lib().orc_tree_n(self.h))
        self.depth = int(lib().orc_tree_depth(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_tree_free(self.h)

    @property
    def perm(self):
        out = np.zeros(self.n, np.int64)
        lib().orc_tree_perm(self.h, _i64(out))
        return out

    @property
    def points(self):
        out = np.zeros((self.n, 3), np.float64)
        lib().orc_tree_points(self.h, _d(out))
        return out

    def ranges(self):
        nc = (2 << self.depth) - 1
        b = np.zeros(nc, np.int64)
        e = np.zeros(nc, np.int64)
        lib().orc_tree_ranges(self.h, _i64(b), _i64(e))
        return b, e

    def dense_solve(self, kernel, b):
        b = _cplx(b, self.n)
        x = np.zeros(self.n, np.complex128)
        _check(lib().orc_dense_solve(self.h, *kernel.args(), _d(b.view(np.float64)), _d(x.view(np.float64))))
        return x

    def kernel_rows_matvec(self, kernel, rows, x):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        x = _cplx(x, self.n)
        y = np.zeros(rows.size, np.complex128)
        _check(lib().orc_kernel_rows_matvec(self.h, *kernel.args(), _i64(rows), rows.size, _d(x.view(np.float64)), _d(y.view(np.float64))))
        return y


class Blocks:
    def __init__(self, tree, eta=1.0):
        self.tree = tree
        self.h = lib().orc_blocks_new(tree.h, eta)
        if not self.h:
            _raise()
        self.eta = eta
        self.depth = tree.depth
        self.l0 = int(lib().orc_blocks_l0(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_blocks_free(self.h)

    def csp(self, level):
        return int(lib().orc_blocks_csp(self.h, level))

    def counts(self):
        a = np.zeros(self.depth + 1, np.int64)
        s = np.zeros(self.depth + 1, np.int64)
        n = np.zeros(1, np.int64)
        lib().orc_blocks_counts(self.h, _i64(a), _i64(s), _i64(n))
        return a, s, int(n[0])

    def pairs(self, kind, level=0):
        a, s, n = self.counts()
        cnt = a[level] if kind == 0 else s[level] if kind == 1 else n
        out = np.zeros((int(cnt), 2), np.int32)
        if cnt:
            lib().orc_blocks_pairs(self.h, kind, level, _i32(out))
        return out

    def admissible(self, level):
        return self.pairs(0, level)

    def split(self, level):
        return self.pairs(1, level)

    def inadmissible_leaves(self):
        return self.pairs(2)


class H2:
    """Oracle H² matrix (built by the restated build_h2, or imported)."""

    def __init__(self, blocks, kernel=None, eps_h2=None, handle=None):
        self.blocks = blocks
        self.tree = blocks.tree
        self.kernel = kernel
        self.eps_h2 = eps_h2
        if handle is None:
            handle = lib().orc_h2_build(blocks.h, *kernel.args(), eps_h2)
            if not handle:
                _raise()
        self.h = handle
        self.n = self.tree.n

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_h2_free(self.h)

    def rank(self, cid):
        return int(lib().orc_h2_rank(self.h, cid))

    def export(self):
        """Flat arrays in the include/h2g.h layout."""
        sz = np.zeros(6, np.int64)
        lib().orc_h2_sizes(self.h, _i64(sz))
        nc, be, na, ce, nl, de = (int(v) for v in sz)
        out = dict(
            basis_rows=np.zeros(nc, np.int64),
            basis_rank=np.zeros(nc, np.int64),
            basis_offset=np.zeros(nc, np.int64),
            basis_data=np.zeros(be, np.complex128),
            coupling_offset=np.zeros(max(na, 1), np.int64),
            coupling_data=np.zeros(max(ce, 1), np.complex128),
            dense_offset=np.zeros(max(nl, 1), np.int64),
            dense_data=np.zeros(max(de, 1), np.complex128),
        )
        lib().orc_h2_export(
            self.h,
            _i64(out["basis_rows"]),
            _i64(out["basis_rank"]),
            _i64(out["basis_offset"]),
            _d(out["basis_data"].view(np.float64)),
            _i64(out["coupling_offset"]),
            _d(out["coupling_data"].view(np.float64)),
            _i64(out["dense_offset"]),
            _d(out["dense_data"].view(np.float64)),
        )
        return out

    def arrays(self):
        """Tree + partition + numerical data: the full include/h2g.h matrix
        description (what the GPU path's h2g_matrix_upload consumes)."""
        out = self.export()
        b, e = self.tree.ranges()
        L = self.tree.depth
        adm = [self.blocks.admissible(l) for l in range(L + 1)]
        spl = [self.blocks.split(l) for l in range(L + 1)]
        out.update(
            n=self.n,
            depth=L,
            eta=self.blocks.eta,
            eps_h2=self.eps_h2 or 0.0,
            cluster_begin=b,
            cluster_end=e,
            adm_offsets=np.concatenate([[0], np.cumsum([len(a) for a in adm])]).astype(np.int64),
            adm_pairs=np.ascontiguousarray(np.vstack(adm + [np.zeros((0, 2), np.int32)]).astype(np.int32)),
            split_offsets=np.concatenate([[0], np.cumsum([len(a) for a in spl])]).astype(np.int64),
            split_pairs=np.ascontiguousarray(np.vstack(spl + [np.zeros((0, 2), np.int32)]).astype(np.int32)),
            leaf_pairs=np.ascontiguousarray(self.blocks.inadmissible_leaves().astype(np.int32)),
        )
        for k in ("adm_pairs", "split_pairs", "leaf_pairs"):
            if out[k].shape[0] == 0:
                out[k] = np.zeros((1, 2), np.int32)
        return out

    @classmethod
    def from_arrays(cls, blocks, eps_h2, arrs, kernel=None):
        a = {k: np.ascontiguousarray(v) for k, v in arrs.items()}
        h = lib().orc_h2_import(
            blocks.h,
            eps_h2,
            _i64(a["basis_rows"]),
            _i64(a["basis_rank"]),
            _i64(a["basis_offset"]),
            _d(a["basis_data"].view(np.float64)),
            _i64(a["coupling_offset"]),
            _d(a["coupling_data"].view(np.float64)),
            _i64(a["dense_offset"]),
            _d(a["dense_data"].view(np.float64)),
        )
        if not h:
            _raise()
        return cls(blocks, kernel, eps_h2, handle=h)

    def matvec(self, x):
        x = _cplx(x, self.n)
        y = np.zeros(self.n, np.complex128)
        _check(lib().orc_h2_matvec(self.h, _d(x.view(np.float64)), _d(y.view(np.float64))))
        return y

    def dense_shadow(self):
        Z = np.zeros((self.n, self.n), np.complex128, order="F")
        _check(lib().orc_h2_dense_shadow(self.h, Z.ctypes.data_as(D)))
        return Z

    def shadow_solve(self, b):
        b = _cplx(b, self.n)
        x = np.zeros(self.n, np.complex128)
        _check(lib().orc_shadow_solve(self.h, _d(b.view(np.float64)), _d(x.view(np.float64))))
        return x

    def relative_residual(self, x, b):
        x = _cplx(x, self.n)
        b = _cplx(b, self.n)
        out = C.c_double(0.0)
        _check(lib().orc_relative_residual(self.h, _d(x.view(np.float64)), _d(b.view(np.float64)), C.byref(out)))
        return out.value

    def factorize(self, eps, stop_level=None, schedule=SCHEDULE_REFERENCE):
        secs = C.c_double(0.0)
        h = lib().orc_factorize(self.h, eps, -1 if stop_level is None else stop_level, schedule, C.byref(secs))
        if not h:
            _raise()
        return Chain(h, secs.value)

    def test_stepwise(self, eps_fill, schedule=SCHEDULE_REFERENCE):
        out = np.zeros(7)
        _check(lib().orc_test_stepwise(self.h, eps_fill, schedule, _d(out)))
        return dict(worst=out[0], stop_level=int(out[1]), root_size=int(out[2]), eliminated=int(out[3]),
                    root_err=out[4], orth=out[5], unitary=out[6])

    def test_fill_free_bits(self, eps_fill):
        out = np.zeros(3)
        _check(lib().orc_test_fill_free_bits(self.h, eps_fill, _d(out)))
        return dict(same_bits=bool(out[0]), ledger=int(out[1]), growth=bool(out[2]))

    def test_carried_embed(self):
        out = np.zeros(5)
        _check(lib().orc_test_carried_embed(self.h, _d(out)))
        return dict(shadow_err=out[0], carried_empty=bool(out[1]), ledger_found=bool(out[2]), quad_err=out[3], rest_norm=out[4])


REC_FIELDS = ("cluster", "level", "pos", "bsize", "eliminated", "rank_before", "rank_after", "fill_targets", "n_lbar", "n_ubar")
LEVEL_FIELDS = ("level", "nrecs", "rank_sum_before", "rank_sum_after", "eliminated", "ledger_blocks", "chain_bytes", "perm_len", "active_after")


class Chain:
    def __init__(self, h, seconds=0.0):
        self.h = h
        self.seconds = seconds
        info = np.zeros(5, np.int64)
        lib().orc_chain_info(h, _i64(info))
        self.n, self.stop_level, self.root_size, self.num_levels, self.storage_bytes = (int(v) for v in info)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_chain_free(self.h)

    def level(self, li):
        out = np.zeros(9, np.int64)
        lib().orc_chain_level(self.h, li, _i64(out))
        return dict(zip(LEVEL_FIELDS, (int(v) for v in out)))

    def levels(self):
        return [self.level(i) for i in range(self.num_levels)]

    def records(self, li):
        nrec = self.level(li)["nrecs"]
        out = np.zeros((nrec, 10), np.int64)
        if nrec:
            lib().orc_chain_records(self.h, li, _i64(out))
        return [dict(zip(REC_FIELDS, (int(v) for v in row))) for row in out]

    def all_records(self):
        recs = []
        for li in range(self.num_levels):
            recs.extend(self.records(li))
        return recs

    def perm(self, li):
        n = self.level(li)["perm_len"]
        out = np.zeros(n, np.int64)
        if n:
            lib().orc_chain_perm(self.h, li, _i64(out))
        return out

    def root(self):
        r = self.root_size
        L = np.zeros((r, r), np.complex128, order="F")
        U = np.zeros((r, r), np.complex128, order="F")
        if r:
            lib().orc_chain_root(self.h, L.ctypes.data_as(D), U.ctypes.data_as(D))
        return L, U

    def record_mats(self, li, ri):
        rec = self.records(li)[ri]
        b, e = rec["bsize"], rec["eliminated"]
        Q = np.zeros((b, b), np.complex128, order="F")
        L = np.zeros((e, e), np.complex128, order="F")
        U = np.zeros((e, e), np.complex128, order="F")
        lib().orc_chain_record_mats(self.h, li, ri, Q.ctypes.data_as(D), L.ctypes.data_as(D) if e else None, U.ctypes.data_as(D) if e else None)
        return Q, L, U

    def hash(self):
        return int(lib().orc_chain_hash(self.h))

    def _solve(self, b, mode):
        b = _cplx(b, None)
        x = np.zeros(b.size, np.complex128)
        _check(lib().orc_solve(self.h, _d(b.view(np.float64)), b.size, _d(x.view(np.float64)), mode))
        return x

    def solve(self, b):
        return self._solve(b, 0)

    def forward(self, b):
        return self._solve(b, 1)

    def backward(self, b):
        return self._solve(b, 2)

    def apply_inverse(self, b):
        return self._solve(b, 3)

    def replay_error(self, h2):
        out = C.c_double(0.0)
        _check(lib().orc_replay(self.h, h2.h, C.byref(out)))
        return out.value

    def replay_factors(self):
        n = self.n
        L = np.zeros((n, n), np.complex128, order="F")
        U = np.zeros((n, n), np.complex128, order="F")
        _check(lib().orc_replay_factors(self.h, L.ctypes.data_as(D), U.ctypes.data_as(D)))
        return L, U


def partial_lu(F):
    F = np.asfortranarray(F, dtype=np.complex128)
    n = F.shape[0]
    L = np.zeros((n, n), np.complex128, order="F")
    U = np.zeros((n, n), np.complex128, order="F")
    _check(lib().orc_partial_lu(F.ctypes.data_as(D), n, L.ctypes.data_as(D), U.ctypes.data_as(D)))
    return L, U


def unitary_completion(V):
    V = np.asfortranarray(V, dtype=np.complex128)
    m, k = V.shape
    Pm = np.zeros((m, m - k), np.complex128, order="F")
    _check(lib().orc_unitary_completion(V.ctypes.data_as(D), m, k, Pm.ctypes.data_as(D)))
    return Pm


def truncated_row_basis(B, eps, floor=0.0):
    B = np.asfortranarray(B, dtype=np.complex128)
    m, f = B.shape
    U = np.zeros((m, max(min(m, f), 1)), np.complex128, order="F")
    r = np.zeros(1, np.int64)
    _check(lib().orc_truncated_row_basis(B.ctypes.data_as(D), m, f, eps, floor, U.ctypes.data_as(D), _i64(r)))
    return U[:, : int(r[0])]


# ------------------------------------------- H2LU v1 container (serialize.hpp)
def save_h2(A, path):
    _check(lib().orc_h2_save(A.h, os.fsencode(path)))


def load_h2(path):
    """load_h2: tree from the file, partition recomputed (serialize.hpp:198-243)."""
    h = lib().orc_h2_load(os.fsencode(path))
    if not h:
        _raise()
    A = H2.__new__(H2)
    A.h = h
    A.kernel = None
    A.eps_h2 = None
    A.blocks = None
    A.tree = None
    A.n = int(lib().orc_h2_n(h))
    return A


def save_chain(ch, path):
    _check(lib().orc_chain_save(ch.h, os.fsencode(path)))


def load_chain(path):
    h = lib().orc_chain_load(os.fsencode(path))
    if not h:
        _raise()
    return Chain(h)


def save_vector(path, v):
    v = np.ascontiguousarray(v, dtype=np.complex128).reshape(-1)
    _check(lib().orc_vector_save(os.fsencode(path), _d(v.view(np.float64)), v.size))


def load_vector(path):
    n = np.zeros(1, np.int64)
    _check(lib().orc_vector_load(os.fsencode(path), None, _i64(n)))
    v = np.zeros(int(n[0]), np.complex128)
    _check(lib().orc_vector_load(os.fsencode(path), _d(v.view(np.float64)), _i64(n)))
    return v


def set_gemm_order(reverse):
    """Oracle self-noise switch: GEMM inner products accumulated last-to-first."""
    lib().orc_set_gemm_order(1 if reverse else 0)


def set_truncation(mode):
    """Oracle self-noise switch: 1 = step-0 truncation through the Gram of the
    projected fill (the paper's Eq. 16-18, as the GPU does), 0 = QR + SVD."""
    lib().orc_set_truncation(int(mode))
