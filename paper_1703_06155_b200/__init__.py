"""B200-native H² factorize / solve (arXiv 1703.06155), Python mirror of the
reference h2lu API over the C ABI of ``include/h2g.h`` (``libh2g.so``).

Reference interface mirrored (paths under /root/reference/proj):
  factorize(A, eps_fill_in, stop_level_override)  include/h2lu/factorization.hpp:600
  solve / solve_in_place / apply_inverse           include/h2lu/solve.hpp:99-113
  forward_substitute / backward_substitute         include/h2lu/solve.hpp:85-97
  FactorChain fields (levels, records, root)       include/h2lu/factorization.hpp:22-98
  error types                                      include/h2lu/types.hpp:18-47
Vectors are in tree order, like the reference library. The compute path is
CUDA only: without the built library or without a device every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import geometry  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("H2G_LIB", os.path.join(_HERE, "libh2g.so"))

SCHEDULES = {"reference": 0, "colored": 1, "serial": 2, "interior-first": 3, "subtree": 4}
KERNEL_LAPLACE, KERNEL_HELMHOLTZ, KERNEL_ZERO = 0, 1, 2
_SOLVE, _FORWARD, _BACKWARD, _APPLY_INVERSE, _APPLY_INVERSE_EXPLICIT = 0, 1, 2, 3, 4


class H2GError(RuntimeError):
    code = 9

    def __init__(self, msg, cluster=-1, level=-1, pivot_index=-1, pivot_magnitude=0.0):
        super().__init__(msg)
        self.cluster = cluster
        self.level = level
        self.pivot_index = pivot_index
        self.pivot_magnitude = pivot_magnitude


class InvalidInputError(H2GError):
    code = 1


class SizeGuardError(H2GError):
    code = 2


class NonFiniteError(H2GError):
    code = 3


class SingularPivotError(H2GError):
    code = 4


class UndefinedMetricError(H2GError):
    code = 5


class CudaError(H2GError):
    code = 8


_ERR = {1: InvalidInputError, 2: SizeGuardError, 3: NonFiniteError, 4: SingularPivotError, 5: UndefinedMetricError, 8: CudaError}


class _Err(C.Structure):
    _fields_ = [
        ("code", C.c_int32),
        ("cluster", C.c_int32),
        ("level", C.c_int32),
        ("pad", C.c_int32),
        ("pivot_index", C.c_int64),
        ("pivot_magnitude", C.c_double),
        ("msg", C.c_char * 256),
    ]


class _Kernel(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("pad", C.c_int32),
        ("wavenumber_re", C.c_double),
        ("wavenumber_im", C.c_double),
        ("scale_re", C.c_double),
        ("scale_im", C.c_double),
        ("diag_re", C.c_double),
        ("diag_im", C.c_double),
    ]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_I32 = C.POINTER(C.c_int32)


class _Desc(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("depth", C.c_int32),
        ("pad", C.c_int32),
        ("eta", C.c_double),
        ("eps_h2", C.c_double),
        ("cluster_begin", _I64),
        ("cluster_end", _I64),
        ("adm_offsets", _I64),
        ("adm_pairs", _I32),
        ("split_offsets", _I64),
        ("split_pairs", _I32),
        ("num_leaf_pairs", C.c_int64),
        ("leaf_pairs", _I32),
        ("basis_rows", _I64),
        ("basis_rank", _I64),
        ("basis_offset", _I64),
        ("basis_data", _D),
        ("coupling_offset", _I64),
        ("coupling_data", _D),
        ("dense_offset", _I64),
        ("dense_data", _D),
        ("points_tree", _D),
        ("perm", _I64),
        ("leafsize", C.c_int64),
    ]


# Public C symbols (kept in sync with include/h2g.h; the CPU tests check both).
SYMBOLS = {
    "h2g_version": (C.c_char_p, []),
    "h2g_device_count": (C.c_int, []),
    "h2g_context_create": (C.c_int, [C.c_int, C.POINTER(_P), C.POINTER(_Err)]),
    "h2g_context_destroy": (C.c_int, [_P]),
    "h2g_last_error": (C.c_int, [C.POINTER(_Err)]),
    "h2g_matrix_upload": (C.c_int, [_P, C.POINTER(_Desc), C.POINTER(_P), C.POINTER(_Err)]),
    "h2g_matrix_build": (C.c_int, [_P, _D, C.c_int64, C.c_int64, C.c_double, C.POINTER(_Kernel), C.c_double, C.POINTER(_P), C.POINTER(_Err)]),
    "h2g_matrix_destroy": (C.c_int, [_P]),
    "h2g_matrix_sizes": (C.c_int, [_P, _I64]),
    "h2g_matrix_download": (C.c_int, [_P, _I64, _I64, _I64, _I64, _I32, _I64, _I32, _I32, _I64, _I64, _I64, _D, _I64, _D, _I64, _D]),
    "h2g_matvec": (C.c_int, [_P, _P, _D, _D, C.c_int32, C.POINTER(_Err)]),
    "h2g_kernel_rows_matvec": (C.c_int, [_P, _D, C.c_int64, C.POINTER(_Kernel), _I64, C.c_int64, _D, _D, C.c_int32, C.POINTER(_Err)]),
    "h2g_factorize": (C.c_int, [_P, _P, C.c_double, C.c_int32, C.c_int32, C.POINTER(_P), C.POINTER(_Err)]),
    "h2g_chain_destroy": (C.c_int, [_P]),
    "h2g_solve": (C.c_int, [_P, _D, _D, C.c_int64, C.c_int32, C.c_int32, C.POINTER(_Err)]),
    "h2g_solve_device": (C.c_int, [_P, _D, C.c_int64, C.c_int32, C.c_int32, C.POINTER(_Err)]),
    "h2g_chain_info": (C.c_int, [_P, _I64]),
    "h2g_chain_level": (C.c_int, [_P, C.c_int32, _I64]),
    "h2g_chain_records": (C.c_int, [_P, C.c_int32, _I64]),
    "h2g_chain_perm": (C.c_int, [_P, C.c_int32, _I64]),
    "h2g_chain_record_mats": (C.c_int, [_P, C.c_int32, C.c_int32, _D, _D, _D]),
    "h2g_chain_record_blocks_sizes": (C.c_int, [_P, C.c_int32, C.c_int32, _I64]),
    "h2g_chain_record_blocks": (C.c_int, [_P, C.c_int32, C.c_int32, _I64, _I64, _D, _I64, _I64, _D]),
    "h2g_chain_root": (C.c_int, [_P, _D, _D]),
    "h2g_chain_hash": (C.c_uint64, [_P]),
    "h2g_chain_timing": (C.c_int, [_P, _D, _D, _I64, _I64]),
    "h2g_chain_work": (C.c_int, [_P, _D]),
    "h2g_chain_schur_executed": (C.c_int, [_P, _D]),
    "h2g_random_rhs": (None, [C.c_int64, C.c_uint64, _D]),
    "h2g_set_profiling": (C.c_int, [_P, C.c_int32]),
    "h2g_chain_plan": (C.c_int, [_P, _D, _I32]),
    "h2g_matrix_save": (C.c_int, [_P, C.c_char_p, C.POINTER(_Err)]),
    "h2g_matrix_load": (C.c_int, [_P, C.c_char_p, C.POINTER(_P), C.POINTER(_Err)]),
    "h2g_chain_save": (C.c_int, [_P, _P, C.c_char_p, C.POINTER(_Err)]),
    "h2g_chain_load": (C.c_int, [_P, C.c_char_p, C.POINTER(_P), C.POINTER(_Err)]),
    "h2g_vector_save": (C.c_int, [C.c_char_p, _D, C.c_int64, C.POINTER(_Err)]),
    "h2g_chain_perm_tree": (C.c_int, [_P, _I64]),
    "h2g_factorize_hooked": (C.c_int, [_P, _P, C.c_double, C.c_int32, C.c_void_p, C.POINTER(_P), C.POINTER(_Err)]),
    "h2g_state_info": (C.c_int, [_P, _I64]),
    "h2g_state_cluster": (C.c_int, [_P, C.c_int32, _I64]),
    "h2g_state_qtilde": (C.c_int, [_P, C.c_int32, _D]),
    "h2g_state_shadow": (C.c_int, [_P, _D]),
    "h2g_state_perm": (C.c_int, [_P, _I64, _I64]),
    "h2g_vector_load": (C.c_int, [C.c_char_p, _D, _I64, C.POINTER(_Err)]),
    "h2g_context_clear_plans": (C.c_int, [_P]),
    "h2g_chain_kernel_stats": (C.c_int, [_P, C.c_int32, _D]),
    "h2g_factorize_dist": (C.c_int, [_P, _P, C.c_double, C.c_int32, C.c_void_p, C.POINTER(_P), C.POINTER(_Err)]),
    "h2g_chain_dist_stats": (C.c_int, [_P, _D]),
    "h2g_chain_schur_levels": (C.c_int, [_P, _I32, _D]),
    "h2g_partition_plan": (C.c_int, [C.POINTER(_Desc), C.c_int32, C.c_int32, _I64, _I32, _I32, _I32, _I32, _I32, _I32, C.POINTER(_Err)]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load libh2g.so (raises if it was not built: there is no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C paper_1703_06155_b200)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SYMBOLS.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _raise(err):
    cls = _ERR.get(err.code, H2GError)
    raise cls(err.msg.decode(errors="replace"), err.cluster, err.level, err.pivot_index, err.pivot_magnitude)


def _check(rc, err):
    if rc != 0:
        _raise(err)


def _d(a):
    return a.ctypes.data_as(_D)


def _i64(a):
    return a.ctypes.data_as(_I64)


def _i32(a):
    return a.ctypes.data_as(_I32)


def _desc_from_arrays(arrays, keep):
    """h2g_matrix_desc over host arrays; the converted arrays are appended to
    `keep`, which must outlive the C call."""
    # every array converted to the dtype the C ABI reads; the converted
    # arrays stay referenced by `a` until h2g_matrix_upload returns
    i64 = ("cluster_begin", "cluster_end", "adm_offsets", "split_offsets", "basis_rows", "basis_rank", "basis_offset",
           "coupling_offset", "dense_offset")
    i32 = ("adm_pairs", "split_pairs", "leaf_pairs")
    cpx = ("basis_data", "coupling_data", "dense_data")
    a = {}
    keep.append(a)
    for k in i64:
        a[k] = np.ascontiguousarray(arrays[k], dtype=np.int64)
    for k in i32:
        a[k] = np.ascontiguousarray(np.asarray(arrays[k]).reshape(-1, 2), dtype=np.int32)
    for k in cpx:
        a[k] = np.ascontiguousarray(arrays[k], dtype=np.complex128)
    d = _Desc()

    def scalar(v):
        return np.asarray(v).reshape(-1)[0]

    d.n = int(scalar(arrays["n"]))
    d.depth = int(scalar(arrays["depth"]))
    d.eta = float(scalar(arrays.get("eta", 1.0)))
    d.eps_h2 = float(scalar(arrays.get("eps_h2", 0.0)))
    d.cluster_begin = _i64(a["cluster_begin"])
    d.cluster_end = _i64(a["cluster_end"])
    d.adm_offsets = _i64(a["adm_offsets"])
    d.adm_pairs = _i32(a["adm_pairs"])
    d.split_offsets = _i64(a["split_offsets"])
    d.split_pairs = _i32(a["split_pairs"])
    d.num_leaf_pairs = int(a["leaf_pairs"].shape[0])
    d.leaf_pairs = _i32(a["leaf_pairs"])
    d.basis_rows = _i64(a["basis_rows"])
    d.basis_rank = _i64(a["basis_rank"])
    d.basis_offset = _i64(a["basis_offset"])
    d.basis_data = _d(a["basis_data"].view(np.float64))
    d.coupling_offset = _i64(a["coupling_offset"])
    d.coupling_data = _d(a["coupling_data"].view(np.float64))
    d.dense_offset = _i64(a["dense_offset"])
    d.dense_data = _d(a["dense_data"].view(np.float64))
    if arrays.get("points_tree") is not None and arrays.get("perm") is not None:
        a["points_tree"] = np.ascontiguousarray(arrays["points_tree"], dtype=np.float64).reshape(-1, 3)
        a["perm"] = np.ascontiguousarray(arrays["perm"], dtype=np.int64)
        d.points_tree = _d(a["points_tree"])
        d.perm = _i64(a["perm"])
        d.leafsize = int(scalar(arrays.get("leafsize", 0)))
    return d


class Context:
    """One CUDA device + stream."""

    _default = {}

    def __init__(self, device=0):
        err = _Err()
        h = _P()
        _check(lib().h2g_context_create(device, C.byref(h), C.byref(err)), err)
        self.h = h
        self.device = device

    def set_profiling(self, on=True):
        lib().h2g_set_profiling(self.h, 1 if on else 0)

    def clear_plans(self):
        """Forget the structure-keyed plan cache (next factorize of a new
        matrix builds its symbolic plan from scratch)."""
        lib().h2g_context_clear_plans(self.h)

    @classmethod
    def default(cls, device=0):
        if device not in cls._default:
            cls._default[device] = cls(device)
        return cls._default[device]

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.h2g_context_destroy(self.h)
            self.h = None


def device_count():
    return int(lib().h2g_device_count())


class Kernel:
    """Kernel spec (kernel.hpp:13-61 with a complex diagonal)."""

    def __init__(self, kind=KERNEL_LAPLACE, wavenumber=0.0, scale=1.0, diag=1.0):
        self.kind, self.wavenumber, self.scale, self.diag = kind, complex(wavenumber), complex(scale), complex(diag)

    def c(self):
        return _Kernel(self.kind, 0, self.wavenumber.real, self.wavenumber.imag, self.scale.real, self.scale.imag, self.diag.real, self.diag.imag)


def laplace_kernel(shift=1.0):
    return Kernel(KERNEL_LAPLACE, 0.0, 1.0, shift)


def helmholtz_kernel(k, shift=1.0, scale=1.0):
    return Kernel(KERNEL_HELMHOLTZ, k, scale, shift)


def zero_kernel(shift=0.0):
    return Kernel(KERNEL_ZERO, 0.0, 0.0, shift)


def vie_kernel(cells_per_side, side_lambda, eps_r=4.0):
    k0, scale, diag = geometry.vie_constants(cells_per_side, side_lambda, eps_r)
    return Kernel(KERNEL_HELMHOLTZ, k0, scale, diag)


class H2Matrix:
    """Device-resident H² matrix (the input of factorize; never modified)."""

    def __init__(self, handle, ctx):
        self.h = handle
        self.ctx = ctx
        sz = np.zeros(8, np.int64)
        lib().h2g_matrix_sizes(self.h, _i64(sz))
        self.n, self.depth, self.num_clusters, self.num_adm, self.num_leaf_pairs, self.basis_elems, self.coupling_elems, self.dense_elems = (int(v) for v in sz)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.h2g_matrix_destroy(self.h)
            self.h = None

    @classmethod
    def upload(cls, arrays, ctx=None):
        """From host arrays in the include/h2g.h layout (keys as exported by
        oracle/pyoracle.H2.export() plus the tree/partition arrays)."""
        ctx = ctx or Context.default()
        a = []
        d = _desc_from_arrays(arrays, a)
        err = _Err()
        h = _P()
        rc = lib().h2g_matrix_upload(ctx.h, C.byref(d), C.byref(h), C.byref(err))
        del a
        _check(rc, err)
        return cls(h, ctx)

    @classmethod
    def build(cls, points, leafsize, eta, kernel, eps_h2, ctx=None):
        """Tree + partition on the host, H² construction on the device."""
        ctx = ctx or Context.default()
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        err = _Err()
        h = _P()
        kc = kernel.c()
        _check(lib().h2g_matrix_build(ctx.h, _d(pts), pts.shape[0], leafsize, eta, C.byref(kc), eps_h2, C.byref(h), C.byref(err)), err)
        return cls(h, ctx)

    def save(self, path):
        """save_h2 (serialize.hpp:186-196): the H2LU v1 container."""
        err = _Err()
        _check(lib().h2g_matrix_save(self.h, os.fsencode(path), C.byref(err)), err)

    @classmethod
    def load(cls, path, ctx=None):
        """load_h2 (serialize.hpp:198-243) onto the device."""
        ctx = ctx or Context.default()
        err = _Err()
        h = _P()
        _check(lib().h2g_matrix_load(ctx.h, os.fsencode(path), C.byref(h), C.byref(err)), err)
        return cls(h, ctx)

    def perm(self):
        """Tree permutation (tree index -> original index) without the data."""
        out = np.zeros(self.n, np.int64)
        if lib().h2g_matrix_download(self.h, None, None, _i64(out), *([None] * 13)):
            raise H2GError("download failed")
        return out

    def download(self):
        nc, L = self.num_clusters, self.depth
        o = dict(
            cluster_begin=np.zeros(nc, np.int64),
            cluster_end=np.zeros(nc, np.int64),
            perm=np.zeros(self.n, np.int64),
            adm_offsets=np.zeros(L + 2, np.int64),
            adm_pairs=np.zeros((max(self.num_adm, 1), 2), np.int32),
            split_offsets=np.zeros(L + 2, np.int64),
            split_pairs=np.zeros((max(nc, 1), 2), np.int32),
            leaf_pairs=np.zeros((max(self.num_leaf_pairs, 1), 2), np.int32),
            basis_rows=np.zeros(nc, np.int64),
            basis_rank=np.zeros(nc, np.int64),
            basis_offset=np.zeros(nc, np.int64),
            basis_data=np.zeros(max(self.basis_elems, 1), np.complex128),
            coupling_offset=np.zeros(max(self.num_adm, 1), np.int64),
            coupling_data=np.zeros(max(self.coupling_elems, 1), np.complex128),
            dense_offset=np.zeros(max(self.num_leaf_pairs, 1), np.int64),
            dense_data=np.zeros(max(self.dense_elems, 1), np.complex128),
        )
        # split pair count is only known after the offsets: two passes
        rc = lib().h2g_matrix_download(self.h, *([None] * 3), _i64(o["adm_offsets"]), None, _i64(o["split_offsets"]), *([None] * 10))
        if rc:
            raise H2GError("download failed")
        o["split_pairs"] = np.zeros((max(int(o["split_offsets"][-1]), 1), 2), np.int32)
        rc = lib().h2g_matrix_download(
            self.h, _i64(o["cluster_begin"]), _i64(o["cluster_end"]), _i64(o["perm"]), _i64(o["adm_offsets"]), _i32(o["adm_pairs"]),
            _i64(o["split_offsets"]), _i32(o["split_pairs"]), _i32(o["leaf_pairs"]), _i64(o["basis_rows"]), _i64(o["basis_rank"]),
            _i64(o["basis_offset"]), _d(o["basis_data"].view(np.float64)), _i64(o["coupling_offset"]), _d(o["coupling_data"].view(np.float64)),
            _i64(o["dense_offset"]), _d(o["dense_data"].view(np.float64)))
        if rc:
            raise H2GError("download failed")
        o["n"], o["depth"] = self.n, self.depth
        return o

    def matvec(self, x):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        nrhs = 1 if x.ndim == 1 else x.shape[1]
        xf = np.asfortranarray(x.reshape(self.n, nrhs))
        y = np.zeros((self.n, nrhs), np.complex128, order="F")
        err = _Err()
        _check(lib().h2g_matvec(self.ctx.h, self.h, xf.ctypes.data_as(_D), y.ctypes.data_as(_D), nrhs, C.byref(err)), err)
        return y[:, 0].copy() if x.ndim == 1 else y

    def relative_residual(self, x, b):
        """||A x - b|| / ||b|| through the compressed operator (verify.hpp:14-19)."""
        nb = np.linalg.norm(b)
        if nb == 0.0:
            raise UndefinedMetricError("relative_residual: right-hand side is zero")
        return float(np.linalg.norm(self.matvec(x) - b) / nb)


def kernel_rows_matvec(points_tree, kernel, rows, x, ctx=None):
    """(Z x)[rows] with Z generated from the kernel on the device: the dense
    sampled-row residual of SURVEY §8d(ii). points_tree: n x 3 in tree order;
    rows: tree indices; x: tree order (n or n x nrhs)."""
    ctx = ctx or Context.default()
    pts = np.ascontiguousarray(points_tree, dtype=np.float64).reshape(-1, 3)
    n = pts.shape[0]
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    x = np.asarray(x, dtype=np.complex128)
    nrhs = 1 if x.ndim == 1 else x.shape[1]
    xf = np.asfortranarray(x.reshape(n, nrhs))
    y = np.zeros((rows.size, nrhs), np.complex128, order="F")
    err = _Err()
    kc = kernel.c()
    _check(lib().h2g_kernel_rows_matvec(ctx.h, _d(pts), n, C.byref(kc), _i64(rows), rows.size, xf.ctypes.data_as(_D), y.ctypes.data_as(_D),
                                        nrhs, C.byref(err)), err)
    return y[:, 0].copy() if x.ndim == 1 else y


def sampled_dense_residual(points_tree, kernel, x, b, rows, ctx=None):
    """||(Z x - b)[rows]|| / ||b[rows]|| on the device."""
    zx = kernel_rows_matvec(points_tree, kernel, rows, x, ctx)
    return float(np.linalg.norm(zx - b[rows]) / np.linalg.norm(b[rows]))


REC_FIELDS = ("cluster", "level", "pos", "bsize", "eliminated", "rank_before", "rank_after", "fill_targets", "n_lbar", "n_ubar")
LEVEL_FIELDS = ("level", "nrecs", "rank_sum_before", "rank_sum_after", "eliminated", "ledger_blocks", "chain_bytes", "perm_len", "active_after")


class FactorChain:
    """Device-resident factorization (FactorChain, factorization.hpp:76-98)."""

    def __init__(self, handle, matrix, ctx=None):
        self.h = handle
        self.matrix = matrix  # the factorized matrix (None for a chain loaded from a file)
        self.ctx = ctx or (matrix.ctx if matrix is not None else None)
        info = np.zeros(6, np.int64)
        lib().h2g_chain_info(self.h, _i64(info))
        self.n, self.stop_level, self.root_size, self.num_levels, self.storage_bytes, sch = (int(v) for v in info)
        self.schedule = {v: k for k, v in SCHEDULES.items()}[sch]

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.h2g_chain_destroy(self.h)
            self.h = None

    def tree_perm(self):
        """Tree permutation of the factorized matrix (tree index -> original index)."""
        out = np.zeros(self.n, np.int64)
        lib().h2g_chain_perm_tree(self.h, _i64(out))
        return out

    def level(self, li):
        out = np.zeros(9, np.int64)
        lib().h2g_chain_level(self.h, li, _i64(out))
        return dict(zip(LEVEL_FIELDS, (int(v) for v in out)))

    def levels(self):
        return [self.level(i) for i in range(self.num_levels)]

    def records(self, li):
        n = self.level(li)["nrecs"]
        out = np.zeros((n, 10), np.int64)
        if n:
            lib().h2g_chain_records(self.h, li, _i64(out))
        return [dict(zip(REC_FIELDS, (int(v) for v in row))) for row in out]

    def all_records(self):
        r = []
        for li in range(self.num_levels):
            r.extend(self.records(li))
        return r

    def perm(self, li):
        n = self.level(li)["perm_len"]
        out = np.zeros(n, np.int64)
        if n:
            lib().h2g_chain_perm(self.h, li, _i64(out))
        return out

    def record_mats(self, li, ri):
        rec = self.records(li)[ri]
        b, e = rec["bsize"], rec["eliminated"]
        Q = np.zeros((b, b), np.complex128, order="F")
        L = np.zeros((e, e), np.complex128, order="F")
        U = np.zeros((e, e), np.complex128, order="F")
        lib().h2g_chain_record_mats(self.h, li, ri, Q.ctypes.data_as(_D), L.ctypes.data_as(_D), U.ctypes.data_as(_D))
        return Q, L, U

    def record_blocks(self, li, ri):
        """(Lbar, Ubar) as lists of (pos, matrix) in record order."""
        rec = self.records(li)[ri]
        e = rec["eliminated"]
        sz = np.zeros(4, np.int64)
        lib().h2g_chain_record_blocks_sizes(self.h, li, ri, _i64(sz))
        nl, el, nu, eu = (int(v) for v in sz)
        lp, lr = np.zeros(max(nl, 1), np.int64), np.zeros(max(nl, 1), np.int64)
        up, uc = np.zeros(max(nu, 1), np.int64), np.zeros(max(nu, 1), np.int64)
        ld, ud = np.zeros(max(el, 1), np.complex128), np.zeros(max(eu, 1), np.complex128)
        if nl or nu:
            lib().h2g_chain_record_blocks(self.h, li, ri, _i64(lp), _i64(lr), _d(ld.view(np.float64)), _i64(up), _i64(uc), _d(ud.view(np.float64)))
        Lb, Ub = [], []
        off = 0
        for q in range(nl):
            r = int(lr[q])
            Lb.append((int(lp[q]), ld[off: off + r * e].reshape((r, e), order="F")))
            off += r * e
        off = 0
        for q in range(nu):
            c = int(uc[q])
            Ub.append((int(up[q]), ud[off: off + e * c].reshape((e, c), order="F")))
            off += e * c
        return Lb, Ub

    def root(self):
        r = self.root_size
        L = np.zeros((r, r), np.complex128, order="F")
        U = np.zeros((r, r), np.complex128, order="F")
        if r:
            lib().h2g_chain_root(self.h, L.ctypes.data_as(_D), U.ctypes.data_as(_D))
        return L, U

    def hash(self):
        return int(lib().h2g_chain_hash(self.h))

    def schur_levels(self):
        """k_schur per level: executed flops / bytes and (profiled runs) ms."""
        n = C.c_int32()
        lib().h2g_chain_schur_levels(self.h, C.byref(n), None)
        out = np.zeros(4 * max(n.value, 1))
        lib().h2g_chain_schur_levels(self.h, C.byref(n), _d(out))
        return [dict(level=int(out[4 * i]), flops=out[4 * i + 1], bytes=out[4 * i + 2], ms=out[4 * i + 3]) for i in range(n.value)]

    def dist_stats(self):
        """factorize_dist: bytes this rank contributed / bytes exchanged by all
        ranks / seconds inside the exchange callback."""
        out = np.zeros(3)
        lib().h2g_chain_dist_stats(self.h, _d(out))
        return dict(sent_bytes=out[0], total_bytes=out[1], exchange_s=out[2])

    def timing(self):
        f, s = C.c_double(), C.c_double()
        fl, sl = C.c_int64(), C.c_int64()
        lib().h2g_chain_timing(self.h, C.byref(f), C.byref(s), C.byref(fl), C.byref(sl))
        pm, built = C.c_double(), C.c_int32()
        lib().h2g_chain_plan(self.h, C.byref(pm), C.byref(built))
        return dict(factor_ms=f.value, solve_ms=s.value, factor_launches=fl.value, solve_launches=sl.value, plan_ms=pm.value,
                    plan_built=bool(built.value))

    KERNEL_CLASSES = ("complement", "gram", "colnorm", "eig1", "head", "panel", "schur", "merge", "root", "other", "eigvec", "eig1b")

    def kernel_stats(self):
        """Per kernel class: device ms, launches, algorithmic flops and bytes
        (requires Context.set_profiling(True) before factorize)."""
        out = {}
        for i, name in enumerate(self.KERNEL_CLASSES):
            v = np.zeros(4)
            lib().h2g_chain_kernel_stats(self.h, i, _d(v))
            out[name] = dict(ms=v[0], launches=int(v[1]), flops=v[2], bytes=v[3])
        return out

    def work(self):
        out = np.zeros(4)
        lib().h2g_chain_work(self.h, _d(out))
        ex = np.zeros(2)
        lib().h2g_chain_schur_executed(self.h, _d(ex))
        return dict(factor_flops=out[0], schur_flops=out[1], solve_bytes=out[2], schur_bytes=out[3],
                    schur_flops_executed=ex[0], schur_bytes_executed=ex[1])

    def _solve(self, b, mode):
        b = np.asarray(b)
        nrhs = 1 if b.ndim == 1 else b.shape[1]
        n = b.shape[0]
        bf = np.asfortranarray(b.reshape(n, nrhs), dtype=np.complex128)
        x = np.zeros((n, nrhs), np.complex128, order="F")
        err = _Err()
        _check(lib().h2g_solve(self.h, bf.ctypes.data_as(_D), x.ctypes.data_as(_D), n, nrhs, mode, C.byref(err)), err)
        return x[:, 0].copy() if b.ndim == 1 else x

    def solve(self, b):
        return self._solve(b, _SOLVE)

    def forward(self, b):
        return self._solve(b, _FORWARD)

    def backward(self, y):
        return self._solve(y, _BACKWARD)

    def apply_inverse(self, b):
        return self._solve(b, _APPLY_INVERSE)

    def apply_inverse_explicit(self, b):
        return self._solve(b, _APPLY_INVERSE_EXPLICIT)

    def solve_device(self, ptr, n, nrhs=1, mode=_SOLVE):
        """In-place solve on device memory (pointer from e.g. torch.Tensor.data_ptr())."""
        err = _Err()
        _check(lib().h2g_solve_device(self.h, C.cast(C.c_void_p(ptr), _D), n, nrhs, mode, C.byref(err)), err)


def save_chain(chain, path, matrix=None):
    """save_chain (serialize.hpp:245-284); the tree comes from the factorized matrix."""
    m = matrix or chain.matrix
    if m is None:
        raise InvalidInputError("save_chain: the source matrix is needed for the tree")
    err = _Err()
    _check(lib().h2g_chain_save(chain.h, m.h, os.fsencode(path), C.byref(err)), err)


def load_chain(path, ctx=None):
    """load_chain (serialize.hpp:286-343) into a device chain h2g_solve applies."""
    ctx = ctx or Context.default()
    err = _Err()
    h = _P()
    _check(lib().h2g_chain_load(ctx.h, os.fsencode(path), C.byref(h), C.byref(err)), err)
    return FactorChain(h, None, ctx)


def save_vector(path, v):
    """save_vector (serialize.hpp:345-348)."""
    v = np.ascontiguousarray(v, dtype=np.complex128).reshape(-1)
    err = _Err()
    _check(lib().h2g_vector_save(os.fsencode(path), _d(v.view(np.float64)), v.size, C.byref(err)), err)


def load_vector(path):
    """load_vector (serialize.hpp:350-353)."""
    err = _Err()
    n = C.c_int64(0)
    _check(lib().h2g_vector_load(os.fsencode(path), None, C.byref(n), C.byref(err)), err)
    v = np.zeros(n.value, np.complex128)
    _check(lib().h2g_vector_load(os.fsencode(path), _d(v.view(np.float64)), C.byref(n), C.byref(err)), err)
    return v


_STEP_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_int32)
_MERGE_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class _Hooks(C.Structure):
    _fields_ = [("user", C.c_void_p), ("after_basis_update", _STEP_CB), ("after_projection", _STEP_CB), ("after_elimination", _STEP_CB),
                ("after_merge", _MERGE_CB)]


class FactorState:
    """What a FactorizeHooks callback sees (FactorState, factorization.hpp:115-251);
    valid only inside the callback."""

    def __init__(self, ptr):
        self.p = ptr

    def info(self):
        out = np.zeros(3, np.int64)
        lib().h2g_state_info(self.p, _i64(out))
        return dict(level=int(out[0]), active_len=int(out[1]), n=int(out[2]))

    def cluster(self, cid):
        out = np.zeros(5, np.int64)
        err = _Err()
        if lib().h2g_state_cluster(self.p, cid, _i64(out)):
            lib().h2g_last_error(C.byref(err))
            _raise(err)
        return dict(pos=int(out[0]), bsize=int(out[1]), rank=int(out[2]), rotated=bool(out[3]), eliminated=int(out[4]))

    def qtilde(self, cid):
        b = self.cluster(cid)["bsize"]
        Q = np.zeros((b, b), np.complex128, order="F")
        err = _Err()
        if lib().h2g_state_qtilde(self.p, cid, Q.ctypes.data_as(_D)):
            lib().h2g_last_error(C.byref(err))
            _raise(err)
        return Q

    def shadow(self):
        """FactorState::shadow() (factorization.hpp:240-245) of the device state."""
        n = self.info()["n"]
        Z = np.zeros((n, n), np.complex128, order="F")
        err = _Err()
        if lib().h2g_state_shadow(self.p, Z.ctypes.data_as(_D)):
            lib().h2g_last_error(C.byref(err))
            _raise(err)
        return Z

    def perm(self):
        n = C.c_int64(0)
        lib().h2g_state_perm(self.p, None, C.byref(n))
        out = np.zeros(n.value, np.int64)
        lib().h2g_state_perm(self.p, _i64(out), C.byref(n))
        return out


def factorize_hooked(A, eps_fill_in, after_basis_update=None, after_projection=None, after_elimination=None, after_merge=None,
                     stop_level_override=None):
    """factorize(A, eps, stop, hooks) (factorization.hpp:588-601): the GPU path in
    debug mode (reference order one cluster at a time, synchronised at every
    step); each callback gets (FactorState, cluster heap id) or (FactorState,).
    Exceptions raised inside callbacks are re-raised after the factorization."""
    errors = []

    def wrap_step(f):
        def cb(user, st, cl):
            if f is None or errors:
                return
            try:
                f(FactorState(st), int(cl))
            except BaseException as e:  # noqa: BLE001 - re-raised below
                errors.append(e)
        return _STEP_CB(cb)

    def wrap_merge(f):
        def cb(user, st):
            if f is None or errors:
                return
            try:
                f(FactorState(st))
            except BaseException as e:  # noqa: BLE001
                errors.append(e)
        return _MERGE_CB(cb)

    hk = _Hooks(None, wrap_step(after_basis_update), wrap_step(after_projection), wrap_step(after_elimination), wrap_merge(after_merge))
    err = _Err()
    h = _P()
    stop = -1 if stop_level_override is None else int(stop_level_override)
    rc = lib().h2g_factorize_hooked(A.ctx.h, A.h, float(eps_fill_in), stop, C.cast(C.pointer(hk), C.c_void_p), C.byref(h), C.byref(err))
    if errors:
        if rc == 0:
            FactorChain(h, A)  # released
        raise errors[0]
    _check(rc, err)
    return FactorChain(h, A)


# ---- multi-GPU subtree partition (h2g_factorize_dist) ---------------------
_XCHG_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_int32)


class _Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("exchange", _XCHG_CB), ("user", C.c_void_p)]


class _RawBuffer:
    """A (device or host) pointer as an array-interface object torch can wrap
    without a copy."""

    def __init__(self, ptr, nbytes, device):
        iface = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False), "version": 2}
        if device:
            self.__cuda_array_interface__ = iface
        else:
            self.__array_interface__ = iface


def torch_exchange(group=None, device_buffers=True, errors=None):
    """The `exchange` callback of h2g_dist over torch.distributed: part r of the
    buffer is broadcast from rank r (an all-gather with per-rank sizes). With
    the NCCL backend the parts move GPU to GPU over NVLink; with gloo (tests)
    they are staged through host memory. Returns a Python callable
    (buf_ptr, offsets, nranks) -> 0 / 1."""
    import torch
    import torch.distributed as dist

    def run(buf, offsets, nranks):
        try:
            offs = [int(offsets[i]) for i in range(nranks + 1)]
            me = dist.get_rank(group)
            if dist.get_world_size(group) != nranks:
                raise InvalidInputError(f"exchange: process group has {dist.get_world_size(group)} ranks, the factorization {nranks}")
            if device_buffers:
                t = torch.as_tensor(_RawBuffer(buf, offs[-1], True), device="cuda")
            else:
                t = torch.from_numpy(np.asarray(_RawBuffer(buf, offs[-1], False)))
            direct = dist.get_backend(group) == "nccl" or not device_buffers
            for r in range(nranks):
                part = t[offs[r]:offs[r + 1]]
                if part.numel() == 0:
                    continue
                src = dist.get_global_rank(group, r) if group is not None else r
                if direct:
                    dist.broadcast(part, src=src, group=group)
                else:
                    h = part.cpu() if r == me else torch.empty(part.numel(), dtype=torch.uint8)
                    dist.broadcast(h, src=src, group=group)
                    if r != me:
                        part.copy_(h)
            if device_buffers:
                torch.cuda.synchronize()
            return 0
        except BaseException as e:  # noqa: BLE001 - reported to the C side as a failure, re-raised by factorize_dist
            if errors is not None:
                errors.append(e)
            return 1

    return run


def factorize_dist(A, eps_fill_in, stop_level_override=None, group=None, rank=None, nranks=None, exchange=None):
    """The north_star's multi-GPU factorization (h2g_factorize_dist): every
    rank holds the same H2Matrix on its own GPU; the level-3 subtrees are dealt
    to the ranks, each rank eliminates the interior clusters of its subtrees,
    the ranks exchange the results at every level's interior / boundary border
    and run the boundary clusters replicated. Every rank returns the complete
    FactorChain (bitwise the single-GPU factorization with schedule="subtree").
    Default: rank / nranks / exchange from torch.distributed (`group`)."""
    errors = []
    if exchange is None:
        import torch.distributed as dist

        if rank is None:
            rank = dist.get_rank(group)
        if nranks is None:
            nranks = dist.get_world_size(group)
        exchange = torch_exchange(group, True, errors) if nranks > 1 else None

    def cb(user, buf, offsets, n):
        return int(exchange(buf, offsets, n))

    ccb = _XCHG_CB(cb) if exchange is not None else _XCHG_CB()
    d = _Dist(int(rank), int(nranks), ccb, None)
    err = _Err()
    h = _P()
    stop = -1 if stop_level_override is None else int(stop_level_override)
    rc = lib().h2g_factorize_dist(A.ctx.h, A.h, float(eps_fill_in), stop, C.byref(d), C.byref(h), C.byref(err))
    if errors:
        raise errors[0]
    _check(rc, err)
    return FactorChain(h, A)


def partition_plan(arrays, level, stop_level_override=None):
    """Host-only view of one level's subtree partition (h2g_partition_plan):
    dict(nl, batches, batch_of, part_batch, dense_part, fill_part)."""
    keep = []
    d = _desc_from_arrays(arrays, keep)
    err = _Err()
    counts = np.zeros(4, np.int64)
    stop = -1 if stop_level_override is None else int(stop_level_override)
    _check(lib().h2g_partition_plan(C.byref(d), stop, int(level), _i64(counts), None, None, None, None, None, None, C.byref(err)), err)
    nl, nbat, nd, nf = (int(v) for v in counts)
    batch_of = np.zeros(max(nl, 1), np.int32)
    part_batch = np.zeros(9, np.int32)
    dense_part = np.zeros(max(nd, 1), np.int32)
    fill_part = np.zeros(max(nf, 1), np.int32)
    dense_rc = np.zeros((max(nd, 1), 2), np.int32)
    fill_rc = np.zeros((max(nf, 1), 2), np.int32)
    _check(lib().h2g_partition_plan(C.byref(d), stop, int(level), _i64(counts), _i32(batch_of), _i32(part_batch), _i32(dense_part), _i32(fill_part),
                                    _i32(dense_rc), _i32(fill_rc), C.byref(err)), err)
    return dict(nl=nl, batches=nbat, batch_of=batch_of[:nl], part_batch=part_batch, dense_part=dense_part[:nd], fill_part=fill_part[:nf],
                dense_rc=dense_rc[:nd], fill_rc=fill_rc[:nf])


def factorize(A, eps_fill_in, stop_level_override=None, schedule="reference"):
    """factorize(A, eps_fill_in, stop_level_override) on the GPU."""
    err = _Err()
    h = _P()
    stop = -1 if stop_level_override is None else int(stop_level_override)
    if schedule not in SCHEDULES:
        raise InvalidInputError(f"unknown schedule {schedule!r}")
    _check(lib().h2g_factorize(A.ctx.h, A.h, float(eps_fill_in), stop, SCHEDULES[schedule], C.byref(h), C.byref(err)), err)
    return FactorChain(h, A)


def solve(chain, b):
    return chain.solve(b)


def apply_inverse(chain, b):
    return chain.apply_inverse(b)


def forward_substitute(chain, b):
    return chain.forward(b)


def backward_substitute(chain, y):
    return chain.backward(y)


def solve_in_place(chain, b):
    """Overwrites the 1-D complex128 array b with the solution."""
    if b.dtype != np.complex128 or not b.flags.c_contiguous:
        raise InvalidInputError("solve_in_place: b must be a contiguous complex128 array")
    b[...] = chain.solve(b)
    return b


def random_rhs(n, seed=1234):
    """mt19937_64 + std::normal_distribution complex vector (original order)."""
    out = np.zeros(n, np.complex128)
    lib().h2g_random_rhs(n, seed, _d(out.view(np.float64)))
    return out
