"""CPU ORACLE for ES-SpMM (arXiv 2104.10716).  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_2104_10716_b200``) never does, and this package never imports the product.

Two independent implementations live here:

* ``es_oracle.c`` (loaded through ctypes): the sampled SpMM of Alg. 1
  with Bucket (L1042-1047) and FastRand Eq. 2 (L1064-1067, P'=577 L1058), fp64
  accumulation in slot order rounded once to fp32, mean by k_i (L1570-1575, reading R5);
  and its backward w.r.t. B, dB = A_s^T dC over the same slots (NEXT-2, §6.2).
* ``brute``: a pure-Python/numpy brute force for tiny graphs -- builds the dense
  sampled adjacency A_s (fp64) slot by slot with Python integers and multiplies it by B.

Every public function is pinned by ``tests/test_oracle_pins.py``; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

BUCKET, FASTRAND = 1, 2
SUM, MEAN = 0, 1
PRIME = 577  # P'

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libesoracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle (plain gcc -O2, no fast-math)."""
    src = os.path.join(_HERE, "es_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fno-fast-math", "-ffp-contract=off", "-shared", "-fPIC",
                               src, "-o", _LIB_PATH])
    return _LIB_PATH


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        i64, i32, u64, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p
        lib.oracle_hash.restype = u64
        lib.oracle_hash.argtypes = [u64]
        lib.oracle_offset.restype = i64
        lib.oracle_offset.argtypes = [u64, i64, i64]
        lib.oracle_position.restype = i64
        lib.oracle_position.argtypes = [i32, i64, i64, i64]
        lib.oracle_position_p.restype = i64
        lib.oracle_position_p.argtypes = [i32, i64, i64, i64, i64]
        lib.oracle_rate.restype = ctypes.c_double
        lib.oracle_rate.argtypes = [i64, vp, i64]
        lib.oracle_sample.restype = None
        lib.oracle_sample.argtypes = [i64, vp, vp, vp, i64, i32, u64, i64, i64, vp, vp, vp, vp]
        lib.oracle_spmm.restype = ctypes.c_int
        lib.oracle_spmm.argtypes = [i64, vp, vp, vp, vp, i64, i64, i64, i32, u64, i32, i64, i64, i32,
                                    vp, i64, vp, i64]
        lib.oracle_spmm_backward.restype = ctypes.c_int
        lib.oracle_spmm_backward.argtypes = [i64, vp, vp, vp, vp, i64, i64, i64, i32, u64, i32, i64,
                                             i64, i32, i64, vp, i64]
        lib.oracle_max_threads.restype = ctypes.c_int
        lib.oracle_max_threads.argtypes = []
        lib.oracle_spmm_f32.restype = ctypes.c_int
        lib.oracle_spmm_f32.argtypes = [i64, vp, vp, vp, vp, i64, i64, i64, i32, u64, i32, vp, i64, vp, i64]
        lib.oracle_set_threads.restype = None
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _csr(rowptr, colind, val):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colind = np.ascontiguousarray(colind, dtype=np.int32)
    val = None if val is None else np.ascontiguousarray(val, dtype=np.float32)
    return rowptr, colind, val


def mix64(x: int) -> int:
    return int(_L().oracle_hash(x & (2**64 - 1)))


def offset(seed: int, row: int, d: int) -> int:
    """Seeded FastRand rotation of row ``row`` (reading R6); 0 when seed == 0."""
    return int(_L().oracle_offset(seed & (2**64 - 1), row, d))


def position(strategy: int, j: int, d: int, off: int = 0, prime: int = PRIME) -> int:
    """Eq. 2 (FastRand) / j (Bucket); prime = P' (577, L1058)."""
    if prime == PRIME:
        return int(_L().oracle_position(strategy, j, d, off))
    return int(_L().oracle_position_p(strategy, j, d, off, prime))


def rate(rowptr, s: int) -> float:
    """sum_i min(d_i, s) / nnz."""
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    return float(_L().oracle_rate(len(rowptr) - 1, rowptr.ctypes.data, s))


def sample(rowptr, colind, val, s: int, strategy: int, seed: int = 0, row_base: int = 0,
           prime: int = PRIME):
    """Materialised sampled CSR in slot order: (s_rowptr, s_colind, s_val, s_pos)."""
    rowptr, colind, val = _csr(rowptr, colind, val)
    n = len(rowptr) - 1
    s_rowptr = np.empty(n + 1, dtype=np.int64)
    L = _L()
    L.oracle_sample(n, rowptr.ctypes.data, colind.ctypes.data, _p(val), s, strategy,
                    seed & (2**64 - 1), row_base, prime, s_rowptr.ctypes.data, None, None, None)
    K = int(s_rowptr[-1])
    s_colind = np.empty(K, dtype=np.int32)
    s_val = np.empty(K, dtype=np.float32)
    s_pos = np.empty(K, dtype=np.int64)
    L.oracle_sample(n, rowptr.ctypes.data, colind.ctypes.data, _p(val), s, strategy,
                    seed & (2**64 - 1), row_base, prime, s_rowptr.ctypes.data, s_colind.ctypes.data,
                    s_val.ctypes.data, s_pos.ctypes.data)
    return s_rowptr, s_colind, s_val, s_pos


def spmm(rowptr, colind, val, B, s: int, strategy: int, seed: int = 0, reduce: int = SUM,
         F: int | None = None, rows=None, row_base: int = 0, prime: int = PRIME,
         mean_by_degree: bool = False) -> np.ndarray:
    """Sampled SpMM C (fp32).  B is (n_cols, ldb) fp32; F defaults to ldb.
    ``rows``: optional int64 row list -> returns only those rows (len(rows) x F).
    ``prime`` / ``mean_by_degree``: NEXT-4 variants (P' override; MEAN divides by d_i)."""
    rowptr, colind, val = _csr(rowptr, colind, val)
    B = np.ascontiguousarray(B, dtype=np.float32)
    ldb = B.shape[1]
    F = ldb if F is None else F
    n = len(rowptr) - 1
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        n_out = len(rows)
    else:
        n_out = n
    C = np.empty((n_out, F), dtype=np.float32)
    if n_out == 0 or F == 0:
        return C
    rc = _L().oracle_spmm(n, rowptr.ctypes.data, colind.ctypes.data, _p(val), B.ctypes.data, F,
                          ldb, s, strategy, seed & (2**64 - 1), reduce, row_base, prime,
                          int(mean_by_degree), _p(rows), n_out, C.ctypes.data, F)
    if rc != 0:
        raise MemoryError("oracle_spmm: allocation failed")
    return C


def spmm_backward(rowptr, colind, val, dC, n_cols: int, s: int, strategy: int, seed: int = 0,
                  reduce: int = SUM, F: int | None = None, row_base: int = 0, prime: int = PRIME,
                  mean_by_degree: bool = False) -> np.ndarray:
    """dB = A_s^T dC over the forward's sampled slots (MEAN: rows of A_s scaled by 1/k_i);
    returns a fresh (n_cols, F) fp32 array."""
    rowptr, colind, val = _csr(rowptr, colind, val)
    dC = np.ascontiguousarray(dC, dtype=np.float32)
    F = dC.shape[1] if F is None else F
    dB = np.zeros((n_cols, F), dtype=np.float32)
    if n_cols == 0 or F == 0:
        return dB
    rc = _L().oracle_spmm_backward(len(rowptr) - 1, rowptr.ctypes.data, colind.ctypes.data, _p(val),
                                   dC.ctypes.data, F, dC.shape[1], s, strategy, seed & (2**64 - 1),
                                   reduce, row_base, prime, int(mean_by_degree), n_cols,
                                   dB.ctypes.data, F)
    if rc != 0:
        raise MemoryError("oracle_spmm_backward: allocation failed")
    return dB


def spmm_f32(rowptr, colind, val, B, s: int, strategy: int, seed: int = 0, reduce: int = SUM,
             F: int | None = None, rows=None) -> np.ndarray:
    """TIMING MODE ONLY (bench.py's CPU baseline): the sampled SpMM with fp32 FMA accumulation in
    slot order (a straightforward CPU port of Alg. 1).  Parity uses spmm (fp64)."""
    rowptr, colind, val = _csr(rowptr, colind, val)
    B = np.ascontiguousarray(B, dtype=np.float32)
    ldb = B.shape[1]
    F = ldb if F is None else F
    n = len(rowptr) - 1
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
    n_out = n if rows is None else len(rows)
    C = np.empty((n_out, F), dtype=np.float32)
    if n_out == 0 or F == 0:
        return C
    rc = _L().oracle_spmm_f32(n, rowptr.ctypes.data, colind.ctypes.data, _p(val), B.ctypes.data, F, ldb, s,
                              strategy, seed & (2**64 - 1), reduce, _p(rows), n_out, C.ctypes.data, F)
    if rc != 0:
        raise MemoryError("oracle_spmm_f32: allocation failed")
    return C


def set_threads(n: int) -> None:
    _L().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(_L().oracle_max_threads())


from . import brute  # noqa: E402,F401
