"""Brute-force sampled SpMM for tiny graphs.  TEST INFRASTRUCTURE ONLY.

Builds the dense sampled adjacency A_s (fp64, n_rows x n_cols) slot by slot with plain
Python integers -- slot j of row i adds val[e] at (i, colind[e]), e = rowptr[i] + p_j,
duplicates adding up (reading R2) -- then C = A_s @ B in fp64 (numpy matmul), rounded once.
Independent of es_oracle.c (different route: dense matrix, Python big ints).

Cites: Alg. 1, Bucket L1042-1047, Eq. 2 L1064-1067 with P'=577 L1058,
mean normalisation L1570-1575 (reading R5: divide by k_i).
"""
from __future__ import annotations

import numpy as np

BUCKET, FASTRAND = 1, 2
SUM, MEAN = 0, 1
_M64 = (1 << 64) - 1


def _splitmix(x: int) -> int:
    x &= _M64
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & _M64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & _M64
    x ^= x >> 31
    return x


def positions(strategy: int, d: int, s: int, seed: int = 0, row: int = 0, prime: int = 577) -> list[int]:
    k = min(d, s)
    if strategy == BUCKET:
        return list(range(k))
    off = 0
    if seed and d:
        off = _splitmix(seed + 0x9E3779B97F4A7C15 * (row + 1)) % d
    return [(off + j * prime) % d for j in range(k)]


def sampled_dense(rowptr, colind, val, n_cols: int, s: int, strategy: int, seed: int = 0, prime: int = 577):
    n = len(rowptr) - 1
    A = np.zeros((n, n_cols), dtype=np.float64)
    k = np.zeros(n, dtype=np.int64)
    for i in range(n):
        lo, hi = int(rowptr[i]), int(rowptr[i + 1])
        ps = positions(strategy, hi - lo, s, seed, i, prime)
        k[i] = len(ps)
        for p in ps:
            e = lo + p
            A[i, int(colind[e])] += 1.0 if val is None else float(val[e])
    return A, k


def spmm(rowptr, colind, val, B, s: int, strategy: int, seed: int = 0, reduce: int = SUM,
         prime: int = 577, mean_by_degree: bool = False):
    B = np.asarray(B, dtype=np.float32)
    A, k = sampled_dense(rowptr, colind, val, B.shape[0], s, strategy, seed, prime)
    C = (A @ B.astype(np.float64)).astype(np.float32)
    if reduce == MEAN:
        div = np.diff(np.asarray(rowptr, np.int64)) if mean_by_degree else k
        dd = np.maximum(div, 1).astype(np.float32)[:, None]
        C = np.where(div[:, None] > 0, C / dd, np.float32(0.0)).astype(np.float32)
    return C


def spmm_backward(rowptr, colind, val, dC, n_cols: int, s: int, strategy: int, seed: int = 0,
                  reduce: int = SUM):
    """dB = A_s^T dC with the dense sampled matrix (rows scaled by 1/k_i for MEAN), fp64."""
    A, k = sampled_dense(rowptr, colind, val, n_cols, s, strategy, seed)
    if reduce == MEAN:
        A = A / np.maximum(k, 1)[:, None]
    return (A.T @ np.asarray(dC, dtype=np.float64)).astype(np.float32)
