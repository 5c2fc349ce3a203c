"""Seeded synthetic inputs for ES-SpMM (shared by the oracle tests, the CUDA tests and bench.py).

Holds none of the method's arithmetic: it produces CSR graphs (rowptr, colind, val)
and dense feature matrices B.  The recipe is stated in DESIGN.md ("Input recipe"):

* degree sequences integerised from the CCDF knots in ``degree_knots.json``
  (fitted by ``synth/fit_degrees.py`` to PAPER.md Table dataset L624-644 and
  Table sample_rate), node ids permuted by a seeded hash;
* columns drawn distinct per row with popularity proportional to degree, sorted
  ascending (libsynth.so, counter-based, thread-count independent);
* ``val`` = 1.0 (unweighted graphs) unless a test asks otherwise;
* B[j, c] = (mix64(seed_B + G*(j*F+c+1)) >> 40) * 2^-24 in [0, 1).
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynth.so")
_lib = None

GOLDEN = 0x9E3779B97F4A7C15
SEED_BASE = 2104_10716

# Workload configs (BASELINE.json "configs").
CONFIGS = {
    "pubmed":   dict(index=0, kind="fit", F=16, s=32),
    "arxiv":    dict(index=1, kind="fit", F=128, s=64),
    "proteins": dict(index=2, kind="fit", F=128, s=256),
    "reddit":   dict(index=3, kind="fit", F=602, s=256),
    "scaled":   dict(index=4, kind="pareto", F=256, s=128, n=10_000_000, mean=100.0,
                     alpha=1.5, cap=200_000),
}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", src, "-o", _LIB_PATH])
    return _LIB_PATH


def _get_lib():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.synth_columns.restype = ctypes.c_int
        lib.synth_columns.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
        lib.synth_dense.restype = None
        lib.synth_dense.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_uint64, ctypes.c_void_p]
        lib.synth_perm_keys.restype = None
        lib.synth_perm_keys.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p]
        lib.synth_mix64.restype = ctypes.c_uint64
        lib.synth_mix64.argtypes = [ctypes.c_uint64]
        _lib = lib
    return _lib


def seeds(name: str) -> tuple[int, int]:
    """(seed_graph, seed_B) for a named config (SURVEY.md 8(d) 'Values and RNG')."""
    sg = SEED_BASE + CONFIGS[name]["index"]
    return sg, sg ^ 0xB


# --------------------------------------------------------------------------- degrees
def _knots():
    with open(os.path.join(_HERE, "degree_knots.json")) as f:
        return json.load(f)["configs"]


def ccdf(name: str) -> np.ndarray:
    """Integer CCDF c[t-1] = #{i: d_i >= t}, t = 1..d_max, for a fitted config."""
    k = _knots()[name]
    knots = np.asarray(k["knots"], dtype=np.float64)
    logc = np.asarray(k["logc"], dtype=np.float64)
    dmax = int(k["dmax"])
    t = np.arange(1, dmax + 1, dtype=np.float64)
    c = np.rint(np.exp(np.interp(np.log(t), np.log(knots), logc))).astype(np.int64)
    c[0] = int(k["n"])
    c = np.minimum.accumulate(c)
    c[-1] = max(c[-1], 1)
    return np.minimum.accumulate(c)


def _pareto_degrees(n: int, mean: float, alpha: float, cap: int) -> np.ndarray:
    """Deterministic quantile sequence of a Pareto CCDF (t/dmin)^-alpha, capped."""
    q = (np.arange(n, dtype=np.float64) + 0.5) / n

    def seq(dmin):
        return np.minimum(np.floor(dmin * (1.0 - q) ** (-1.0 / alpha)), cap).astype(np.int64)

    lo, hi = 1.0, mean
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if seq(mid).mean() < mean:
            lo = mid
        else:
            hi = mid
    return seq(hi)


def degrees(name: str) -> np.ndarray:
    """Per-node degree (row nnz) in node-id order, seeded permutation applied."""
    cfg = CONFIGS[name]
    if cfg["kind"] == "fit":
        c = ccdf(name)
        counts = c - np.append(c[1:], 0)                 # #{d_i == t}
        d_sorted = np.repeat(np.arange(1, len(c) + 1, dtype=np.int64), counts)[::-1]
    else:
        d_sorted = _pareto_degrees(cfg["n"], cfg["mean"], cfg["alpha"], cfg["cap"])[::-1]
    n = len(d_sorted)
    keys = np.empty(n, dtype=np.uint64)
    _get_lib().synth_perm_keys(n, seeds(name)[0] ^ 0xD, keys.ctypes.data)
    perm = np.argsort(keys, kind="stable")
    d = np.empty(n, dtype=np.int64)
    d[perm] = d_sorted
    return d


# --------------------------------------------------------------------------- graphs
def columns(rowptr: np.ndarray, n_cols: int, weights: np.ndarray, seed: int) -> np.ndarray:
    """Distinct, ascending columns per row drawn with probability ~ weights (all >= 1)."""
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    cumw = np.ascontiguousarray(np.cumsum(np.asarray(weights, dtype=np.int64)), dtype=np.int64)
    assert len(cumw) == n_cols and (n_cols == 0 or cumw[0] >= 1)
    colind = np.empty(int(rowptr[-1]), dtype=np.int32)
    if n_cols == 0 or len(colind) == 0:
        return colind
    rc = _get_lib().synth_columns(len(rowptr) - 1, n_cols, rowptr.ctypes.data, cumw.ctypes.data,
                                  seed & (2**64 - 1), colind.ctypes.data)
    if rc != 0:
        raise ValueError(f"synth_columns failed ({rc}): a row asks for more columns than exist")
    return colind


def _cache_dir() -> str:
    d = os.environ.get("ES_SYNTH_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "es_synth"))
    os.makedirs(d, exist_ok=True)
    return d


def graph(name: str, cache: bool = True):
    """(rowptr int64[N+1], colind int32[nnz]) for a named config; square N x N.

    Cached as .npy keyed by name + seed (a speed-up only: the bytes are a pure
    function of the committed recipe)."""
    sg, _ = seeds(name)
    path = os.path.join(_cache_dir(), f"{name}_{sg}_v1")
    if cache and os.path.exists(path + "_colind.npy"):
        return np.load(path + "_rowptr.npy"), np.load(path + "_colind.npy", mmap_mode=None)
    d = degrees(name)
    rowptr = np.zeros(len(d) + 1, dtype=np.int64)
    np.cumsum(d, out=rowptr[1:])
    colind = columns(rowptr, len(d), np.maximum(d, 1), sg)
    if cache:
        # atomic publish (several ranks of one node may generate the same graph concurrently);
        # colind is published last because its presence marks the cache entry complete
        for suffix, arr in (("_rowptr.npy", rowptr), ("_colind.npy", colind)):
            tmp = f"{path}{suffix}.{os.getpid()}.tmp.npy"
            np.save(tmp, arr)
            os.replace(tmp, path + suffix)
    return rowptr, colind


def dense(n: int, f: int, seed: int, ld: int | None = None) -> np.ndarray:
    """n x ld float32 (row-major); columns >= f are zero padding."""
    ld = f if ld is None else ld
    assert ld >= f
    out = np.empty((n, ld), dtype=np.float32)
    if n and ld:
        _get_lib().synth_dense(n, f, ld, seed & (2**64 - 1), out.ctypes.data)
    return out


def mix64(x: int) -> int:
    return int(_get_lib().synth_mix64(x & (2**64 - 1)))


# --------------------------------------------------------------------------- small test graphs
def random_csr(n_rows: int, n_cols: int, seed: int, max_deg: int = 64,
               special: tuple = (), p_empty: float = 0.1, weighted: bool = True):
    """Ragged random CSR for parity tests: degrees ~ a heavy-ish tail in [0, max_deg],
    a fraction of empty rows, plus rows with the degrees listed in ``special``
    (e.g. 577, 1154 to hit FastRand duplicates).  Returns (rowptr, colind, val)."""
    rng = np.random.default_rng(seed)
    d = np.minimum((rng.pareto(1.2, n_rows) * 3).astype(np.int64), max_deg)
    d[rng.random(n_rows) < p_empty] = 0
    for k, sd in enumerate(special):
        if n_rows:
            d[(k * 7919) % n_rows] = sd
    d = np.minimum(d, n_cols)
    rowptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(d, out=rowptr[1:])
    w = rng.integers(1, 20, n_cols) if n_cols else np.zeros(0, np.int64)
    colind = columns(rowptr, n_cols, w, seed ^ 0x5EED)
    val = (rng.random(len(colind), dtype=np.float32) + 0.5).astype(np.float32) if weighted \
        else np.ones(len(colind), dtype=np.float32)
    return rowptr, colind, val
