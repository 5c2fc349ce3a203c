"""Shared parity bars of the GPU tests.

bound_ok: the order-independent bound of a sum of fp32 reductions, |g - o| <= (n_c + 2) u sum|terms|
(n_c = contributions to that element, u = 2^-24), computed from the oracle on |val|, |dC| -- used
wherever the GPU's addition order across rows is not fixed (the backward's vector reductions)."""
import numpy as np

import oracle

U = 2.0 ** -24


def bound_ok(g, rowptr, colind, val, dC, n_cols, s, strat, seed, reduce, prime=oracle.PRIME,
             mean_by_degree=False):
    kw = dict(seed=seed, reduce=reduce, prime=prime, mean_by_degree=mean_by_degree)
    o = oracle.spmm_backward(rowptr, colind, val, dC, n_cols, s, strat, **kw)
    mag = oracle.spmm_backward(rowptr, colind, None if val is None else np.abs(val), np.abs(dC), n_cols, s,
                               strat, **kw).astype(np.float64)
    _, sc, _, _ = oracle.sample(rowptr, colind, val, s, strat, seed, prime=prime)
    nc = np.bincount(sc, minlength=n_cols).astype(np.float64)[:, None]
    tol = (nc + 2) * U * mag + 1e-30
    err = np.abs(np.asarray(g, np.float64) - o)
    return bool(np.all(err <= tol)), float(np.max(err / np.maximum(mag, 1e-30)))
