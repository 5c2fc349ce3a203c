"""Oracle GNN forward (TEST INFRASTRUCTURE ONLY): fp64 numpy GEMMs + the C oracle's sampled
SpMM (oracle.spmm) for every aggregation.  Same model definitions as
paper_2104_10716_b200/gnn.py (Eq. 1; GraphSage mean L1256, normalisation
inside the aggregation L1570-1575).  Used to report argmax agreement of the GPU logits
(north_star: "argmax agreement against the oracle is reported")."""
from __future__ import annotations

import numpy as np

from . import MEAN, SUM, spmm


def forward(model: str, rowptr, colind, val, X, layers, s: int, strategy: int, seed: int = 0):
    h = np.asarray(X, dtype=np.float64)
    n = len(layers)
    for li, w in enumerate(layers):
        W = w["W"].astype(np.float64)
        b = w["b"].astype(np.float64)
        h = h[:, :W.shape[0]]
        if model == "gcn":
            hw = (h @ W).astype(np.float32)
            out = spmm(rowptr, colind, val, hw, s, strategy, seed=seed, reduce=SUM).astype(np.float64) + b
        else:
            agg = spmm(rowptr, colind, None, h.astype(np.float32), s, strategy, seed=seed,
                       reduce=MEAN).astype(np.float64)
            out = h @ W + agg @ w["W_neigh"].astype(np.float64) + b
        h = np.maximum(out, 0.0) if li + 1 < n else out
    return h
