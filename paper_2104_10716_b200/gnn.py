"""GNN inference on top of the sampled SpMM (the downstream check of north_star).

Eq. 1: H^{l+1} = sigma(A H^l W^l).  GEMMs use torch.matmul with TF32
disabled (fp32, cuBLAS -- a plain library GEMM); every aggregation A.(.) is the sampled
SpMM of this package (es_spmm_run).  Models follow Table model (L1206-1234): 2 layers on
Pubmed/Reddit (hidden 32 / 128), 3 layers on Arxiv/Proteins (hidden 256).

* GCN (sum aggregation, L588-599): h' = sigma(A_s (h W)) -- GEMM first, then SpMM at the
  narrower width (Eq. 1 grouping); A's values carry the normalisation (caller's val).
* GraphSage-mean (L1256): h' = sigma(h W_self + mean_s(h) W_neigh) -- mean over the
  sampled neighbours at the input width, divided by k_i inside the kernel (L1570-1575).
Weights are seeded random (no trained weights exist here).

With a `workspace` (es_spmm_workspace(...) sized for the widest aggregation, has_val as the
model's A), every aggregation the library's plan sends to the slab path runs there, and all
but the first reuse the slots the first one sampled (reuse_sampled): the layers aggregate over
one sampled graph, sampled once per forward.
"""
from __future__ import annotations

import numpy as np

from . import ES_REDUCE_MEAN, ES_REDUCE_SUM, es_spmm_run, es_spmm_run_ex, es_spmm_workspace_bytes


def init_weights(model: str, dims: list[int], seed: int = 0) -> list[dict]:
    """Seeded Glorot-uniform weights (numpy fp32), identical for the GPU and oracle paths."""
    rng = np.random.default_rng(seed)
    layers = []
    for fi, fo in zip(dims[:-1], dims[1:]):
        lim = np.sqrt(6.0 / (fi + fo))
        w = {"W": rng.uniform(-lim, lim, (fi, fo)).astype(np.float32)}
        if model == "sage":
            w["W_neigh"] = rng.uniform(-lim, lim, (fi, fo)).astype(np.float32)
        w["b"] = rng.uniform(-0.1, 0.1, fo).astype(np.float32)
        layers.append(w)
    return layers


def forward(model: str, rowptr, colind, val, X, layers, s: int, strategy: int, seed: int = 0,
            workspace=None):
    """Logits on the GPU.  rowptr/colind/val/X are CUDA tensors; returns an (N, classes) tensor.
    X may carry row padding (X.shape[1] >= the first layer's input width, e.g. ldb 604 for
    F = 602 so the aggregation gathers 16-B rows)."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    n_rows, nnz = rowptr.numel() - 1, colind.numel()
    sampled = [False]

    def aggregate(rp, ci, v, B, s_, strat, seed_, reduce, F=None):
        """The sampled SpMM through the library's plan (slab path + slot reuse with a workspace)."""
        F = B.shape[1] if F is None else F
        # the slab path runs (and leaves slots to reuse) only where the library asks for a
        # workspace AND B's rows are 16-B aligned; a reuse the library cannot honour is an error
        if (workspace is not None and B.data_ptr() % 16 == 0
                and es_spmm_workspace_bytes(n_rows, B.shape[0], nnz, F, B.shape[1], s_, v is not None) > 0):
            out = es_spmm_run_ex(rp, ci, v, B, s_, strat, seed_, reduce, F=F, workspace=workspace,
                                 reuse_sampled=sampled[0])
            sampled[0] = True
            return out
        return es_spmm_run(rp, ci, v, B, s_, strat, seed_, reduce, F=F)

    try:
        h = X
        n = len(layers)
        for li, w in enumerate(layers):
            W = torch.from_numpy(w["W"]).to(X.device)
            b = torch.from_numpy(w["b"]).to(X.device)
            fi = W.shape[0]
            hv = h[:, :fi]
            if model == "gcn":
                hw = (hv @ W).contiguous()
                out = aggregate(rowptr, colind, val, hw, s, strategy, seed, ES_REDUCE_SUM) + b
            else:
                Wn = torch.from_numpy(w["W_neigh"]).to(X.device)
                agg = aggregate(rowptr, colind, None, h.contiguous(), s, strategy, seed, ES_REDUCE_MEAN,
                                  F=fi)
                out = hv @ W + agg @ Wn + b
            h = torch.relu(out) if li + 1 < n else out
        return h
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def argmax_lowest(logits: np.ndarray) -> np.ndarray:
    """Argmax with ties broken toward the lowest index."""
    return np.argmax(logits, axis=1)   # numpy returns the first maximal index
