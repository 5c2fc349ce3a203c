#!/usr/bin/env python3
"""End-to-end GNN inference timing on the Reddit-shaped graph (the paper's
Fig. cs_e2e analogue: ~10x end-to-end at S=64 over cuSPARSE on V100).

2-layer GraphSage-mean and GCN (602 -> 128 -> 41, seeded random weights, fp32 GEMMs with TF32
off) -- the whole forward (GEMMs, aggregations, bias, ReLU) timed with CUDA events, L2 flushed
before each, median of 7:
  * ours: the sampled SpMM through the library's plan (gnn.forward with a workspace: the slab
    path where es_spmm_workspace_bytes asks for it, one sampling per forward, later layers
    reuse the slots), for each (strategy, s);
  * cusparse_exact: the same network with EXACT aggregation by torch.sparse (cuSPARSE CSR SpMM;
    MEAN = sum / d_i) -- the paper's baseline;
Prints one JSON line per case with the speedup over cusparse_exact.  Timing only (the parity
of these logits against the oracle is scripts/downstream.py)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2104_10716_b200 as es  # noqa: E402
from paper_2104_10716_b200 import gnn  # noqa: E402


def cusparse_forward(model, A, deg, X, layers):
    h = X
    for li, w in enumerate(layers):
        W = torch.from_numpy(w["W"]).to(X.device)
        b = torch.from_numpy(w["b"]).to(X.device)
        hv = h[:, :W.shape[0]].contiguous()
        if model == "gcn":
            out = torch.sparse.mm(A, hv @ W) + b
        else:
            Wn = torch.from_numpy(w["W_neigh"]).to(X.device)
            agg = torch.sparse.mm(A, hv) / deg
            out = hv @ W + agg @ Wn + b
        h = torch.relu(out) if li + 1 < len(layers) else out
    return h


def timed(fn, flush, reps=7):
    ts = []
    for i in range(2 + reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    name = "reddit"
    dims = [602, 128, 41]
    dev = torch.device("cuda:0")
    torch.backends.cuda.matmul.allow_tf32 = False
    rowptr, colind = synth.graph(name)
    n = len(rowptr) - 1
    d = np.diff(rowptr).astype(np.float64)
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    val_gcn = (1.0 / np.sqrt(np.maximum(d[rows], 1) * np.maximum(d[colind], 1))).astype(np.float32)
    X = synth.dense(n, 602, synth.seeds(name)[1], ld=608)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    rp, ci, Xd = t(rowptr), t(colind), t(X)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    deg = t(np.maximum(d, 1).astype(np.float32))[:, None]
    dmax = int(d.max())
    for model in ("sage", "gcn"):
        layers = gnn.init_weights(model, dims, seed=7)
        v = t(val_gcn) if model == "gcn" else None
        A = torch.sparse_csr_tensor(rp, ci.to(torch.int64), v if v is not None else torch.ones(len(colind), device=dev),
                                    size=(n, n))
        ms_cu = timed(lambda: cusparse_forward(model, A, deg, Xd[:, :602], layers), flush)
        print(json.dumps({"graph": name, "model": model, "variant": "cusparse_exact", "ms": round(ms_cu, 3)}),
              flush=True)
        for strat, s in [(1, 16), (2, 16), (1, 64), (2, 64), (2, 256), (1, dmax)]:
            ws = es.es_spmm_workspace(n, n, len(colind), 602, 608, s, v is not None, device=dev)
            ms = timed(lambda: gnn.forward(model, rp, ci, v, Xd, layers, s, strat, workspace=ws), flush)
            print(json.dumps({"graph": name, "model": model, "variant": "ours",
                              "strategy": "bucket" if strat == 1 else "fastrand", "s": s, "exact": s >= dmax,
                              "slab_path": ws is not None, "ms": round(ms, 3),
                              "speedup_vs_cusparse_exact": round(ms_cu / ms, 2)}), flush=True)


if __name__ == "__main__":
    main()
