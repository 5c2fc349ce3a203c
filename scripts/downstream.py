#!/usr/bin/env python3
"""Downstream GNN check on the Reddit-shaped graph (north_star: "Downstream GCN/GraphSage
logits run with random-init weights, and argmax agreement against the oracle is reported").

For each model (GCN sum, GraphSage mean; 2 layers, hidden 128, 41 classes -- Table model
L1218-1227 / Table dataset) and each (strategy, s): GPU logits (sampled SpMM kernels
+ fp32 GEMM, TF32 off) vs oracle logits (fp64 GEMM + C oracle SpMM): argmax agreement, max
|error| / max|logit|, and GPU inference time (CUDA events; exact SpMM = Bucket with s >= max
degree, the paper's Fig. cs_e2e analogue).  Prints one JSON line per case."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import oracle.gnn as ognn  # noqa: E402
import synth  # noqa: E402
from paper_2104_10716_b200 import gnn  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
    dims = {"reddit": [602, 128, 41], "pubmed": [500, 32, 3], "arxiv": [128, 256, 256, 40],
            "proteins": [8, 256, 256, 112]}[name]
    dev = torch.device("cuda:0")
    rowptr, colind = synth.graph(name)
    n = len(rowptr) - 1
    d = np.diff(rowptr).astype(np.float64)
    # GCN values: symmetric normalisation 1/sqrt(d_i d_j) computed once on the host (the
    # caller's A.data; the kernel multiplies by whatever val holds)
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    val = (1.0 / np.sqrt(np.maximum(d[rows], 1) * np.maximum(d[colind], 1))).astype(np.float32)
    F0 = dims[0]
    ld0 = (F0 + 3) // 4 * 4
    X = synth.dense(n, F0, synth.seeds(name)[1], ld=ld0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    rp, ci, va, Xd = t(rowptr), t(colind), t(val), t(X)
    dmax = int(d.max())
    for model in ("sage", "gcn"):
        layers = gnn.init_weights(model, dims, seed=7)
        for strat, s in [(1, 16), (2, 16), (1, 32), (2, 32), (2, 64), (2, 256), (1, dmax)]:
            v = va if model == "gcn" else None
            for _ in range(2):
                g = gnn.forward(model, rp, ci, v, Xd, layers, s, strat)
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g = gnn.forward(model, rp, ci, v, Xd, layers, s, strat)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            g = g.cpu().numpy()
            t0 = time.perf_counter()
            o = ognn.forward(model, rowptr, colind, val if model == "gcn" else None, X, layers, s, strat)
            t_or = time.perf_counter() - t0
            agree = float(np.mean(gnn.argmax_lowest(g) == gnn.argmax_lowest(o)))
            err = float(np.max(np.abs(g - o)) / max(1e-30, np.max(np.abs(o))))
            print(json.dumps({"graph": name, "model": model, "strategy": "bucket" if strat == 1 else "fastrand",
                              "s": s, "exact": s >= dmax, "argmax_agreement": agree,
                              "max_abs_err_over_max_logit": err, "gpu_forward_ms": round(float(np.median(ts)), 3),
                              "oracle_forward_s": round(t_or, 2), "oracle_threads": oracle.max_threads()}),
                  flush=True)


if __name__ == "__main__":
    main()
