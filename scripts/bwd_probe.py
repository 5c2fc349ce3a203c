#!/usr/bin/env python3
"""Probe (tuning evidence only): backward dB = A_s^T dC on the Reddit-shaped graph -- fused
(es_spmm_backward_ex, one launch, reductions into the full-width dB) vs the feature-sliced
backward (workspace; reuse_sampled: the forward's slots), L2 flushed, median of 6."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2104_10716_b200 as es  # noqa: E402
from bench import ldb_for  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "reddit"
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 602
    s = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    ldb = ldb_for(F)
    dev = torch.device("cuda:0")
    rowptr, colind = synth.graph(cfg)
    n = len(rowptr) - 1
    K = int(np.minimum(np.diff(rowptr), s).sum())
    rp = torch.from_numpy(rowptr).to(dev)
    ci = torch.from_numpy(colind).to(dev)
    va = torch.ones(len(colind), dtype=torch.float32, device=dev)
    dC = torch.from_numpy(synth.dense(n, F, 77, ld=ldb)).to(dev)
    dB = torch.zeros((n, ldb), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ws = es.es_spmm_workspace(n, n, len(colind), F, ldb, s, True, device=dev, kernel="slab")
    B = torch.from_numpy(synth.dense(n, F, 5, ld=ldb)).to(dev)
    es.es_spmm_run_ex(rp, ci, va, B, s, 2, 0, 1, F=F, workspace=ws, kernel="slab")   # forward: samples into ws

    def timed(fn, reps=6):
        ts = []
        for i in range(2 + reps):
            dB.zero_()
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    res = {}
    for name, kw in [("fused", {}), ("slab", {"workspace": ws}), ("slab_reuse", {"workspace": ws, "reuse_sampled": True})]:
        ms = timed(lambda: es.es_spmm_backward_ex(rp, ci, va, dC, n, s, 2, 0, 1, F=F, dB=dB, **kw))
        res[name] = dB[:, :F].clone()
        print(json.dumps({"variant": name, "ms": round(ms, 3), "GBps_red": round(4 * F * K / ms / 1e6, 1),
                          "max_rel_vs_fused": None if name == "fused" else float(
                              ((res[name] - res["fused"]).abs() / res["fused"].abs().clamp_min(1e-3)).max())}),
              flush=True)


if __name__ == "__main__":
    main()
