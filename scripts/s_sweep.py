#!/usr/bin/env python3
"""The BASELINE.json metric "vs s": sampled-SpMM GFLOP/s, algorithmic GB/s and roofline fraction
for s in {16..512} x {Bucket, FastRand} on the dataset-shaped graphs (1 GPU, L2 flushed before
every call, CUDA events, median of 5), through the library's plan: es_spmm_run_ex with the
workspace es_spmm_workspace_bytes asks for (the slab path) where it asks, else the fused kernel
(`--kernel fused` as the first argument forces the fused kernel everywhere).  Prints one JSON line per point."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2104_10716_b200 as es  # noqa: E402
from bench import byte_model, l2_peak, ldb_for, measured_peaks  # noqa: E402

L2_BYTES = 126 << 20                # the B200 L2

CASES = [("pubmed", 16, 0), ("arxiv", 128, 0), ("proteins", 128, 0), ("reddit", 128, 1), ("reddit", 602, 1)]


def main():
    dev = torch.device("cuda:0")
    hbm, _ = measured_peaks()
    l2, _ = l2_peak()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    args = sys.argv[1:]
    kernel = None
    if args[:1] == ["--kernel"]:
        kernel, args = args[1], args[2:]
    only = args or None
    for name, F, red in CASES:
        if only and name not in only:
            continue
        rowptr, colind = synth.graph(name)
        n = len(rowptr) - 1
        d = np.diff(rowptr)
        ldb = ldb_for(F)
        B = torch.from_numpy(synth.dense(n, F, synth.seeds(name)[1], ld=ldb)).to(dev)
        rp, ci = torch.from_numpy(rowptr).to(dev), torch.from_numpy(colind).to(dev)
        va = torch.ones(len(colind), device=dev)
        C = torch.empty((n, ldb), device=dev)
        for s in (16, 32, 64, 128, 256, 512):
            K = int(np.minimum(d, s).sum())
            ws = (None if kernel == "fused" else es.es_spmm_workspace(n, n, len(colind), F, ldb, s, True, device=dev))
            for strat in (1, 2):
                ts = []
                lc0 = es.es_launch_count()
                for i in range(7):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    if ws is not None:
                        es.es_spmm_run_ex(rp, ci, va, B, s, strat, 0, red, F=F, C=C, workspace=ws)
                    else:
                        es.es_spmm_run(rp, ci, va, B, s, strat, 0, red, F=F, C=C)
                    e1.record()
                    torch.cuda.synchronize()
                    if i >= 2:
                        ts.append(e0.elapsed_time(e1))
                ms = float(np.median(ts))
                per_call = (es.es_launch_count() - lc0) // 7
                gbs = byte_model(K, n, F) / (ms / 1e3) / 1e9
                # the ceiling that binds (as bench.py without a traffic record): L2 when the gathered
                # operand is L2-resident -- B itself, or on the slab path its widest slab (<= 512 B of
                # each row, within the 126 MB L2)
                resident = (n * min(ldb * 4, 512) if ws is not None else n * ldb * 4) <= L2_BYTES
                # a non-resident B whose gathers still run above the HBM copy rate is being served by
                # L2 (hot rows re-gathered): HBM cannot be the ceiling that binds there
                bound, peak = ("l2", l2) if (l2 and (resident or gbs > hbm)) else ("hbm", hbm)
                print(json.dumps({"graph": name, "F": F, "s": s, "strategy": "bucket" if strat == 1 else "fastrand",
                                  "reduce": "mean" if red else "sum", "K": K, "rate": round(K / d.sum(), 4),
                                  "ms": round(ms, 4), "GFLOPs": round(2 * F * K / (ms / 1e3) / 1e9, 1),
                                  "model_GBs": round(gbs, 1), "bound": bound, "frac": round(gbs / peak, 3),
                                  "step_incl_sampling": True,
                                  "sampled_edges_per_s": round(K / (ms / 1e3)),
                                  "plan": "slab path (spmm_slab_flow x %d + sampling)" % (per_call - 4)
                                  if ws is not None else es.es_spmm_plan(F, ldb, ldb, B, C, s=s, n_rows=n,
                                                                          nnz=len(colind))}), flush=True)


if __name__ == "__main__":
    main()
