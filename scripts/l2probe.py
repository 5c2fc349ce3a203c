#!/usr/bin/env python3
"""Probe: gather throughput vs B footprint (how much of B is L2-resident).

Remaps the Reddit-shaped graph's columns to the first M nodes (colind % M) so the B rows
gathered span M * ldb * 4 bytes, and times the plan's kernel (and the LDG kernel).
Tuning/evidence only."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2104_10716_b200 as es  # noqa: E402
from bench import byte_model, ldb_for  # noqa: E402


def main():
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 602
    dev = torch.device("cuda:0")
    rowptr, colind = synth.graph("reddit")
    n = len(rowptr) - 1
    ldb = ldb_for(F)
    B = torch.from_numpy(synth.dense(n, F, 5, ld=ldb)).to(dev)
    rp = torch.from_numpy(rowptr).to(dev)
    va = torch.ones(len(colind), dtype=torch.float32, device=dev)
    C = torch.empty((n, ldb), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    K = int(np.minimum(np.diff(rowptr), 256).sum())
    ci_full = torch.from_numpy(colind).to(dev)
    for M in [2000, 10000, 20000, 40000, 80000, n]:
        ci = torch.remainder(ci_full, M).to(torch.int32)
        for kern in ["auto", "warp"]:
            os.environ.pop("ES_SPMM_KERNEL", None)
            if kern != "auto":
                os.environ["ES_SPMM_KERNEL"] = kern
            ts = []
            for i in range(6):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                es.es_spmm_run(rp, ci, va, B, 256, 2, 0, 1, F=F, C=C)
                e1.record()
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            print(json.dumps({"F": F, "M": M, "B_MB": round(M * ldb * 4 / 1e6, 1), "kernel": kern,
                              "plan": es.es_spmm_plan(F, ldb, ldb, B, C), "ms": round(ms, 3),
                              "gather_TBs": round(4 * F * K / (ms / 1e3) / 1e12, 2),
                              "model_TBs": round(byte_model(K, n, F) / (ms / 1e3) / 1e12, 2)}), flush=True)


if __name__ == "__main__":
    main()
