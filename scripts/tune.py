#!/usr/bin/env python3
"""In-process kernel-variant sweep (tuning only; the headline number comes from bench.py).

  python scripts/tune.py --config reddit --F 602 --variants "warp;tma:8:8;tma:8:4"
variant syntax: ENV=VAL,ENV=VAL  (ES_SPMM_* knobs; short keys: k=KERNEL st=STAGES r=ROWS_PER_WARP
m=MINB hot=HOT_DEG)
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2104_10716_b200 as es  # noqa: E402
from bench import byte_model, ldb_for, measured_peaks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--F", type=int, default=602)
    ap.add_argument("--s", type=int, default=256)
    ap.add_argument("--strategy", default="fastrand")
    ap.add_argument("--reduce", default="mean")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--variants", default="k=warp;k=tma,st=4")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--ldb", type=int, default=0, help="override the B row pitch (floats)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rowptr, colind = synth.graph(a.config)
    n = len(rowptr) - 1
    F, ldb = a.F, (a.ldb or ldb_for(a.F))
    B = synth.dense(n, F, synth.seeds(a.config)[1], ld=ldb)
    rp = torch.from_numpy(rowptr).to(dev)
    ci = torch.from_numpy(colind).to(dev)
    va = torch.ones(len(colind), dtype=torch.float32, device=dev)
    Bd = torch.from_numpy(B).to(dev)
    C = torch.empty((n, ldb), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    strat = 1 if a.strategy == "bucket" else 2
    red = 1 if a.reduce == "mean" else 0
    K = int(np.minimum(np.diff(rowptr), a.s).sum())
    peak, _ = measured_peaks()
    ref = None
    for v in a.variants.split(";"):
        short = {"k": "KERNEL", "st": "STAGES", "r": "ROWS_PER_WARP", "m": "MINB", "hot": "HOT_DEG"}
        for k in list(os.environ):
            if k.startswith("ES_SPMM_"):
                os.environ.pop(k)
        for kv in filter(None, v.split(",")):
            k, val = kv.split("=")
            os.environ["ES_SPMM_" + short.get(k, k)] = val
        plan = es.es_spmm_plan(F, ldb, ldb, Bd, C)
        ts = []
        for i in range(2 + a.steps):
            if not a.no_flush:
                flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            es.es_spmm_run(rp, ci, va, Bd, a.s, strat, 0, red, F=F, C=C)
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        out = C[:, :F].clone()
        same = None
        if ref is None:
            ref = out
        else:
            same = bool(torch.equal(ref, out)) or float((ref - out).abs().max())
        ms = float(np.median(ts))
        gbs = byte_model(K, n, F) / (ms / 1e3) / 1e9
        print(json.dumps({"variant": v, "plan": plan, "ms": round(ms, 3), "min_ms": round(min(ts), 3),
                          "GFLOPs": round(2 * F * K / (ms / 1e3) / 1e9, 1), "model_GBs": round(gbs, 1),
                          "frac": round(gbs / peak, 3), "same_as_first": same}), flush=True)


if __name__ == "__main__":
    main()
