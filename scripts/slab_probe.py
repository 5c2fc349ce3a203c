#!/usr/bin/env python3
"""Probe (tuning evidence only): the slab path (es_spmm_run_ex + workspace) vs the fused kernels.

  python scripts/slab_probe.py [config] [F]   # default reddit 602
Times each variant with the L2 flushed before every step (as bench.py), prints one JSON line per
variant with ms and the max |difference| to the fused kernel's C.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2104_10716_b200 as es  # noqa: E402

if os.environ.get("ES_LIB"):                 # A/B a library built with other compile-time knobs
    es.load_library(os.environ["ES_LIB"])
from bench import byte_model, ldb_for  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "reddit"
    F = int(sys.argv[2]) if len(sys.argv) > 2 else 602
    s = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    ldb = ldb_for(F)
    dev = torch.device("cuda:0")
    rowptr, colind = synth.graph(cfg)
    n = len(rowptr) - 1
    K = int(np.minimum(np.diff(rowptr), s).sum())
    Bd = torch.from_numpy(synth.dense(n, F, synth.seeds(cfg)[1], ld=ldb)).to(dev)
    rp = torch.from_numpy(rowptr).to(dev)
    ci = torch.from_numpy(colind).to(dev)
    va = torch.ones(len(colind), dtype=torch.float32, device=dev)
    C = torch.zeros((n, ldb), dtype=torch.float32, device=dev)
    C2 = torch.zeros((n, ldb), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    bm = byte_model(K, n, F)

    def timed(fn, reps=8):
        ts = []
        for i in range(3 + reps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
        return float(np.median(ts)), float(min(ts))

    # G:stages[:warps per CTA[:tma warps per CTA]]
    variants = [tuple(x.split(":")) for x in os.environ.get("SLAB_VARIANTS", "16:4,8:4").split(",")]

    def clear():
        for k in [k for k in os.environ if k.startswith("ES_SPMM_")]:
            os.environ.pop(k)

    clear()
    ms, mn = timed(lambda: es.es_spmm_run(rp, ci, va, Bd, s, 2, 0, 1, F=F, C=C))
    print(json.dumps({"variant": "fused", "plan": es.es_spmm_plan(F, ldb, ldb, Bd, C), "ms": round(ms, 3),
                      "min_ms": round(mn, 3), "algo_GBps": round(bm / ms / 1e6, 1)}), flush=True)
    for v in variants:
        g, st = v[0], v[1]
        clear()
        os.environ["ES_SPMM_SLAB"] = "1"
        os.environ["ES_SPMM_SLAB_STAGES"] = st
        os.environ["ES_SPMM_SLAB_G"] = g
        for kv in filter(None, os.environ.get("SLAB_ENV", "").split(",")):   # extra knobs, e.g. ES_SPMM_SLAB_ROWS=8
            k_, v_ = kv.split("=")
            os.environ[k_] = v_
        if len(v) > 2:
            os.environ["ES_SPMM_SLAB_CTA_WARPS"] = v[2]
        if len(v) > 3:
            os.environ["ES_SPMM_SLAB_TMA"] = v[3]
        ws = es.es_spmm_workspace(n, n, len(colind), F, ldb, s, True, device=dev)
        C2.zero_()
        ms, mn = timed(lambda: es.es_spmm_run_ex(rp, ci, va, Bd, s, 2, 0, 1, F=F, C=C2, workspace=ws))
        d = (C2[:, :F] - C[:, :F]).abs().max().item()
        rel = ((C2[:, :F] - C[:, :F]).abs() / C[:, :F].abs().clamp_min(1e-6)).max().item()
        print(json.dumps({"variant": f"slab {':'.join(v)}", "ws_MB": round(ws.numel() / 2**20, 1), "ms": round(ms, 3),
                          "min_ms": round(mn, 3), "algo_GBps": round(bm / ms / 1e6, 1),
                          "max_abs_diff_vs_fused": d, "max_rel_diff_vs_fused": rel}), flush=True)


if __name__ == "__main__":
    main()
